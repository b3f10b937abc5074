// HBM ceiling for the fused pass's traffic mix: read 4 B/px, write 24 B/px
// (1:6), with no arithmetic -- how close to the copy peak of
// MEASURED_PEAKS.json (1:1 mix) can a streaming kernel get on this mix?
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mix_bw mix_bw.cu && ./mix_bw
//
// Variants (each over 64 C3 frames = 134 M px, 3.76 GB, best of 20 after warm-up):
//   copy      1:1 float4 copy (the MEASURED_PEAKS method, for calibration)
//   mix       per warp: 1 coalesced float4 load of 128 px, 6 coalesced float4
//             stores of the 3 KB record block (grid-stride, 2 items unrolled)
//   mix_cs    the same with st.global.cs (streaming / evict-first)
//   write     24 B/px of stores only
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));          \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, long n4) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
    b[i] = a[i];
}

template <bool CS, bool READ>
__global__ void mix_k(const float4* __restrict__ in, float4* __restrict__ out, long n_items) {
  // item = 128 px: 32 float4 in, 192 float4 out
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  for (long it = warp; it < n_items; it += 2 * nw) {
    const long it2 = it + nw;
    float4 v0 = make_float4(1.f, 2.f, 3.f, 4.f), v1 = v0;
    if (READ) {
      v0 = in[it * 32 + lane];
      if (it2 < n_items) v1 = in[it2 * 32 + lane];
    }
    float4* o0 = out + it * 192 + lane;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      if (CS) __stcs(o0 + 32 * k, v0);
      else o0[32 * k] = v0;
    }
    if (it2 < n_items) {
      float4* o1 = out + it2 * 192 + lane;
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        if (CS) __stcs(o1 + 32 * k, v1);
        else o1[32 * k] = v1;
      }
    }
  }
}

int main() {
  const long px = 64L * 2048 * 1024;
  float4 *in, *out;
  CK(cudaMalloc(&in, px * 4));
  CK(cudaMalloc(&out, px * 24));
  CK(cudaMemset(in, 0, px * 4));
  CK(cudaMemset(out, 0, px * 24));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, double bytes, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    float best = 1e30f;
    for (int i = 0; i < 20; ++i) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("%-28s %8.3f ms  %7.1f GB/s  (%.2f us per 2048x1024 frame)\n", name, best,
           bytes / best / 1e6, best * 1000.0 / 64.0 * (bytes / (px * 28.0)));
    return cudaGetLastError();
  };
  const long n_items = px / 128;
  for (int per_sm : {8, 16, 32}) {
    const int grid = sms * per_sm;
    char nm[64];
    snprintf(nm, sizeof nm, "copy 1:1 (grid %d/SM)", per_sm);
    timeit(nm, 2.0 * px * 12, [&] { copy_k<<<grid, 256>>>(out, out + px * 12 / 16, px * 12 / 16); });
    snprintf(nm, sizeof nm, "mix 4:24 (grid %d/SM)", per_sm);
    timeit(nm, px * 28.0, [&] { mix_k<false, true><<<grid, 256>>>(in, out, n_items); });
    snprintf(nm, sizeof nm, "mix_cs 4:24 (grid %d/SM)", per_sm);
    timeit(nm, px * 28.0, [&] { mix_k<true, true><<<grid, 256>>>(in, out, n_items); });
    snprintf(nm, sizeof nm, "write 24 (grid %d/SM)", per_sm);
    timeit(nm, px * 24.0, [&] { mix_k<false, false><<<grid, 256>>>(in, out, n_items); });
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
