// Memory skeleton of the fused pass (fixed_square_kernel): the same items
// (128 columns x 16 rows of 2048x1024 frames), TMA 3D input tiles with halo,
// a padded row-major staging tile written by 256 threads (12 x 16-B shared
// stores each, the pass-H pattern) and one bulk copy per output row -- no
// arithmetic.  Variants probe what the memory pipeline itself can reach:
//
//   NIN      input buffers (2 = one item prefetched, 3 = two)
//   EXTRA    extra shared memory per CTA (the product's (C, Rr) array is 37 KB:
//            EXTRA = 37 KB reproduces its 2 CTAs/SM, 0 lets 3 fit)
//   WRITE    the staging tile written by the threads (else left as is)
//   LOAD     input tiles loaded at all
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2504_15121_b200/csrc -I include -o skel_bw tools/ubench/skel_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "sn_common.cuh"

using namespace sn;

// plain (no cache hint) bulk row copy shared -> global
__device__ __forceinline__ void bulk_store_1d(void* gdst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e = (x);                                                      \
    if (e != cudaSuccess) {                                                   \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));        \
      return 1;                                                               \
    }                                                                         \
  } while (0)

constexpr int kTW = 128, kG = 16, R = 4;
constexpr int NR = kG + 2 * R, BW = 140;
constexpr int kRowPitch = kTW * 24 + 16;
constexpr int STAGE_BYTES = kG * kRowPitch;
constexpr int IN_BYTES = NR * BW * 4;
constexpr int kThreads = 320, kStoreTid = 256;

template <int NIN, bool WRITE, bool LOAD, bool STORE, int LMODE = 0, int SMODE = 0>
__global__ void __launch_bounds__(kThreads, 2)
    skel_kernel(const __grid_constant__ CUtensorMap in_map, float* __restrict__ out6, int W, int H,
                int n_items, int tiles_x, int tiles_y, int extra, const float* __restrict__ in) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  const uint32_t stage_base = smem_u32(smem);
  uint8_t* inb = smem + STAGE_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(inb + NIN * IN_BYTES + extra);
  const int tid = threadIdx.x;
  auto coords = [&](int item, int& x0, int& y0, int& bz) {
    x0 = (item % tiles_x) * kTW;
    const int r = item / tiles_x;
    y0 = (r % tiles_y) * kG;
    bz = r / tiles_y;
  };
  auto load = [&](int item, int buf) {
    int x0, y0, bz;
    coords(item, x0, y0, bz);
    mbar_arrive_expect_tx(bar + buf, IN_BYTES);
    tma_load_3d(inb + buf * IN_BYTES, &in_map, bar + buf, (x0 - R) & ~3, y0 - R, bz);
  };
  if (tid == 0) {
    for (int b = 0; b < NIN; ++b) mbar_init(bar + b, 1);
    fence_mbar_init();
    if (LOAD && LMODE == 0)
      for (int b = 0; b < NIN - 1; ++b)
        if (blockIdx.x + b * gridDim.x < n_items) load(blockIdx.x + b * gridDim.x, b);
  }
  // LSU loads: thread (h, c) holds the 16 rows of column c, half h, of the next item
  const int lh = tid >= 160 ? 1 : 0, lc = tid - lh * 160;
  float pre[16];
  auto lsu_load = [&](int item) {
    int x0, y0, bz;
    coords(item, x0, y0, bz);
    const int gx = min(max(x0 - R + lc, 0), W - 1);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int gy = min(max(y0 - R + lh * 8 + i, 0), H - 1);
      pre[i] = lc < 136 ? __ldg(in + ((int64_t)bz * H + gy) * W + gx) : 0.0f;
    }
  };
  if (LOAD && LMODE == 1) lsu_load(blockIdx.x);
  if (LOAD && LMODE == 2) {  // the first item's tile (any threads; zeros suffice here)
    float4* t = reinterpret_cast<float4*>(inb);
    for (int v = tid; v < NR * (BW / 4); v += kThreads) t[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  int it = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
    const int buf = it % NIN;
    const int nxt = item + (NIN - 1) * gridDim.x;
    if (LOAD && tid == 0 && nxt < n_items) load(nxt, (it + NIN - 1) % NIN);
    int x0, y0, bz;
    coords(item, x0, y0, bz);
    float v = 1.0f;
    if (LOAD && LMODE == 0) {
      mbar_wait(bar + buf, (uint32_t)(it / NIN) & 1u);
      v = reinterpret_cast<const float*>(inb + buf * IN_BYTES)[tid % (NR * BW)];
    }
    if (LOAD && LMODE == 1) {
      // this item's columns from registers into the input tile, then the next item's loads
      float* t = reinterpret_cast<float*>(inb + buf * IN_BYTES);
      if (lc < 136) {
#pragma unroll
        for (int i = 0; i < 16; ++i) t[(lh * 8 + i) * BW + lc] = pre[i];
      }
      if (item + (int)gridDim.x < n_items) lsu_load(item + gridDim.x);
      v = t[tid % (NR * BW)];
    }
    if (LOAD && LMODE == 2) v = reinterpret_cast<const float*>(inb + buf * IN_BYTES)[tid % (NR * BW)];
    if (SMODE == 0 && tid >= kStoreTid && tid < kStoreTid + kG) bulk_wait_read0();
    __syncthreads();
    if (LOAD && LMODE == 2 && tid >= kStoreTid && item + (int)gridDim.x < n_items) {
      // warps 8-9 (idle in pass H) load the next item's tile through the LSU
      int nx0, ny0, nbz;
      coords(item + gridDim.x, nx0, ny0, nbz);
      float4* t = reinterpret_cast<float4*>(inb + ((it + 1) % NIN) * IN_BYTES);
      const int l = tid - kStoreTid;
      const int tx0 = (nx0 - R) & ~3;
      constexpr int NV = NR * (BW / 4);  // 840 vectors
      float4 r[14];
#pragma unroll
      for (int k = 0; k < 14; ++k) {
        const int v = l + 64 * k;
        r[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (v < NV) {
          const int row = v / (BW / 4), cv = v - row * (BW / 4);
          const int gy = ny0 - R + row, gx = tx0 + 4 * cv;
          if (gy >= 0 && gy < H && gx >= 0 && gx + 4 <= W)
            r[k] = __ldg(reinterpret_cast<const float4*>(in + ((int64_t)nbz * H + gy) * W + gx));
        }
      }
#pragma unroll
      for (int k = 0; k < 14; ++k)
        if (l + 64 * k < NV) t[l + 64 * k] = r[k];
    }
    if (WRITE && tid < 256) {
      const int g = tid & 15, q = tid >> 4;
      const uint32_t row_a = stage_base + (uint32_t)g * kRowPitch + (uint32_t)q * 192u;
#pragma unroll
      for (int c = 0; c < 12; ++c) st_shared_v4(row_a + c * 16u, v, v, v, v);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (STORE && SMODE == 1 && tid >= kStoreTid) {
      // warps 8-9 copy the staging tile out: 16 rows x 192 16-B chunks
      const int l = tid - kStoreTid;
      for (int b = 0; b < kG; ++b) {
        if (y0 + b >= H) break;
        float4* dst = reinterpret_cast<float4*>(out6 + (((int64_t)bz * H + y0 + b) * W + x0) * 6);
        const float4* src = reinterpret_cast<const float4*>(smem + (size_t)b * kRowPitch);
#pragma unroll
        for (int c = 0; c < 3; ++c) dst[l + 64 * c] = src[l + 64 * c];
      }
    }
    if (STORE && SMODE == 0 && tid >= kStoreTid && tid < kStoreTid + kG) {
      const int b = tid - kStoreTid;
      if (y0 + b < H)
        bulk_store_1d(out6 + (((int64_t)bz * H + y0 + b) * W + x0) * 6, smem + (size_t)b * kRowPitch,
                      (uint32_t)kTW * 24u);
      bulk_commit();
    }
  }
  if (tid >= kStoreTid && tid < kStoreTid + kG) bulk_wait0();
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main() {
  const int B = 64, H = 1024, W = 2048;
  const long px = (long)B * H * W;
  float *in, *out;
  CK(cudaMalloc(&in, px * 4));
  CK(cudaMalloc(&out, px * 24));
  CK(cudaMemset(in, 0, px * 4));
  CK(cudaMemset(out, 0, px * 24));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q));
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
  cuuint32_t box[3] = {BW, NR, 1}, es[3] = {1, 1, 1};
  if (((EncodeFn)fnp)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, in, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  const int tiles_x = W / kTW, tiles_y = H / kG, n_items = tiles_x * tiles_y * B;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern, int nin, int extra) -> int {
    const int smem = STAGE_BYTES + nin * IN_BYTES + extra + 64 + 128;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem));
    const int grid = per_sm * sms;
    auto launch = [&] {
      kern<<<grid, kThreads, smem>>>(map, out, W, H, n_items, tiles_x, tiles_y, extra, in);
    };
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    float tot = 0;
    const int n = 10;
    cudaEventRecord(e0);
    for (int i = 0; i < n; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&tot, e0, e1);
    const double us = tot * 1000.0 / n / B;
    printf("%-34s smem %6d B  %d CTA/SM  %6.2f us/frame  %6.0f GB/s (28 B/px)\n", name, smem, per_sm,
           us, 28.0 * H * W / us / 1e3);
    return cudaGetLastError();
  };
  const int CR = 136 * 17 * 16;  // the product's (C, Rr) array
  run("skeleton (product shape)", skel_kernel<2, true, true, true>, 2, CR);
  run("skeleton, no staging writes", skel_kernel<2, false, true, true>, 2, CR);
  run("stores only", skel_kernel<2, true, false, true>, 2, CR);
  run("loads only", skel_kernel<2, true, true, false>, 2, CR);
  run("skeleton, 3 input buffers", skel_kernel<3, true, true, true>, 3, CR - IN_BYTES - 256);
  run("skeleton, no CR (3 CTA/SM)", skel_kernel<2, true, true, true>, 2, 0);
  run("skeleton, no CR, 3 input buffers", skel_kernel<3, true, true, true>, 3, 0);
  run("stores only, no CR", skel_kernel<2, true, false, true>, 2, 0);
  run("loads only, 3 input buffers", skel_kernel<3, true, true, false>, 3, CR - IN_BYTES - 256);
  run("skeleton, loader warps 8-9 (LSU)", skel_kernel<2, true, true, true, 2>, 2, CR);
  run("loads only, loader warps 8-9", skel_kernel<2, true, true, false, 2>, 2, CR);
  run("stores only, LSU (warps 8-9)", skel_kernel<2, true, false, true, 0, 1>, 2, CR);
  run("skeleton, LSU stores", skel_kernel<2, true, true, true, 0, 1>, 2, CR);
  run("loads only, LSU", skel_kernel<2, true, true, false, 1>, 2, CR);
  run("skeleton, LSU loads", skel_kernel<2, true, true, true, 1>, 2, CR);
  run("skeleton, LSU loads + stores", skel_kernel<2, true, true, true, 1, 1>, 2, CR);
  CK(cudaDeviceSynchronize());
  return 0;
}
