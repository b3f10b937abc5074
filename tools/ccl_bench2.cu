// Experiment harness (not part of the product): variants of the band-run
// tile union-find at the product's 128x128 tile (ccl_bench.cu holds the
// earlier 128x64 variants V0-V6).  Reads a passable bit mask (tools/data/bits_*.bin, made
// from oracle passable sets of C3/C4 frames), runs several tile-local
// labelling variants over a 64-frame batch, checks they agree with a CPU
// flood fill per tile, and prints per-variant kernel time.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -o tools/ccl_bench tools/ccl_bench.cu && tools/ccl_bench tools/data/bits_c3.bin
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

constexpr int TW = 128, TH = 128, WPR = TW / 32, NT = TH * WPR;

__device__ unsigned long long g_find_it, g_find_calls, g_unite_calls, g_phase[4];
__device__ __forceinline__ int uf_find(volatile int32_t* L, int x) {
#ifdef COUNT
  atomicAdd(&g_find_calls, 1ull);
#endif
  while (true) {
#ifdef COUNT
    atomicAdd(&g_find_it, 1ull);
#endif
    const int p = L[x];
    if (p == x) return x;
    const int gp = L[p];
    if (gp == p) return p;
    L[x] = gp;
    x = gp;
  }
}
__device__ __forceinline__ int uf_root(const volatile int32_t* L, int x) {
  int p = L[x];
  while (p != x) {
    x = p;
    p = L[x];
  }
  return x;
}
__device__ __forceinline__ void uf_unite(int32_t* L, int a, int b) {
  volatile int32_t* V = L;
  while (true) {
    a = uf_find(V, a);
    b = uf_find(V, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(&L[b], a);
    if (old == b) return;
    b = old;
  }
}

__device__ __forceinline__ uint32_t run_starts(uint32_t A) { return A & ~(A << 1); }
__device__ __forceinline__ int start_of(uint32_t st, int p) {
  const uint32_t upto = (p == 31) ? 0xffffffffu : ((2u << p) - 1u);
  return 31 - __clz(st & upto);
}
__device__ __forceinline__ uint32_t run_mask(uint32_t G, int s) {
  const uint32_t hi = 0xffffffffu << s;
  const uint32_t zer = ~G & hi;
  return zer ? ((zer & (0u - zer)) - 1u) & hi : hi;
}

template <bool PAD>
__device__ __forceinline__ int ix(int n) { return PAD ? n + (n >> 5) : n; }

// uf over an index-mapped array: indices are logical slots
template <bool PAD>
__device__ __forceinline__ int f_find(volatile int32_t* L, int x) {
  while (true) {
    const int p = L[ix<PAD>(x)];
    if (p == x) return x;
    const int gp = L[ix<PAD>(p)];
    if (gp == p) return p;
    L[ix<PAD>(x)] = gp;
    x = gp;
  }
}
template <bool PAD>
__device__ __forceinline__ int f_root(const volatile int32_t* L, int x) {
  int p = L[ix<PAD>(x)];
  while (p != x) {
    x = p;
    p = L[ix<PAD>(x)];
  }
  return x;
}
template <bool PAD>
__device__ __forceinline__ void f_unite(int32_t* L, int a, int b) {
  volatile int32_t* V = L;
  while (true) {
    a = f_find<PAD>(V, a);
    b = f_find<PAD>(V, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(&L[ix<PAD>(b)], a);
    if (old == b) return;
    b = old;
  }
}

constexpr int NB = TH / 2, NTB = NB * WPR;  // 64 bands, 256 threads
constexpr int NSLOT = NB * TW;

// HALVE: path halving in the compress phase; DIRECT: a band run's initial
// parent is its first overlapping run of the band above (same word), so
// unions handle only the extra links; PAD: one pad word per 32 slots
template <bool HALVE, bool DIRECT, bool PAD>
__global__ void __launch_bounds__(NTB) tile_kernel7(const uint32_t* __restrict__ gbits, int nsrc,
                                                    int H, int W, int WW, int32_t* out,
                                                    long long* clk) {
  extern __shared__ int32_t L[];
  __shared__ uint32_t bits[NT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH, f = blockIdx.z;
  const uint32_t* src = gbits + (size_t)(f % nsrc) * H * WW;
  long long t0 = clock64(), ts[6];
  for (int i = tid; i < NT; i += NTB) {
    const int r = i / WPR, wc = blockIdx.x * WPR + i % WPR;
    bits[i] = (y0 + r < H && wc < WW) ? src[(size_t)(y0 + r) * WW + wc] : 0u;
  }
  __syncthreads();
  ts[0] = clock64();
  const int k = tid / WPR, w = tid % WPR;
  const uint32_t A0 = bits[(2 * k) * WPR + w], A1 = bits[(2 * k + 1) * WPR + w];
  const uint32_t G = A0 | A1, stG = run_starts(G);
  const int base = k * TW + w * 32;
  const int rb = (2 * k - 1) * WPR + w;
  const uint32_t B = k > 0 ? bits[rb] : 0u;
  const uint32_t Gb = k > 0 ? bits[rb - WPR] | B : 0u, stGb = run_starts(Gb);
  const int bbase = base - TW;
  for (uint32_t m = stG; m; m &= m - 1u) {
    const int s = __ffs(m) - 1, n = base + s;
    int par = n;
    if (DIRECT && k > 0) {
      const uint32_t a = A0 & run_mask(G, s);
      const uint32_t o = (a | (a << 1) | (a >> 1)) & B;
      if (o) par = bbase + start_of(stGb, __ffs(o) - 1);
    }
    L[ix<PAD>(n)] = par;
  }
  __syncthreads();
  ts[1] = clock64();
  if ((G & 1u) && w > 0) {
    const uint32_t Gl = bits[(2 * k) * WPR + w - 1] | bits[(2 * k + 1) * WPR + w - 1];
    if (Gl >> 31) f_unite<PAD>(L, base, base - 32 + (31 - __clz(run_starts(Gl))));
  }
  if (k > 0) {
    const uint32_t BL = w > 0 ? bits[rb - 1] : 0u, BR = w + 1 < WPR ? bits[rb + 1] : 0u;
    for (uint32_t m = stG; m; m &= m - 1u) {
      const int s = __ffs(m) - 1;
      const uint32_t a = A0 & run_mask(G, s);
      if (!a) continue;
      const int n = base + s;
      uint32_t o = (a | (a << 1) | (a >> 1)) & B;
      bool first = true;
      while (o) {
        const int p = __ffs(o) - 1;
        if (!(DIRECT && first)) f_unite<PAD>(L, n, bbase + start_of(stGb, p));
        first = false;
        const uint32_t upto = (p == 31) ? 0xffffffffu : ((2u << p) - 1u);
        const uint32_t zb = ~Gb & ~upto;
        if (!zb) break;
        o &= ~((zb & (0u - zb)) - 1u);
      }
      if ((a & 1u) && (BL >> 31)) {
        const uint32_t GbL = bits[rb - WPR - 1] | BL;
        f_unite<PAD>(L, n, bbase - 32 + (31 - __clz(run_starts(GbL))));
      }
      if ((a >> 31) && (BR & 1u)) f_unite<PAD>(L, n, bbase + 32);
    }
  }
  __syncthreads();
  ts[2] = clock64();
  for (uint32_t m = stG; m; m &= m - 1u) {
    const int n = base + __ffs(m) - 1;
    L[ix<PAD>(n)] = HALVE ? f_find<PAD>(L, n) : f_root<PAD>(L, n);
  }
  __syncthreads();
  ts[3] = clock64();
  for (uint32_t m = stG; m; m &= m - 1u) {
    const int s = __ffs(m) - 1;
    const uint32_t run = run_mask(G, s);
    const uint32_t a0 = A0 & run;
    const int mp = a0 ? (2 * k) * TW + w * 32 + __ffs(a0) - 1
                      : (2 * k + 1) * TW + w * 32 + __ffs(A1 & run) - 1;
    const int pr = L[ix<PAD>(base + s)];
    atomicMin(&L[ix<PAD>(pr >= 0 ? pr : base + s)], mp - 0x40000000);
  }
  __syncthreads();
  long long t1 = clock64();
  ts[4] = t1;
  for (int rw = warp; rw < NT; rw += NTB / 32) {
    const int r = rw / WPR, ww = rw % WPR;
    const int kk = r >> 1;
    const uint32_t A = bits[rw];
    const uint32_t Gk = bits[(2 * kk) * WPR + ww] | bits[(2 * kk + 1) * WPR + ww];
    int v = -1;
    if ((A >> lane) & 1u) {
      const int pr = L[ix<PAD>(kk * TW + ww * 32 + start_of(run_starts(Gk), lane))];
      v = (pr >= 0 ? L[ix<PAD>(pr)] : pr) + 0x40000000;
    }
    const int gy = y0 + r, gx = x0 + ww * 32 + lane;
    if (gy < H && gx < W) out[((int64_t)f * H + gy) * W + gx] = v;
  }
  __syncthreads();
  ts[5] = clock64();
  if (tid == 0 && clk) {
    const size_t t = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    clk[t * 7] = t1 - t0;
    long long prev = t0;
    for (int i = 0; i < 6; ++i) {
      clk[t * 7 + 1 + i] = ts[i] - prev;
      prev = ts[i];
    }
  }
}

// CPU reference: per-tile 8-connected flood fill, label = min tile pixel index
static void cpu_tiles(const std::vector<uint32_t>& bits, int nsrc, int H, int W, int WW,
                      std::vector<int32_t>& out) {
  out.assign((size_t)nsrc * H * W, -1);
  std::vector<int> stack;
  for (int f = 0; f < nsrc; ++f)
    for (int ty = 0; ty * TH < H; ++ty)
      for (int tx = 0; tx * TW < W; ++tx) {
        auto P = [&](int x, int y) {
          if (x < 0 || y < 0 || x >= TW || y >= TH) return false;
          const int gx = tx * TW + x, gy = ty * TH + y;
          if (gx >= W || gy >= H) return false;
          return ((bits[((size_t)f * H + gy) * WW + gx / 32] >> (gx % 32)) & 1u) != 0;
        };
        std::vector<int> lab(TW * TH, -1);
        for (int y = 0; y < TH; ++y)
          for (int x = 0; x < TW; ++x) {
            if (!P(x, y) || lab[y * TW + x] >= 0) continue;
            const int id = y * TW + x;
            stack.assign(1, id);
            lab[id] = id;
            while (!stack.empty()) {
              const int c = stack.back();
              stack.pop_back();
              const int cx = c % TW, cy = c / TW;
              for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx)
                  if (P(cx + dx, cy + dy) && lab[(cy + dy) * TW + cx + dx] < 0) {
                    lab[(cy + dy) * TW + cx + dx] = id;
                    stack.push_back((cy + dy) * TW + cx + dx);
                  }
            }
          }
        for (int y = 0; y < TH; ++y)
          for (int x = 0; x < TW; ++x) {
            const int gx = tx * TW + x, gy = ty * TH + y;
            if (gx < W && gy < H) out[((size_t)f * H + gy) * W + gx] = lab[y * TW + x];
          }
      }
}

int main(int argc, char** argv) {
  if (argc < 2) return 1;
  FILE* fp = fopen(argv[1], "rb");
  int hdr[4];
  if (!fp || fread(hdr, 4, 4, fp) != 4) return 2;
  const int nsrc = hdr[0], H = hdr[1], W = hdr[2], WW = hdr[3];
  std::vector<uint32_t> bits((size_t)nsrc * H * WW);
  if (fread(bits.data(), 4, bits.size(), fp) != bits.size()) return 3;
  fclose(fp);
  const int B = argc > 2 ? atoi(argv[2]) : 64;
  std::vector<int32_t> ref;
  cpu_tiles(bits, nsrc, H, W, WW, ref);
  uint32_t* dbits;
  int32_t* dout;
  long long* dclk;
  cudaMalloc(&dbits, bits.size() * 4);
  cudaMemcpy(dbits, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&dout, (size_t)B * H * W * 4);
  dim3 grid((W + TW - 1) / TW, (H + TH - 1) / TH, B);
  const size_t ntiles = (size_t)grid.x * grid.y * grid.z;
  cudaMalloc(&dclk, ntiles * 8 * 7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t sm = (NSLOT + NSLOT / 32) * 4;
#define SET(...) cudaFuncSetAttribute(__VA_ARGS__, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)
  SET(tile_kernel7<false, false, false>); SET(tile_kernel7<true, false, false>);
  SET(tile_kernel7<false, true, false>); SET(tile_kernel7<true, true, false>);
  SET(tile_kernel7<true, true, true>); SET(tile_kernel7<false, false, true>);
  auto run = [&](int v, long long* clk) {
    switch (v) {
      case 0: tile_kernel7<false, false, false><<<grid, NTB, sm>>>(dbits, nsrc, H, W, WW, dout, clk); break;
      case 1: tile_kernel7<true, false, false><<<grid, NTB, sm>>>(dbits, nsrc, H, W, WW, dout, clk); break;
      case 2: tile_kernel7<false, true, false><<<grid, NTB, sm>>>(dbits, nsrc, H, W, WW, dout, clk); break;
      case 3: tile_kernel7<true, true, false><<<grid, NTB, sm>>>(dbits, nsrc, H, W, WW, dout, clk); break;
      case 4: tile_kernel7<true, true, true><<<grid, NTB, sm>>>(dbits, nsrc, H, W, WW, dout, clk); break;
      case 5: tile_kernel7<false, false, true><<<grid, NTB, sm>>>(dbits, nsrc, H, W, WW, dout, clk); break;
    }
  };
  const char* names[] = {"W0 product (128x128)", "W1 + halving compress", "W2 + direct init",
                         "W3 halving + direct", "W4 halving + direct + pad", "W5 pad only"};
  std::vector<int32_t> got((size_t)nsrc * H * W);
  std::vector<long long> clk(ntiles * 7);
  for (int v = 0; v < 6; ++v) {
    run(v, dclk);
    cudaMemcpy(got.data(), dout, got.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(clk.data(), dclk, ntiles * 8 * 7, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (size_t i = 0; i < got.size(); ++i) bad += got[i] != ref[i];
    double cs = 0, cmax = 0, ph[6] = {0, 0, 0, 0, 0, 0};
    for (size_t t = 0; t < ntiles; ++t) {
      const double c = (double)clk[t * 7];
      cs += c;
      if (c > cmax) cmax = c;
      for (int i = 0; i < 6; ++i) ph[i] += (double)clk[t * 7 + 1 + i];
    }
    printf("   phases (clk/tile): load %.0f init %.0f union %.0f compress %.0f min %.0f out %.0f\n",
           ph[0] / ntiles, ph[1] / ntiles, ph[2] / ntiles, ph[3] / ntiles, ph[4] / ntiles,
           ph[5] / ntiles);
    for (int i = 0; i < 3; ++i) run(v, nullptr);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) run(v, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-30s %8.2f us/frame  tile clk mean %8.0f max %8.0f  mismatches %zu  %s\n", names[v],
           ms * 1e3 / reps / B, cs / ntiles, cmax, bad, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
