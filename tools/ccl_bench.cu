// Experiment harness for the tile-local union-find of the labeller (not part
// of the product).  Reads a passable bit mask (tools/data/bits_*.bin, made
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

constexpr int TW = 128, TH = 64, WPR = TW / 32, NT = TH * WPR;

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
// padded shared-memory layout: one pad word per 32 nodes, so the lanes of a
// warp (8 rows x 4 words) touching the same bit position hit distinct banks
__device__ __forceinline__ int px_(int x) { return x + (x >> 5); }
__device__ __forceinline__ int pfind(volatile int32_t* L, int x) {
  while (true) {
    const int p = L[px_(x)];
    if (p == x) return x;
    const int gp = L[px_(p)];
    if (gp == p) return p;
    L[px_(x)] = gp;
    x = gp;
  }
}
__device__ __forceinline__ int proot(const volatile int32_t* L, int x) {
  int p = L[px_(x)];
  while (p != x) {
    x = p;
    p = L[px_(x)];
  }
  return x;
}
__device__ __forceinline__ void punite(int32_t* L, int a, int b) {
  volatile int32_t* V = L;
  while (true) {
    a = pfind(V, a);
    b = pfind(V, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicMin(&L[px_(b)], a);
    if (old == b) return;
    b = old;
  }
}
__device__ __forceinline__ uint32_t run_starts(uint32_t A) { return A & ~(A << 1); }
__device__ __forceinline__ int start_of(uint32_t st, int p) {
  const uint32_t upto = (p == 31) ? 0xffffffffu : ((2u << p) - 1u);
  return 31 - __clz(st & upto);
}

// unions of the run starting at bit s of word (r, w) with the row above
template <bool PAD = false>
__device__ __forceinline__ void vertical_unions(int32_t* L, const uint32_t* bits, int r, int w,
                                                int s) {
  auto unite = [&](int a, int b) { if (PAD) punite(L, a, b); else uf_unite(L, a, b); };
  const int rw = r * WPR + w;
  const uint32_t A = bits[rw];
  const uint32_t B = bits[rw - WPR];
  const uint32_t BL = w > 0 ? bits[rw - WPR - 1] : 0u;
  const uint32_t BR = w + 1 < WPR ? bits[rw - WPR + 1] : 0u;
  const uint32_t stB = run_starts(B);
  const int base = r * TW + w * 32, bbase = base - TW;
  const uint32_t hi = 0xffffffffu << s;
  const uint32_t zer = ~A & hi;
  const uint32_t run = zer ? ((zer & (0u - zer)) - 1u) & hi : hi;
  const int n = base + s;
  uint32_t o = (run | (run << 1) | (run >> 1)) & B;
  while (o) {
    const int p = __ffs(o) - 1;
    unite(n, bbase + start_of(stB, p));
    const uint32_t upto = (p == 31) ? 0xffffffffu : ((2u << p) - 1u);
    const uint32_t zb = ~B & ~upto;
    if (!zb) break;
    o &= ~((zb & (0u - zb)) - 1u);
  }
  if ((run & 1u) && (BL >> 31)) unite(n, bbase - 32 + (31 - __clz(run_starts(BL))));
  if ((run >> 31) && (BR & 1u)) unite(n, bbase + 32);
}

template <bool PAD = false>
__device__ __forceinline__ void horizontal_union(int32_t* L, const uint32_t* bits, int r, int w) {
  const int rw = r * WPR + w;
  if ((bits[rw] & 1u) && w > 0) {
    const uint32_t Al = bits[rw - 1];
    const int a = r * TW + w * 32, b = r * TW + w * 32 - 32 + (31 - __clz(run_starts(Al)));
    if (Al >> 31) { if (PAD) punite(L, a, b); else uf_unite(L, a, b); }
  }
}

__device__ __forceinline__ int slot_row(int slot) {
  if (slot == TH - 1) return 0;
  int k = 0, cnt = TH / 2;
  while (slot >= cnt) {
    slot -= cnt;
    cnt >>= 1;
    ++k;
  }
  return (2 * slot + 1) << k;
}

// write per-pixel local root (tile pixel index) or -1
template <bool PAD = false>
__device__ void emit(const int32_t* L, const uint32_t* bits, int32_t* out, int frame, int H, int W,
                     int x0, int y0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int rw = warp; rw < NT; rw += NT / 32) {
    const int r = rw / WPR, w = rw % WPR;
    const uint32_t A = bits[rw];
    int v = -1;
    if ((A >> lane) & 1u) {
      const int n = r * TW + w * 32 + start_of(run_starts(A), lane);
      v = L[PAD ? px_(n) : n];
    }
    const int gy = y0 + r, gx = x0 + w * 32 + lane;
    if (gy < H && gx < W) out[((int64_t)frame * H + gy) * W + gx] = v;
  }
}

template <int V>
__global__ void __launch_bounds__(NT) tile_kernel(const uint32_t* __restrict__ gbits, int nsrc,
                                                  int H, int W, int WW, int32_t* out,
                                                  long long* clk) {
  __shared__ int32_t L[TH * TW + TH * TW / 32];
  __shared__ uint32_t bits[NT];
  __shared__ uint16_t lst[NT / 32][32 * 16];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH, f = blockIdx.z;
  const uint32_t* src = gbits + (size_t)(f % nsrc) * H * WW;
  long long t0 = clock64();
  {
    const int r = tid / WPR, wc = blockIdx.x * WPR + tid % WPR;
    bits[tid] = (y0 + r < H && wc < WW) ? src[(size_t)(y0 + r) * WW + wc] : 0u;
  }
  __syncthreads();
  if (V == 0 || V == 2) {
    const int r = tid / WPR, w = tid % WPR;
    const uint32_t st = run_starts(bits[tid]);
    for (uint32_t m = st; m; m &= m - 1u) L[r * TW + w * 32 + __ffs(m) - 1] = r * TW + w * 32 + __ffs(m) - 1;
    __syncthreads();
    long long ta = clock64();
    if (V == 0) {
      horizontal_union(L, bits, r, w);
      if (r > 0)
        for (uint32_t m = st; m; m &= m - 1u) vertical_unions(L, bits, r, w, __ffs(m) - 1);
    } else {
      // warp-balanced: the warp's 32 row-words' runs as one list
      const int cnt = __popc(st);
      int pre = cnt;
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, pre, d);
        if (lane >= d) pre += v;
      }
      const int total = __shfl_sync(0xffffffffu, pre, 31);
      int k = pre - cnt;
      for (uint32_t m = st; m; m &= m - 1u) lst[warp][k++] = (uint16_t)(r * TW + w * 32 + __ffs(m) - 1);
      __syncwarp();
      horizontal_union(L, bits, r, w);
      for (int i = lane; i < total; i += 32) {
        const int n = lst[warp][i];
        const int rr = n >> 7;
        if (rr > 0) vertical_unions(L, bits, rr, (n >> 5) & 3, n & 31);
      }
    }
    __syncthreads();
    long long tb = clock64();
    for (uint32_t m = st; m; m &= m - 1u) {
      const int n = r * TW + w * 32 + __ffs(m) - 1;
      L[n] = uf_root(L, n);
    }
    __syncthreads();
    long long tc = clock64();
    if (tid == 0) {
      atomicAdd(&g_phase[0], (unsigned long long)(ta - t0));
      atomicAdd(&g_phase[1], (unsigned long long)(tb - ta));
      atomicAdd(&g_phase[2], (unsigned long long)(tc - tb));
    }
  } else if (V == 4) {
    const int r = tid / WPR, w = tid % WPR;
    const uint32_t st = run_starts(bits[tid]);
    for (uint32_t m = st; m; m &= m - 1u) {
      const int n = r * TW + w * 32 + __ffs(m) - 1;
      L[px_(n)] = n;
    }
    __syncthreads();
    horizontal_union<true>(L, bits, r, w);
    if (r > 0)
      for (uint32_t m = st; m; m &= m - 1u) vertical_unions<true>(L, bits, r, w, __ffs(m) - 1);
    __syncthreads();
    for (uint32_t m = st; m; m &= m - 1u) {
      const int n = r * TW + w * 32 + __ffs(m) - 1;
      L[px_(n)] = proot(L, n);
    }
  } else if (V == 1) {
    const int r = slot_row(tid / WPR), w = tid % WPR;
    const uint32_t st = run_starts(bits[r * WPR + w]);
    for (uint32_t m = st; m; m &= m - 1u) L[r * TW + w * 32 + __ffs(m) - 1] = r * TW + w * 32 + __ffs(m) - 1;
    __syncthreads();
    horizontal_union(L, bits, r, w);
    __syncthreads();
    const int my_round = r > 0 ? __ffs(r) - 1 : -1;
    for (int k = 0; (1 << k) < TH; ++k) {
      if (my_round == k)
        for (uint32_t m = st; m; m &= m - 1u) vertical_unions(L, bits, r, w, __ffs(m) - 1);
      __syncthreads();
    }
    for (uint32_t m = st; m; m &= m - 1u) {
      const int n = r * TW + w * 32 + __ffs(m) - 1;
      L[n] = uf_root(L, n);
    }
  } else if (V == 3) {
    // pixel lanes: warp <-> row-word, lane <-> pixel; only run starts work
    for (int rw = warp; rw < NT; rw += NT / 32) {
      const uint32_t A = bits[rw];
      const int n = (rw / WPR) * TW + (rw % WPR) * 32 + lane;
      if ((run_starts(A) >> lane) & 1u) L[n] = n;
    }
    __syncthreads();
    for (int rw = warp; rw < NT; rw += NT / 32) {
      const uint32_t A = bits[rw];
      const int r = rw / WPR, w = rw % WPR;
      if (lane == 0) horizontal_union(L, bits, r, w);
      if (r > 0 && ((run_starts(A) >> lane) & 1u)) vertical_unions(L, bits, r, w, lane);
    }
    __syncthreads();
    for (int rw = warp; rw < NT; rw += NT / 32) {
      const uint32_t A = bits[rw];
      const int n = (rw / WPR) * TW + (rw % WPR) * 32 + lane;
      if ((run_starts(A) >> lane) & 1u) L[n] = uf_root(L, n);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (V == 4) emit<true>(L, bits, out, f, H, W, x0, y0);
  else emit(L, bits, out, f, H, W, x0, y0);
  if (tid == 0 && clk) clk[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t1 - t0;
}


// V5: nodes are runs of G = (row 2k | row 2k+1) ("band runs"): every band run
// is 8-connected inside its two rows, so nodes drop ~3x and rows to merge
// halve.  Node slot = band*128 + word*32 + start bit of the band run.  Roots
// are min slots; the component label (min pixel) is a min-reduction after
// compression.
constexpr int NB = TH / 2;          // bands per tile
constexpr int NT5 = NB * WPR;       // 128 threads
__global__ void __launch_bounds__(NT5) tile_kernel5(const uint32_t* __restrict__ gbits, int nsrc,
                                                    int H, int W, int WW, int32_t* out,
                                                    long long* clk) {
  __shared__ int32_t L[NB * TW];
  __shared__ int32_t M[NB * TW];
  __shared__ uint32_t bits[NT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH, f = blockIdx.z;
  const uint32_t* src = gbits + (size_t)(f % nsrc) * H * WW;
  long long t0 = clock64();
  for (int i = tid; i < NT; i += NT5) {
    const int r = i / WPR, wc = blockIdx.x * WPR + i % WPR;
    bits[i] = (y0 + r < H && wc < WW) ? src[(size_t)(y0 + r) * WW + wc] : 0u;
  }
  __syncthreads();
  const int k = tid / WPR, w = tid % WPR;
  const uint32_t A0 = bits[(2 * k) * WPR + w], A1 = bits[(2 * k + 1) * WPR + w];
  const uint32_t G = A0 | A1, stG = run_starts(G);
  const int base = k * TW + w * 32;
  for (uint32_t m = stG; m; m &= m - 1u) {
    const int n = base + __ffs(m) - 1;
    L[n] = n;
    M[n] = 0x7fffffff;
  }
  __syncthreads();
  if ((G & 1u) && w > 0) {
    const uint32_t Gl = bits[(2 * k) * WPR + w - 1] | bits[(2 * k + 1) * WPR + w - 1];
    if (Gl >> 31) uf_unite(L, base, base - 32 + (31 - __clz(run_starts(Gl))));
  }
  if (k > 0) {
    const int rb = (2 * k - 1) * WPR + w;  // row 2k-1 (second row of band k-1)
    const uint32_t B = bits[rb];
    const uint32_t Gb = bits[rb - WPR] | B, stGb = run_starts(Gb);
    const uint32_t BL = w > 0 ? bits[rb - 1] : 0u, BR = w + 1 < WPR ? bits[rb + 1] : 0u;
    const int bbase = base - TW;
    for (uint32_t m = stG; m; m &= m - 1u) {
      const int s = __ffs(m) - 1;
      const uint32_t hi = 0xffffffffu << s;
      const uint32_t zer = ~G & hi;
      const uint32_t run = zer ? ((zer & (0u - zer)) - 1u) & hi : hi;
      const uint32_t a = A0 & run;  // row-2k pixels of this band run
      if (!a) continue;
      const int n = base + s;
      uint32_t o = (a | (a << 1) | (a >> 1)) & B;
      while (o) {
        const int p = __ffs(o) - 1;
        uf_unite(L, n, bbase + start_of(stGb, p));
        const uint32_t upto = (p == 31) ? 0xffffffffu : ((2u << p) - 1u);
        const uint32_t zb = ~Gb & ~upto;
        if (!zb) break;
        o &= ~((zb & (0u - zb)) - 1u);
      }
      if ((a & 1u) && (BL >> 31)) {
        const uint32_t GbL = bits[rb - WPR - 1] | BL;
        uf_unite(L, n, bbase - 32 + (31 - __clz(run_starts(GbL))));
      }
      if ((a >> 31) && (BR & 1u)) uf_unite(L, n, bbase + 32);
    }
  }
  __syncthreads();
  for (uint32_t m = stG; m; m &= m - 1u) {
    const int n = base + __ffs(m) - 1;
    L[n] = uf_root(L, n);
  }
  __syncthreads();
  for (uint32_t m = stG; m; m &= m - 1u) {
    const int s = __ffs(m) - 1;
    const uint32_t hi = 0xffffffffu << s;
    const uint32_t zer = ~G & hi;
    const uint32_t run = zer ? ((zer & (0u - zer)) - 1u) & hi : hi;
    const uint32_t a0 = A0 & run;
    const int mp = a0 ? (2 * k) * TW + w * 32 + __ffs(a0) - 1
                      : (2 * k + 1) * TW + w * 32 + __ffs(A1 & run) - 1;
    atomicMin(&M[L[base + s]], mp);
  }
  __syncthreads();
  long long t1 = clock64();
  for (int rw = warp; rw < NT; rw += NT5 / 32) {
    const int r = rw / WPR, ww = rw % WPR;
    const int kk = r >> 1;
    const uint32_t A = bits[rw];
    const uint32_t Gk = bits[(2 * kk) * WPR + ww] | bits[(2 * kk + 1) * WPR + ww];
    int v = -1;
    if ((A >> lane) & 1u) v = M[L[kk * TW + ww * 32 + start_of(run_starts(Gk), lane)]];
    const int gy = y0 + r, gx = x0 + ww * 32 + lane;
    if (gy < H && gx < W) out[((int64_t)f * H + gy) * W + gx] = v;
  }
  if (tid == 0 && clk) clk[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(NT5) tile_kernel6(const uint32_t* __restrict__ gbits, int nsrc,
                                                    int H, int W, int WW, int32_t* out,
                                                    long long* clk) {
  __shared__ int32_t L[NB * TW];  // parents; after compression roots hold enc(min pixel) < 0
  __shared__ uint32_t bits[NT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH, f = blockIdx.z;
  const uint32_t* src = gbits + (size_t)(f % nsrc) * H * WW;
  long long t0 = clock64();
  for (int i = tid; i < NT; i += NT5) {
    const int r = i / WPR, wc = blockIdx.x * WPR + i % WPR;
    bits[i] = (y0 + r < H && wc < WW) ? src[(size_t)(y0 + r) * WW + wc] : 0u;
  }
  __syncthreads();
  const int k = tid / WPR, w = tid % WPR;
  const uint32_t A0 = bits[(2 * k) * WPR + w], A1 = bits[(2 * k + 1) * WPR + w];
  const uint32_t G = A0 | A1, stG = run_starts(G);
  const int base = k * TW + w * 32;
  for (uint32_t m = stG; m; m &= m - 1u) {
    const int n = base + __ffs(m) - 1;
    L[n] = n;
  }
  __syncthreads();
  if ((G & 1u) && w > 0) {
    const uint32_t Gl = bits[(2 * k) * WPR + w - 1] | bits[(2 * k + 1) * WPR + w - 1];
    if (Gl >> 31) uf_unite(L, base, base - 32 + (31 - __clz(run_starts(Gl))));
  }
  if (k > 0) {
    const int rb = (2 * k - 1) * WPR + w;  // row 2k-1 (second row of band k-1)
    const uint32_t B = bits[rb];
    const uint32_t Gb = bits[rb - WPR] | B, stGb = run_starts(Gb);
    const uint32_t BL = w > 0 ? bits[rb - 1] : 0u, BR = w + 1 < WPR ? bits[rb + 1] : 0u;
    const int bbase = base - TW;
    for (uint32_t m = stG; m; m &= m - 1u) {
      const int s = __ffs(m) - 1;
      const uint32_t hi = 0xffffffffu << s;
      const uint32_t zer = ~G & hi;
      const uint32_t run = zer ? ((zer & (0u - zer)) - 1u) & hi : hi;
      const uint32_t a = A0 & run;  // row-2k pixels of this band run
      if (!a) continue;
      const int n = base + s;
      uint32_t o = (a | (a << 1) | (a >> 1)) & B;
      while (o) {
        const int p = __ffs(o) - 1;
        uf_unite(L, n, bbase + start_of(stGb, p));
        const uint32_t upto = (p == 31) ? 0xffffffffu : ((2u << p) - 1u);
        const uint32_t zb = ~Gb & ~upto;
        if (!zb) break;
        o &= ~((zb & (0u - zb)) - 1u);
      }
      if ((a & 1u) && (BL >> 31)) {
        const uint32_t GbL = bits[rb - WPR - 1] | BL;
        uf_unite(L, n, bbase - 32 + (31 - __clz(run_starts(GbL))));
      }
      if ((a >> 31) && (BR & 1u)) uf_unite(L, n, bbase + 32);
    }
  }
  __syncthreads();
  for (uint32_t m = stG; m; m &= m - 1u) {
    const int n = base + __ffs(m) - 1;
    L[n] = uf_root(L, n);
  }
  __syncthreads();
  for (uint32_t m = stG; m; m &= m - 1u) {
    const int s = __ffs(m) - 1;
    const uint32_t hi = 0xffffffffu << s;
    const uint32_t zer = ~G & hi;
    const uint32_t run = zer ? ((zer & (0u - zer)) - 1u) & hi : hi;
    const uint32_t a0 = A0 & run;
    const int mp = a0 ? (2 * k) * TW + w * 32 + __ffs(a0) - 1
                      : (2 * k + 1) * TW + w * 32 + __ffs(A1 & run) - 1;
    const int pr = L[base + s];
    atomicMin(&L[pr >= 0 ? pr : base + s], mp - 0x40000000);
  }
  __syncthreads();
  long long t1 = clock64();
  for (int rw = warp; rw < NT; rw += NT5 / 32) {
    const int r = rw / WPR, ww = rw % WPR;
    const int kk = r >> 1;
    const uint32_t A = bits[rw];
    const uint32_t Gk = bits[(2 * kk) * WPR + ww] | bits[(2 * kk + 1) * WPR + ww];
    int v = -1;
    if ((A >> lane) & 1u) {
      const int pr = L[kk * TW + ww * 32 + start_of(run_starts(Gk), lane)];
      v = (pr >= 0 ? L[pr] : pr) + 0x40000000;
    }
    const int gy = y0 + r, gx = x0 + ww * 32 + lane;
    if (gy < H && gx < W) out[((int64_t)f * H + gy) * W + gx] = v;
  }
  if (tid == 0 && clk) clk[((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t1 - t0;
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
  cudaMalloc(&dclk, ntiles * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](int v, long long* clk) {
    switch (v) {
      case 0: tile_kernel<0><<<grid, NT>>>(dbits, nsrc, H, W, WW, dout, clk); break;
      case 1: tile_kernel<1><<<grid, NT>>>(dbits, nsrc, H, W, WW, dout, clk); break;
      case 2: tile_kernel<2><<<grid, NT>>>(dbits, nsrc, H, W, WW, dout, clk); break;
      case 3: tile_kernel<3><<<grid, NT>>>(dbits, nsrc, H, W, WW, dout, clk); break;
      case 4: tile_kernel<4><<<grid, NT>>>(dbits, nsrc, H, W, WW, dout, clk); break;
      case 5: tile_kernel5<<<grid, NT5>>>(dbits, nsrc, H, W, WW, dout, clk); break;
      case 6: tile_kernel6<<<grid, NT5>>>(dbits, nsrc, H, W, WW, dout, clk); break;
    }
  };
  const char* names[] = {"V0 concurrent (row,word)", "V1 rounds+remap", "V2 warp-balanced list",
                         "V3 pixel lanes (run starts)", "V4 = V0 + padded smem",
                         "V5 band runs (2-row nodes)", "V6 = V5, one smem array"};
  std::vector<int32_t> got((size_t)nsrc * H * W);
  std::vector<long long> clk(ntiles);
  for (int v = 0; v < 7; ++v) {
    run(v, dclk);
    cudaMemcpy(got.data(), dout, got.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(clk.data(), dclk, ntiles * 8, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (size_t i = 0; i < got.size(); ++i) bad += got[i] != ref[i];
    double cs = 0, cmax = 0;
    for (auto c : clk) {
      cs += c;
      if (c > cmax) cmax = c;
    }
    for (int i = 0; i < 3; ++i) run(v, nullptr);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int i = 0; i < reps; ++i) run(v, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long ph[4] = {0, 0, 0, 0}, fi = 0, fc = 0;
    cudaMemcpyFromSymbol(ph, g_phase, sizeof(ph));
    cudaMemcpyFromSymbol(&fi, g_find_it, 8);
    cudaMemcpyFromSymbol(&fc, g_find_calls, 8);
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_phase, z, sizeof(z));
    cudaMemcpyToSymbol(g_find_it, z, 8);
    cudaMemcpyToSymbol(g_find_calls, z, 8);
    const double nrun = 14.0 * (3 + 10);  // per-tile calls across the runs above
    printf("   phases per tile (clk): init %.0f union %.0f compress %.0f ; finds %.3g iters %.3g (%.2f/find)\n",
           ph[0] / (double)ntiles / 14, ph[1] / (double)ntiles / 14, ph[2] / (double)ntiles / 14,
           (double)fc, (double)fi, fc ? (double)fi / fc : 0.0);
    (void)nrun;
    printf("%-30s %8.2f us/frame  tile clk mean %8.0f max %8.0f  mismatches %zu  %s\n", names[v],
           ms * 1e3 / reps / B, cs / ntiles, cmax, bad, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
