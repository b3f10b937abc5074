// Passable-set predicate and connected-component labelling for sm_100a.
//
// Predicate (bit-exact with the reference): depth
// z = (fx*b)/d valid iff d finite, d > 0 and z finite (geometry.py:39-45,
// 169-172); edge e = |((((4c - left) - right) - up) - down)| evaluated in
// numpy's left-to-right order with correctly rounded fp64 operations
// (adaptive.py:80-97), valid only at interior pixels with all five depths
// valid; passable = edge valid and e <= t (the ST ray test,
// adaptive.py:130-132, 218-221).  The labeller evaluates it as an fp32
// filter with a rigorous error bound and falls back to the exact fp64
// evaluation only when |e32 - t| is inside the bound, so every decision is
// the fp64 decision (see fast_passable below).
//
// Labelling (no reference function): 8-connected
// components of the passable set, canonical label = smallest raster index in
// the component.  The passable set is a BIT mask (one uint32 word per 32
// pixels of a row) and the union-find runs over word-runs (maximal runs of
// set bits inside one word), not pixels: ~4x fewer nodes and unions than a
// pixel union-find on street scenes.  Every link goes from the larger node
// to the smaller (atomicMin), so a root is always its component's minimum
// and the result is independent of scheduling.  Three launches per batch:
//
//   1. ccl_tile_kernel   128x64 tile per CTA, 256 threads = (row, word).
//      (predicate -> bits by ballot, unless the fused pass already emitted
//      them), run union-find in shared memory, tile-border labels -> compact
//      seam rows / columns, global node init G[root] = root for
//      border-touching roots, and the tile's parent array (2-byte node ids,
//      roots at run starts) + border-root flags for pass 3.
//   2. ccl_seam_kernel   unions across tile seams in global memory (G is the
//      label array itself; only border-touching roots are ever nodes).
//   3. ccl_resolve_kernel  walks G once per border-touching root, then maps
//      each pixel to its run start (bit ops), the run to its root (the tile's
//      parent array) and the root to its label, with coalesced stores.
//
// HBM traffic per pixel from the fused pass's bit mask: 1/8 B bits in, 2 B
// local roots out and back, 4 B labels out (+ the sparse seam/root traffic),
// against the 4 B/px floor of writing the labels.

#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "sn_internal.h"

namespace sn {

constexpr int kLTW = 128;             // label tile columns
constexpr int kLTH = 64;              // label tile rows
constexpr int kLWords = kLTW / 32;    // words per tile row
constexpr int kLThreads = kLTH * kLWords;  // 256: one thread per (row, word)
constexpr int kZW = kLTW + 2, kZH = kLTH + 2;  // fp32 depth tile with a 1-pixel halo

__device__ __forceinline__ double depth_of(float d, double fxb) {
  // NaN marks an invalid depth sample
  double z = __longlong_as_double(0x7ff8000000000000ll);
  if (d > 0.0f && d <= FLT_MAX) {
    const double q = __ddiv_rn(fxb, (double)d);
    if (fabs(q) <= DBL_MAX) z = q;
  }
  return z;
}

__device__ __forceinline__ double edge_value(double c, double l, double r, double u, double dn) {
  return fabs(__dsub_rn(__dsub_rn(__dsub_rn(__dsub_rn(__dmul_rn(4.0, c), l), r), u), dn));
}

__device__ __forceinline__ bool valid_z(double z) { return z == z; }

// exact fp64 predicate at interior pixel (x, y) of frame f (row pitch W)
__device__ __noinline__ bool exact_passable(const float* __restrict__ f, int64_t W, int64_t x,
                                            int64_t y, double fxb, double t) {
  const double c = depth_of(f[y * W + x], fxb);
  const double l = depth_of(f[y * W + x - 1], fxb);
  const double r = depth_of(f[y * W + x + 1], fxb);
  const double u = depth_of(f[(y - 1) * W + x], fxb);
  const double dn = depth_of(f[(y + 1) * W + x], fxb);
  if (!(valid_z(c) && valid_z(l) && valid_z(r) && valid_z(u) && valid_z(dn))) return false;
  return edge_value(c, l, r, u, dn) <= t;
}

// ---------------------------------------------------------------------------
// standalone predicate (API sn_passable; exact fp64 per pixel, optional edges)

__global__ void passable_kernel(const float* __restrict__ disp, const CclParams p,
                                uint8_t* __restrict__ pas, double* __restrict__ edges) {
  const int64_t total = p.B * p.H * p.W;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = idx % p.W;
    const int64_t y = (idx / p.W) % p.H;
    const float* f = disp + (idx - y * p.W - x);
    bool ok = false;
    double e = __longlong_as_double(0x7ff8000000000000ll);
    if (x >= 1 && x + 1 < p.W && y >= 1 && y + 1 < p.H) {
      const double c = depth_of(f[y * p.W + x], p.fxb);
      const double l = depth_of(f[y * p.W + x - 1], p.fxb);
      const double r = depth_of(f[y * p.W + x + 1], p.fxb);
      const double u = depth_of(f[(y - 1) * p.W + x], p.fxb);
      const double dn = depth_of(f[(y + 1) * p.W + x], p.fxb);
      if (valid_z(c) && valid_z(l) && valid_z(r) && valid_z(u) && valid_z(dn)) {
        e = edge_value(c, l, r, u, dn);
        ok = true;
      }
    }
    if (pas) pas[idx] = (ok && e <= p.t) ? 1 : 0;
    if (edges) edges[idx] = e;
  }
}

// ---------------------------------------------------------------------------
// union-find helpers (indices only ever point to smaller indices)

// find with path halving: every write replaces a parent by an ancestor, so it
// commutes with concurrent unions (which only atomicMin roots)
__device__ __forceinline__ int uf_find(volatile int32_t* L, int x) {
  while (true) {
    const int p = L[x];
    if (p == x) return x;
    const int gp = L[p];
    if (gp == p) return p;
    L[x] = gp;
    x = gp;
  }
}

// read-only find
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

// start bit of the run (inside word A, starts st) that contains bit p
__device__ __forceinline__ int start_of(uint32_t st, int p) {
  const uint32_t upto = (p == 31) ? 0xffffffffu : ((2u << p) - 1u);
  return 31 - __clz(st & upto);
}

// ---------------------------------------------------------------------------
// tile union-find over word-runs
//
// Node id = local pixel index r * 128 + c of a run's first pixel; L (shared)
// holds parents at node ids only.  On return every node points at its root
// (the smallest node of its tile component) and `flag` has bit `root` set for
// every root whose component touches the tile border.

__device__ __forceinline__ void tile_union_find(int32_t* L, const uint32_t* bits, uint32_t* flag,
                                                int tid) {
  const int r = tid >> 2, w = tid & 3;
  const int base = r * kLTW + w * 32;
  const uint32_t A = bits[tid];
  const uint32_t st = run_starts(A);
  for (uint32_t m = st; m; m &= m - 1u) {
    const int n = base + __ffs(m) - 1;
    L[n] = n;
  }
  flag[tid] = 0u;
  __syncthreads();

  // a run crossing into this word from the left neighbour word
  if ((A & 1u) && w > 0) {
    const uint32_t Al = bits[tid - 1];
    if (Al >> 31) uf_unite(L, base, base - 32 + (31 - __clz(run_starts(Al))));
  }
  // runs of the row above (8-connected: the run dilated by one pixel).  All
  // rows at once: measured (tools/ccl_bench.cu) 2.3x faster than merging rows
  // in log-depth rounds -- finds average 1.3 steps here, so the tile is
  // latency-bound on its barriers, not on chain length.
  if (r > 0) {
    const uint32_t B = bits[tid - kLWords];
    const uint32_t BL = w > 0 ? bits[tid - kLWords - 1] : 0u;
    const uint32_t BR = w + 1 < kLWords ? bits[tid - kLWords + 1] : 0u;
    const uint32_t stB = run_starts(B);
    const int bbase = base - kLTW;
    for (uint32_t m = st; m; m &= m - 1u) {
      const int s = __ffs(m) - 1;
      const uint32_t hi = 0xffffffffu << s;
      const uint32_t zer = ~A & hi;  // zeros of A at or above s (bit s itself is set)
      const uint32_t run = zer ? ((zer & (0u - zer)) - 1u) & hi : hi;
      const int n = base + s;
      uint32_t o = (run | (run << 1) | (run >> 1)) & B;
      while (o) {
        const int p = __ffs(o) - 1;
        uf_unite(L, n, bbase + start_of(stB, p));
        const uint32_t upto = (p == 31) ? 0xffffffffu : ((2u << p) - 1u);
        const uint32_t zb = ~B & ~upto;  // zeros of B above p: end of that run
        if (!zb) break;
        o &= ~((zb & (0u - zb)) - 1u);
      }
      if ((run & 1u) && (BL >> 31)) uf_unite(L, n, bbase - 32 + (31 - __clz(run_starts(BL))));
      if ((run >> 31) && (BR & 1u)) uf_unite(L, n, bbase + 32);
    }
  }
  __syncthreads();
  // every node -> its root (only root values are written in this phase)
  for (uint32_t m = st; m; m &= m - 1u) {
    const int n = base + __ffs(m) - 1;
    L[n] = uf_root(L, n);
  }
  __syncthreads();
  // roots of components that touch the tile border
  auto mark = [&](int n) {
    const int root = L[n];
    atomicOr(&flag[root >> 5], 1u << (root & 31));
  };
  if (r == 0 || r == kLTH - 1)
    for (uint32_t m = st; m; m &= m - 1u) mark(base + __ffs(m) - 1);
  else {
    if (w == 0 && (A & 1u)) mark(base);
    if (w == kLWords - 1 && (A >> 31)) mark(base + (31 - __clz(st)));
  }
  __syncthreads();
}

constexpr int kTilePx = kLTW * kLTH;  // 8192: tile pixel index fits 13 bits

struct CclWorkspace {
  uint32_t* bits;  // [B][H][WW]
  uint16_t* roots;  // [tile][kTilePx] tile parent array (roots at run starts), tile-major
  uint32_t* flags;  // [tile][kTilePx / 32] border-touching roots
  int32_t* top;    // [B][n_ty][W]  first row of each tile row
  int32_t* bot;    // [B][n_ty][W]  last row of each tile row
  int32_t* left;   // [B][n_tx][H]  first column of each tile column
  int32_t* right;  // [B][n_tx][H]  last column of each tile column
  int WW, n_tx, n_ty;
};

__device__ __forceinline__ int frame_index(int node, int x0, int y0, int W) {
  return (y0 + (node >> 7)) * W + x0 + (node & (kLTW - 1));
}

// ---------------------------------------------------------------------------
// 1. tile pass.  MODE 0: predicate from fp32 disparity; MODE 1: uint8 passable

template <int MODE>
__global__ void __launch_bounds__(kLThreads)
    ccl_tile_kernel(const float* __restrict__ disp, const uint8_t* __restrict__ pas_in,
                    const CclParams p, const CclWorkspace ws, int32_t* __restrict__ labels) {
  __shared__ __align__(16) int32_t smem[kZH * kZW];  // fp32 depth tile, then the parent array
  __shared__ uint32_t bits[kLThreads];
  __shared__ uint32_t flag[kLThreads];
  static_assert(kZH * kZW >= kLTH * kLTW, "parent array must fit the depth tile");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int W = (int)p.W, H = (int)p.H;
  const int tx = blockIdx.x, ty = blockIdx.y;
  const int x0 = tx * kLTW, y0 = ty * kLTH;
  const int64_t fbase = (int64_t)blockIdx.z * p.H * p.W;

  if (MODE == 0) {
    const float* f = disp + fbase;
    float* zs = reinterpret_cast<float*>(smem);
    for (int i = tid; i < kZH * kZW; i += kLThreads) {
      const int iy = i / kZW, ix = i - iy * kZW;
      const int gx = x0 - 1 + ix, gy = y0 - 1 + iy;
      float z = __int_as_float(0x7fc00000);  // outside the frame: invalid sample
      if ((unsigned)gx < (unsigned)W && (unsigned)gy < (unsigned)H)
        z = p.exact_only ? __int_as_float(0x7f800000) : zfast(f[(int64_t)gy * W + gx], p.fxb_f);
      zs[i] = z;
    }
    __syncthreads();
    for (int rw = warp; rw < kLThreads; rw += kLThreads / 32) {
      const int r = rw >> 2, c = (rw & 3) * 32 + lane;
      const int gx = x0 + c, gy = y0 + r;
      bool pk = false;
      if (gx < W && gy < H) {
        const int zi = (r + 1) * kZW + c + 1;
        const int dec = (int)zpred(zs[zi], zs[zi - 1], zs[zi + 1], zs[zi - kZW], zs[zi + kZW],
                                   p.t_f);
        if (dec == 2) pk = exact_passable(f, W, gx, gy, p.fxb, p.t);
        else pk = dec == 1;
      }
      const uint32_t b = __ballot_sync(0xffffffffu, pk);
      if (lane == 0) bits[rw] = b;
    }
  } else if (MODE == 1) {
    for (int rw = warp; rw < kLThreads; rw += kLThreads / 32) {
      const int r = rw >> 2, c = (rw & 3) * 32 + lane;
      const int gx = x0 + c, gy = y0 + r;
      const bool pk = gx < W && gy < H && pas_in[fbase + (int64_t)gy * W + gx] != 0;
      const uint32_t b = __ballot_sync(0xffffffffu, pk);
      if (lane == 0) bits[rw] = b;
    }
  } else {
    // MODE 2: the bit mask is the input (emitted by the fused pass)
    const int r = tid >> 2, wc = tx * kLWords + (tid & 3);
    bits[tid] = (y0 + r < H && wc < ws.WW)
                    ? ws.bits[((int64_t)blockIdx.z * H + y0 + r) * ws.WW + wc]
                    : 0u;
  }
  __syncthreads();
  if (MODE != 2) {
    const int r = tid >> 2, wc = tx * kLWords + (tid & 3);
    if (y0 + r < H && wc < ws.WW)
      ws.bits[((int64_t)blockIdx.z * H + y0 + r) * ws.WW + wc] = bits[tid];
  }

  int32_t* L = smem;
  tile_union_find(L, bits, flag, tid);

  // seam rows / columns: frame index of each border pixel's root, -1 if not passable
  const int64_t seam_row = ((int64_t)blockIdx.z * ws.n_ty + ty) * W;
  const int64_t seam_col = ((int64_t)blockIdx.z * ws.n_tx + tx) * H;
  if (warp < 2) {
    const int r = warp == 0 ? 0 : kLTH - 1;
    int32_t* dst = (warp == 0 ? ws.top : ws.bot) + seam_row;
    if (y0 + r < H) {
#pragma unroll
      for (int w = 0; w < kLWords; ++w) {
        const uint32_t A = bits[r * kLWords + w];
        const int gx = x0 + w * 32 + lane;
        if (gx < W) {
          int32_t v = -1;
          if ((A >> lane) & 1u)
            v = frame_index(L[r * kLTW + w * 32 + start_of(run_starts(A), lane)], x0, y0, W);
          dst[gx] = v;
        }
      }
    }
  } else if (warp < 4) {
    // warp 2: first column, warp 3: last column; lanes <-> rows
    for (int r = lane; r < kLTH; r += 32) {
      if (y0 + r >= H) break;
      int32_t v = -1;
      if (warp == 2) {
        const uint32_t A = bits[r * kLWords];
        if (A & 1u) v = frame_index(L[r * kLTW], x0, y0, W);
        ws.left[seam_col + y0 + r] = v;
      } else {
        const uint32_t A = bits[r * kLWords + kLWords - 1];
        if (A >> 31)
          v = frame_index(L[r * kLTW + (kLWords - 1) * 32 + (31 - __clz(run_starts(A)))], x0, y0,
                          W);
        ws.right[seam_col + y0 + r] = v;
      }
    }
  }
  // global union-find nodes (border-touching roots only), border flags and
  // every pixel's local root for the resolve pass
  const int64_t tile = ((int64_t)blockIdx.z * ws.n_ty + ty) * ws.n_tx + tx;
  {
    const int r = tid >> 2, w = tid & 3;
    const int base = r * kLTW + w * 32;
    int32_t* G = labels + fbase;
    for (uint32_t m = run_starts(bits[tid]); m; m &= m - 1u) {
      const int n = base + __ffs(m) - 1;
      if (L[n] == n && ((flag[n >> 5] >> (n & 31)) & 1u)) {
        const int g = frame_index(n, x0, y0, W);
        G[g] = g;
      }
    }
    ws.flags[tile * (kTilePx / 32) + tid] = flag[tid];
  }
  // the tile's parent array (run-start entries = roots) as 2-byte node ids;
  // the resolve pass maps pixels to their run start itself
  uint2* dst = reinterpret_cast<uint2*>(ws.roots + tile * kTilePx);
  const int4* src = reinterpret_cast<const int4*>(L);
#pragma unroll
  for (int i = 0; i < kTilePx / 4 / kLThreads; ++i) {
    const int4 v = src[i * kLThreads + tid];
    dst[i * kLThreads + tid] = make_uint2(__byte_perm(v.x, v.y, 0x5410), __byte_perm(v.z, v.w, 0x5410));
  }
}

// ---------------------------------------------------------------------------
// 2. seams between tiles (global union-find on G = labels)
//
// Horizontal seams: pixel (x, y) in the last row of tile row ty against
// (x-1 .. x+1, y+1) in the first row of tile row ty+1 -- diagonals across tile
// columns included, so tile corners need no extra case.  Vertical seams:
// (x, y) in the last column of tile column tx against (x+1, y-1 .. y+1).
// A straight neighbour makes the diagonal links redundant (the diagonal
// pixels are 8-adjacent to it along the seam row/column).

__global__ void ccl_seam_kernel(const CclParams p, const CclWorkspace ws,
                                int32_t* __restrict__ labels) {
  const int W = (int)p.W, H = (int)p.H;
  const int64_t n_h = (int64_t)(ws.n_ty - 1) * W;  // horizontal seam positions per frame
  const int64_t n_v = (int64_t)(ws.n_tx - 1) * H;
  const int64_t per_frame = n_h + n_v;
  const int64_t total = per_frame * p.B;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = idx / per_frame;
    int64_t k = idx - f * per_frame;
    int32_t* G = labels + f * p.H * p.W;
    const int32_t* a_row;
    const int32_t* b_row;
    int i, n;
    if (k < n_h) {
      const int s = (int)(k / W);
      i = (int)(k - (int64_t)s * W);
      n = W;
      a_row = ws.bot + (f * ws.n_ty + s) * W;
      b_row = ws.top + (f * ws.n_ty + s + 1) * W;
    } else {
      k -= n_h;
      const int s = (int)(k / H);
      i = (int)(k - (int64_t)s * H);
      n = H;
      a_row = ws.right + (f * ws.n_tx + s) * H;
      b_row = ws.left + (f * ws.n_tx + s + 1) * H;
    }
    const int32_t a = a_row[i];
    if (a < 0) continue;
    const int32_t b = b_row[i];
    if (b >= 0) {
      if (a != b) uf_unite(G, a, b);
    } else {
      if (i > 0) {
        const int32_t bl = b_row[i - 1];
        if (bl >= 0 && bl != a) uf_unite(G, a, bl);
      }
      if (i + 1 < n) {
        const int32_t br = b_row[i + 1];
        if (br >= 0 && br != a) uf_unite(G, a, br);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// 3. resolve: border-touching roots through G (one walk per root), then one
// 2-byte read and one coalesced 4-byte label store per pixel

__global__ void __launch_bounds__(kLThreads)
    ccl_resolve_kernel(const CclParams p, const CclWorkspace ws, int32_t* __restrict__ labels) {
  __shared__ __align__(16) uint16_t Ls[kTilePx];  // tile parents (roots at run starts)
  __shared__ uint32_t bits[kLThreads];
  __shared__ uint32_t flag[kLThreads];
  __shared__ int32_t rank0[kLThreads];  // flagged roots before word i
  __shared__ int32_t fin[kLThreads * 2];  // final label per flagged root (<= border pixels)
  __shared__ int32_t warp_sum[kLThreads / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int W = (int)p.W, H = (int)p.H;
  const int tx = blockIdx.x, ty = blockIdx.y;
  const int x0 = tx * kLTW, y0 = ty * kLTH;
  const int64_t fbase = (int64_t)blockIdx.z * p.H * p.W;
  const int64_t tile = ((int64_t)blockIdx.z * ws.n_ty + ty) * ws.n_tx + tx;
  {
    const uint4* src = reinterpret_cast<const uint4*>(ws.roots + tile * kTilePx);
    uint4* dst = reinterpret_cast<uint4*>(Ls);
#pragma unroll
    for (int i = 0; i < kTilePx / 8 / kLThreads; ++i) dst[i * kLThreads + tid] = src[i * kLThreads + tid];
    const int r = tid >> 2, wc = tx * kLWords + (tid & 3);
    bits[tid] = (y0 + r < H && wc < ws.WW)
                    ? ws.bits[((int64_t)blockIdx.z * H + y0 + r) * ws.WW + wc]
                    : 0u;
  }
  const uint32_t fw = ws.flags[tile * (kTilePx / 32) + tid];
  flag[tid] = fw;
  // exclusive prefix of popcounts over the 256 flag words
  const int c = __popc(fw);
  int inc = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += v;
  }
  if (lane == 31) warp_sum[warp] = inc;
  __syncthreads();
  int off = 0;
  for (int i = 0; i < warp; ++i) off += warp_sum[i];
  const int excl = off + inc - c;
  rank0[tid] = excl;
  // walk G once per flagged root.  Nodes are only ever roots of tile
  // components, and a concurrent resolve of another tile overwrites such a
  // node with its final label -- an ancestor -- so the read-only walk is valid.
  {
    const volatile int32_t* G = labels + fbase;
    int k = excl;
    for (uint32_t m = fw; m; m &= m - 1u) {
      const int n = tid * 32 + __ffs(m) - 1;
      if (k < kLThreads * 2) fin[k] = uf_root(G, frame_index(n, x0, y0, W));
      ++k;
    }
  }
  __syncthreads();
  int32_t* out = labels + fbase;
  const bool full = x0 + kLTW <= W && y0 + kLTH <= H;
  for (int rw = warp; rw < kLThreads; rw += kLThreads / 32) {
    const int r = rw >> 2, w = rw & 3;
    const int gx = x0 + w * 32 + lane, gy = y0 + r;
    if (!full && (gx >= W || gy >= H)) continue;
    const uint32_t A = bits[rw];
    int32_t lab = -1;
    if ((A >> lane) & 1u) {
      const int v = Ls[r * kLTW + w * 32 + start_of(run_starts(A), lane)];
      const uint32_t fwv = flag[v >> 5];
      const uint32_t bit = 1u << (v & 31);
      lab = (fwv & bit) ? fin[rank0[v >> 5] + __popc(fwv & (bit - 1u))] : frame_index(v, x0, y0, W);
    }
    out[(int64_t)gy * W + gx] = lab;
  }
}

__global__ void add_offset_kernel(int32_t* __restrict__ labels, int64_t n, int64_t base) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = labels[idx];
    if (v >= 0) labels[idx] = (int32_t)(v + base);
  }
}

// relabel: scatter the (key -> root) map into a dense scratch indexed by
// key - base, then gather per pixel
__global__ void relabel_scatter_kernel(int32_t* __restrict__ scratch, int64_t n, int64_t base,
                                       const int32_t* __restrict__ keys,
                                       const int32_t* __restrict__ vals,
                                       const int32_t* __restrict__ n_map) {
  const int m = *n_map;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int64_t k = (int64_t)keys[i] - base;
    if (k >= 0 && k < n) scratch[k] = vals[i];
  }
}

__global__ void relabel_gather_kernel(int32_t* __restrict__ labels, int64_t n, int64_t base,
                                      const int32_t* __restrict__ scratch) {
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = labels[idx];
    if (v >= 0) {
      const int64_t k = (int64_t)v - base;
      if (k >= 0 && k < n) {
        const int32_t r = scratch[k];
        if (r >= 0) labels[idx] = r;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// launchers

static unsigned grid_for(const LaunchCtx& ctx, int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)ctx.num_sms * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

CclParams make_ccl_params(int64_t B, int64_t H, int64_t W, double fxb, double t) {
  CclParams p{};
  p.B = B;
  p.H = H;
  p.W = W;
  p.fxb = fxb;
  p.t = t;
  p.fxb_f = (float)fxb;
  p.t_f = (float)t;
  // the filter's error bound assumes normal fp32 operands (fxb_f, t_f, zf)
  p.exact_only = !(fxb >= 1e-20 && fxb <= 1e20 && t >= 1e-30 && t <= 1e30);
  return p;
}

static size_t align256(size_t v) { return (v + 255) / 256 * 256; }

size_t ccl_workspace_bytes(int64_t B, int64_t H, int64_t W) {
  const int64_t WW = (W + 31) / 32;
  const int64_t n_tx = (W + kLTW - 1) / kLTW, n_ty = (H + kLTH - 1) / kLTH;
  const int64_t tiles = B * n_tx * n_ty;
  return align256((size_t)(B * H * WW) * 4) + 2 * align256((size_t)(B * n_ty * W) * 4) +
         2 * align256((size_t)(B * n_tx * H) * 4) + align256((size_t)(tiles * kTilePx) * 2) +
         align256((size_t)(tiles * kTilePx / 32) * 4);
}

int run_passable(const LaunchCtx& ctx, const float* disp, const CclParams& p, uint8_t* pas,
                 double* edges) {
  const int64_t n = p.B * p.H * p.W;
  if (n == 0) return SN_OK;
  passable_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx.stream>>>(disp, p, pas, edges);
  return check_launch("passable_kernel");
}

// standalone passable bit mask (fallback for the fused emission): one warp
// per 32-pixel word, the same fp32 filter + fp64 fallback as the fused pass
__global__ void passable_bits_kernel(const float* __restrict__ disp, const FixedParams p,
                                     uint32_t* __restrict__ bits) {
  const int W = (int)p.W, H = (int)p.H;
  const int lane = threadIdx.x & 31;
  const int64_t n_words = p.B * p.H * p.bits_ww;
  for (int64_t wi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < n_words;
       wi += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t row = wi / p.bits_ww;
    const int x = (int)(wi - row * p.bits_ww) * 32 + lane;
    const int y = (int)(row % p.H);
    const float* f = disp + (row - y) * p.W;
    uint32_t pk = 0;
    if (x >= 1 && x + 1 < W && y >= 1 && y + 1 < H) {
      const float* c = f + (int64_t)y * W + x;
      pk = pred_bit(c[0], c[-1], c[1], c[-W], c[W], p);
    }
    const uint32_t b = __ballot_sync(0xffffffffu, pk != 0u);
    if (lane == 0) bits[wi] = b;
  }
}

int run_passable_bits(const LaunchCtx& ctx, const float* disp, const FixedParams& p,
                      uint32_t* bits) {
  const int64_t n = p.B * p.H * p.bits_ww * 32;
  if (n == 0) return SN_OK;
  passable_bits_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx.stream>>>(disp, p, bits);
  return check_launch("passable_bits_kernel");
}

int run_ccl(const LaunchCtx& ctx, const float* disp, const uint8_t* pas, const CclParams& p,
            int64_t index_base, int32_t* labels, void* workspace, size_t ws_bytes,
            const uint32_t* bits_in) {
  const int64_t n = p.B * p.H * p.W;
  if (n == 0) return SN_OK;
  if (p.H * p.W > 0x7fffffffLL || p.B > 65535)
    return set_error(SN_EINVAL, "frame too large for int32 labels");
  if (!workspace || ws_bytes < ccl_workspace_bytes(p.B, p.H, p.W))
    return set_error(SN_EINVAL, "labeller workspace too small (%zu < %zu bytes)", ws_bytes,
                     ccl_workspace_bytes(p.B, p.H, p.W));
  CclWorkspace ws;
  ws.WW = (int)((p.W + 31) / 32);
  ws.n_tx = (int)((p.W + kLTW - 1) / kLTW);
  ws.n_ty = (int)((p.H + kLTH - 1) / kLTH);
  uint8_t* q = static_cast<uint8_t*>(workspace);
  ws.bits = reinterpret_cast<uint32_t*>(q);
  q += align256((size_t)(p.B * p.H * ws.WW) * 4);
  ws.top = reinterpret_cast<int32_t*>(q);
  q += align256((size_t)(p.B * ws.n_ty * p.W) * 4);
  ws.bot = reinterpret_cast<int32_t*>(q);
  q += align256((size_t)(p.B * ws.n_ty * p.W) * 4);
  ws.left = reinterpret_cast<int32_t*>(q);
  q += align256((size_t)(p.B * ws.n_tx * p.H) * 4);
  ws.right = reinterpret_cast<int32_t*>(q);
  q += align256((size_t)(p.B * ws.n_tx * p.H) * 4);
  const int64_t tiles = p.B * ws.n_tx * ws.n_ty;
  ws.roots = reinterpret_cast<uint16_t*>(q);
  q += align256((size_t)(tiles * kTilePx) * 2);
  ws.flags = reinterpret_cast<uint32_t*>(q);

  if (bits_in) ws.bits = const_cast<uint32_t*>(bits_in);  // read-only in MODE 2
  dim3 grid((unsigned)ws.n_tx, (unsigned)ws.n_ty, (unsigned)p.B);
  if (bits_in)
    ccl_tile_kernel<2><<<grid, kLThreads, 0, ctx.stream>>>(nullptr, nullptr, p, ws, labels);
  else if (disp)
    ccl_tile_kernel<0><<<grid, kLThreads, 0, ctx.stream>>>(disp, nullptr, p, ws, labels);
  else
    ccl_tile_kernel<1><<<grid, kLThreads, 0, ctx.stream>>>(nullptr, pas, p, ws, labels);
  int rc = check_launch("ccl_tile_kernel");
  if (rc) return rc;
  const int64_t n_seam = ((int64_t)(ws.n_ty - 1) * p.W + (int64_t)(ws.n_tx - 1) * p.H) * p.B;
  if (n_seam > 0) {
    ccl_seam_kernel<<<grid_for(ctx, n_seam, 256), 256, 0, ctx.stream>>>(p, ws, labels);
    if ((rc = check_launch("ccl_seam_kernel"))) return rc;
  }
  ccl_resolve_kernel<<<grid, kLThreads, 0, ctx.stream>>>(p, ws, labels);
  if ((rc = check_launch("ccl_resolve_kernel"))) return rc;
  if (index_base != 0) {
    add_offset_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx.stream>>>(labels, n, index_base);
    rc = check_launch("add_offset_kernel");
  }
  return rc;
}

int run_relabel(const LaunchCtx& ctx, int32_t* labels, int64_t n, int64_t base,
                const int32_t* keys, const int32_t* vals, const int32_t* n_map, int32_t cap,
                int32_t* scratch) {
  if (n == 0) return SN_OK;
  if (cudaMemsetAsync(scratch, 0xff, (size_t)n * sizeof(int32_t), ctx.stream) != cudaSuccess)
    return set_cuda_error("cudaMemsetAsync(relabel scratch)");
  relabel_scatter_kernel<<<grid_for(ctx, cap, 256), 256, 0, ctx.stream>>>(scratch, n, base, keys,
                                                                          vals, n_map);
  int rc = check_launch("relabel_scatter_kernel");
  if (rc) return rc;
  relabel_gather_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx.stream>>>(labels, n, base, scratch);
  return check_launch("relabel_gather_kernel");
}

}  // namespace sn
