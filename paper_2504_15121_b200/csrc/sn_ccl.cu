// Passable-set predicate and connected-component labelling for sm_100a.
//
// Predicate (bit-exact with the reference): depth
// z = (fx*b)/d valid iff d finite, d > 0 and z finite (geometry.py:39-45,
// 169-172); edge e = |((((4c - left) - right) - up) - down)| evaluated in
// numpy's left-to-right order with correctly rounded fp64 operations
// (adaptive.py:80-97), valid only at interior pixels with all five depths
// valid; passable = edge valid and e <= t (the ST ray test,
// adaptive.py:130-132, 218-221).
//
// Labelling (no reference function): 8-connected
// components of the passable set, canonical label = smallest raster index in
// the component.  Union-find where every link goes from the larger index to
// the smaller (atomicMin), so a tree's root is always its minimum element and
// the result is independent of scheduling:
//   1. ccl_local: 32x64 tile in shared memory -- each warp owns a tile row,
//      __ballot_sync gives the passable bits of the row and every pixel links
//      to the first pixel of its horizontal run (no atomics), then rows are
//      merged with the pixels above (3 candidates, redundant unions pruned);
//      tile roots are written as frame raster indices.
//   2. ccl_merge: unions across tile edges in global memory.
//   3. ccl_flatten: global path compression, label = root index.

#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "sn_internal.h"

namespace sn {

constexpr int kCT = 32;  // CCL tile edge
constexpr int kCclThreads = 256;

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

// ---------------------------------------------------------------------------
// standalone predicate (API sn_passable; the CCL kernel evaluates it inline)

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

// read-only find: used where concurrent writers store final roots (flatten),
// so a late path-halving store can never overwrite a root with an ancestor
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

// ---------------------------------------------------------------------------
// 1. tile-local labelling (+ fused predicate when disp != nullptr)
//
// Tile = 32 columns x 64 rows; warp w owns rows w, w+8, ..., lane = column.

constexpr int kTY = 64;                 // CCL tile rows (kCT = 32 columns)
constexpr int kZW = kCT + 2, kZH = kTY + 2;
constexpr int kRowsPerWarp = kTY / (kCclThreads / 32);

__global__ void __launch_bounds__(kCclThreads)
    ccl_local_kernel(const float* __restrict__ disp, const uint8_t* __restrict__ pas_in,
                     const CclParams p, int32_t* __restrict__ labels) {
  __shared__ double zs[kZH * kZW];
  __shared__ int32_t L[kTY * kCT];
  __shared__ uint32_t rowbits[kTY];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int W = (int)p.W, H = (int)p.H;
  const int x0 = blockIdx.x * kCT, y0 = blockIdx.y * kTY;
  const int64_t fbase = (int64_t)blockIdx.z * p.H * p.W;
  if (disp) {
    const float* f = disp + fbase;
    for (int i = tid; i < kZH * kZW; i += kCclThreads) {
      const int iy = i / kZW, ix = i - iy * kZW;
      const int gx = x0 - 1 + ix, gy = y0 - 1 + iy;
      double z = __longlong_as_double(0x7ff8000000000000ll);
      if ((unsigned)gx < (unsigned)W && (unsigned)gy < (unsigned)H)
        z = depth_of(f[(int64_t)gy * W + gx], p.fxb);
      zs[i] = z;
    }
    __syncthreads();
  }
  uint32_t Pbits = 0;  // bit k: pixel (warp + 8k, lane) passable
#pragma unroll
  for (int k = 0; k < kRowsPerWarp; ++k) {
    const int ly = warp + 8 * k;
    const int gx = x0 + lane, gy = y0 + ly;
    bool pk = false;
    if (disp) {
      if (gx >= 1 && gx + 1 < W && gy >= 1 && gy + 1 < H) {
        const int zi = (ly + 1) * kZW + lane + 1;
        const double c = zs[zi], l = zs[zi - 1], r = zs[zi + 1], u = zs[zi - kZW],
                     dn = zs[zi + kZW];
        if (valid_z(c) && valid_z(l) && valid_z(r) && valid_z(u) && valid_z(dn))
          pk = edge_value(c, l, r, u, dn) <= p.t;
      }
    } else if (gx < W && gy < H) {
      pk = pas_in[fbase + (int64_t)gy * W + gx] != 0;
    }
    Pbits |= (pk ? 1u : 0u) << k;
    const uint32_t b = __ballot_sync(0xffffffffu, pk);
    const uint32_t starts = b & ~(b << 1);
    const uint32_t upto = starts & (0xffffffffu >> (31 - lane));
    L[ly * kCT + lane] = pk ? ly * kCT + (31 - __clz(upto)) : -1;
    if (lane == 0) rowbits[ly] = b;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kRowsPerWarp; ++k) {
    const int ly = warp + 8 * k;
    if (!((Pbits >> k) & 1u) || ly == 0) continue;
    const uint32_t b = rowbits[ly], up = rowbits[ly - 1];
    const bool left = lane > 0 && ((b >> (lane - 1)) & 1u);
    const bool right = lane < 31 && ((b >> (lane + 1)) & 1u);
    const bool u = (up >> lane) & 1u;
    const bool ul = lane > 0 && ((up >> (lane - 1)) & 1u);
    const bool ur = lane < 31 && ((up >> (lane + 1)) & 1u);
    const int i = ly * kCT + lane;
    // a run shares its connections: only the pixels whose upper neighbours are
    // not already reached through the horizontal neighbour do the union
    if (u) {
      if (!(left && ul)) uf_unite(L, i, i - kCT);
    } else {
      if (ul && !left) uf_unite(L, i, i - kCT - 1);
      if (ur && !right) uf_unite(L, i, i - kCT + 1);
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kRowsPerWarp; ++k) {
    const int ly = warp + 8 * k;
    const int gx = x0 + lane, gy = y0 + ly;
    if (gx >= W || gy >= H) continue;
    int32_t out = -1;
    if ((Pbits >> k) & 1u) {
      const int root = uf_find(L, ly * kCT + lane);
      out = (y0 + (root >> 5)) * W + x0 + (root & 31);
    }
    labels[fbase + (int64_t)gy * W + gx] = out;
  }
}

// ---------------------------------------------------------------------------
// 2. merge across tile edges (global union-find on the label array)
//
// One thread per pixel on the first column / first row of a tile (except the
// image's own first column / row).  Same pruning as the in-tile rule: the
// pixel unites with its straight neighbour across the edge if passable, else
// with the diagonal ones not already reached through its along-edge neighbour.

__global__ void ccl_merge_kernel(const CclParams p, int32_t* __restrict__ labels, int n_col,
                                 int n_row) {
  const int W = (int)p.W, H = (int)p.H;
  const int per_frame = n_col + n_row;
  const int64_t total = (int64_t)per_frame * p.B;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(idx / per_frame);
    int r = (int)(idx - (int64_t)f * per_frame);
    int32_t* L = labels + (int64_t)f * p.H * p.W;
    volatile int32_t* V = L;
    if (r < n_col) {
      // vertical tile edge at x = (r / H + 1) * 32; across-edge neighbours at x - 1
      const int y = r % H;
      const int x = (r / H + 1) * kCT;
      const int i = y * W + x;
      if (V[i] < 0) continue;
      // pruning may only lean on an along-edge neighbour of the SAME tile
      // (already connected by ccl_local); across a tile corner both links stay
      const bool up_same = (y % kTY) != 0, down_same = ((y + 1) % kTY) != 0;
      if (V[i - 1] >= 0) {
        if (!(up_same && V[i - W] >= 0 && V[i - W - 1] >= 0)) uf_unite(L, i, i - 1);
      } else {
        if (y > 0 && V[i - W - 1] >= 0 && !(up_same && V[i - W] >= 0)) uf_unite(L, i, i - W - 1);
        if (y + 1 < H && V[i + W - 1] >= 0 && !(down_same && V[i + W] >= 0))
          uf_unite(L, i, i + W - 1);
      }
    } else {
      // horizontal tile edge at y = (r / W + 1) * kTY; neighbours in row y - 1
      r -= n_col;
      const int x = r % W;
      const int y = (r / W + 1) * kTY;
      const int i = y * W + x;
      if (V[i] < 0) continue;
      const bool left_same = (x % kCT) != 0, right_same = ((x + 1) % kCT) != 0;
      const bool left = x > 0 && V[i - 1] >= 0;
      const bool right = x + 1 < W && V[i + 1] >= 0;
      if (V[i - W] >= 0) {
        if (!(left_same && left && V[i - W - 1] >= 0)) uf_unite(L, i, i - W);
      } else {
        if (x > 0 && V[i - W - 1] >= 0 && !(left_same && left)) uf_unite(L, i, i - W - 1);
        if (x + 1 < W && V[i - W + 1] >= 0 && !(right_same && right)) uf_unite(L, i, i - W + 1);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// 3. flatten (+ optional raster-index offset for strips, second pass)

__global__ void ccl_flatten_kernel(const CclParams p, int32_t* __restrict__ labels) {
  const int64_t total = p.B * p.H * p.W;
  const int64_t HW = p.H * p.W;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int32_t* L = labels + (idx / HW) * HW;
    const int i = (int)(idx % HW);
    const int v = L[i];
    if (v >= 0 && v != i) L[i] = uf_root(L, v);
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

int run_passable(const LaunchCtx& ctx, const float* disp, const CclParams& p, uint8_t* pas,
                 double* edges) {
  const int64_t n = p.B * p.H * p.W;
  if (n == 0) return SN_OK;
  passable_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx.stream>>>(disp, p, pas, edges);
  return check_launch("passable_kernel");
}

int run_ccl(const LaunchCtx& ctx, const float* disp, const uint8_t* pas, const CclParams& p,
            int64_t index_base, int32_t* labels) {
  const int64_t n = p.B * p.H * p.W;
  if (n == 0) return SN_OK;
  if (p.H * p.W > 0x7fffffffLL || p.B > 65535) return set_error(SN_EINVAL, "frame too large for int32 labels");
  dim3 grid((unsigned)((p.W + kCT - 1) / kCT), (unsigned)((p.H + kTY - 1) / kTY), (unsigned)p.B);
  ccl_local_kernel<<<grid, kCclThreads, 0, ctx.stream>>>(disp, pas, p, labels);
  int rc = check_launch("ccl_local_kernel");
  if (rc) return rc;
  const int n_col = (int)(((p.W - 1) / kCT) * p.H);
  const int n_row = (int)(((p.H - 1) / kTY) * p.W);
  if (n_col + n_row > 0) {
    ccl_merge_kernel<<<grid_for(ctx, (int64_t)(n_col + n_row) * p.B, 256), 256, 0, ctx.stream>>>(
        p, labels, n_col, n_row);
    rc = check_launch("ccl_merge_kernel");
    if (rc) return rc;
    ccl_flatten_kernel<<<grid_for(ctx, n, 256), 256, 0, ctx.stream>>>(p, labels);
    rc = check_launch("ccl_flatten_kernel");
    if (rc) return rc;
  }
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
