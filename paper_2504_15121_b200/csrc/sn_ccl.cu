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
//   1. ccl_local: 32x32 tile in shared memory -- each warp owns a tile row,
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

__device__ __forceinline__ int uf_find(const int32_t* L, int x) {
  int px = L[x];
  while (px != x) {
    x = px;
    px = L[x];
  }
  return x;
}

__device__ __forceinline__ int uf_find_vol(volatile int32_t* L, int x) {
  int px = L[x];
  while (px != x) {
    x = px;
    px = L[x];
  }
  return x;
}

__device__ __forceinline__ void uf_unite(int32_t* L, int a, int b) {
  while (true) {
    a = uf_find_vol(L, a);
    b = uf_find_vol(L, b);
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

__global__ void __launch_bounds__(kCclThreads)
    ccl_local_kernel(const float* __restrict__ disp, const uint8_t* __restrict__ pas_in,
                     const CclParams p, int32_t* __restrict__ labels) {
  __shared__ double zs[(kCT + 2) * (kCT + 2)];
  __shared__ int32_t L[kCT * kCT];
  __shared__ uint32_t rowbits[kCT];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t x0 = (int64_t)blockIdx.x * kCT, y0 = (int64_t)blockIdx.y * kCT;
  const int64_t fbase = (int64_t)blockIdx.z * p.H * p.W;
  if (disp) {
    const float* f = disp + fbase;
    for (int i = tid; i < (kCT + 2) * (kCT + 2); i += kCclThreads) {
      const int64_t gx = x0 - 1 + i % (kCT + 2), gy = y0 - 1 + i / (kCT + 2);
      double z = __longlong_as_double(0x7ff8000000000000ll);
      if (gx >= 0 && gx < p.W && gy >= 0 && gy < p.H) z = depth_of(f[gy * p.W + gx], p.fxb);
      zs[i] = z;
    }
    __syncthreads();
  }
  bool P[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int ly = warp + 8 * k, lx = lane;
    const int64_t gx = x0 + lx, gy = y0 + ly;
    bool pk = false;
    if (disp) {
      if (gx >= 1 && gx + 1 < p.W && gy >= 1 && gy + 1 < p.H) {
        const int zi = (ly + 1) * (kCT + 2) + lx + 1;
        const double c = zs[zi], l = zs[zi - 1], r = zs[zi + 1], u = zs[zi - (kCT + 2)],
                     dn = zs[zi + (kCT + 2)];
        if (valid_z(c) && valid_z(l) && valid_z(r) && valid_z(u) && valid_z(dn))
          pk = edge_value(c, l, r, u, dn) <= p.t;
      }
    } else if (gx < p.W && gy < p.H) {
      pk = pas_in[fbase + gy * p.W + gx] != 0;
    }
    P[k] = pk;
    const uint32_t b = __ballot_sync(0xffffffffu, pk);
    const uint32_t starts = b & ~(b << 1);
    const uint32_t upto = starts & (0xffffffffu >> (31 - lx));
    L[ly * kCT + lx] = pk ? ly * kCT + (31 - __clz(upto)) : -1;
    if (lane == 0) rowbits[ly] = b;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int ly = warp + 8 * k, lx = lane;
    if (!P[k] || ly == 0) continue;
    const uint32_t b = rowbits[ly], up = rowbits[ly - 1];
    const bool left = lx > 0 && ((b >> (lx - 1)) & 1u);
    const bool right = lx < 31 && ((b >> (lx + 1)) & 1u);
    const bool u = (up >> lx) & 1u;
    const bool ul = lx > 0 && ((up >> (lx - 1)) & 1u);
    const bool ur = lx < 31 && ((up >> (lx + 1)) & 1u);
    const int i = ly * kCT + lx;
    if (u) {
      if (!(left && ul)) uf_unite(L, i, i - kCT);
    } else {
      if (ul && !left) uf_unite(L, i, i - kCT - 1);
      if (ur && !right) uf_unite(L, i, i - kCT + 1);
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int ly = warp + 8 * k, lx = lane;
    const int64_t gx = x0 + lx, gy = y0 + ly;
    if (gx >= p.W || gy >= p.H) continue;
    int32_t out = -1;
    if (P[k]) {
      const int root = uf_find(L, ly * kCT + lx);
      out = (int32_t)((y0 + root / kCT) * p.W + x0 + root % kCT);
    }
    labels[fbase + gy * p.W + gx] = out;
  }
}

// ---------------------------------------------------------------------------
// 2. merge across tile edges

__global__ void ccl_merge_kernel(const CclParams p, int32_t* __restrict__ labels, int64_t n_col,
                                 int64_t n_row) {
  const int64_t per_frame = n_col + n_row;
  const int64_t total = per_frame * p.B;
  const int64_t tiles_x = (p.W + kCT - 1) / kCT;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = idx / per_frame;
    int64_t r = idx % per_frame;
    int32_t* L = labels + f * p.H * p.W;
    int64_t x, y;
    if (r < n_col) {
      // vertical tile edges: x = k*32, k >= 1; neighbours at x-1, rows y-1..y+1
      y = r % p.H;
      x = (r / p.H + 1) * kCT;
      const int64_t i = y * p.W + x;
      if (L[i] < 0) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int64_t yy = y + dy;
        if (yy < 0 || yy >= p.H) continue;
        const int64_t j = yy * p.W + x - 1;
        if (L[j] >= 0) uf_unite(L, (int)i, (int)j);
      }
    } else {
      r -= n_col;
      x = r % p.W;
      y = (r / p.W + 1) * kCT;
      const int64_t i = y * p.W + x;
      if (L[i] < 0) continue;
      for (int dx = -1; dx <= 1; ++dx) {
        const int64_t xx = x + dx;
        if (xx < 0 || xx >= p.W) continue;
        const int64_t j = (y - 1) * p.W + xx;
        if (L[j] >= 0) uf_unite(L, (int)i, (int)j);
      }
    }
    (void)tiles_x;
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
    if (v >= 0 && v != i) L[i] = uf_find(L, v);
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
  dim3 grid((unsigned)((p.W + kCT - 1) / kCT), (unsigned)((p.H + kCT - 1) / kCT), (unsigned)p.B);
  ccl_local_kernel<<<grid, kCclThreads, 0, ctx.stream>>>(disp, pas, p, labels);
  int rc = check_launch("ccl_local_kernel");
  if (rc) return rc;
  const int64_t n_col = ((p.W - 1) / kCT) * p.H;
  const int64_t n_row = ((p.H - 1) / kCT) * p.W;
  if (n_col + n_row > 0) {
    ccl_merge_kernel<<<grid_for(ctx, (n_col + n_row) * p.B, 256), 256, 0, ctx.stream>>>(
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
