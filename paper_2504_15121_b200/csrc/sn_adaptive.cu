// Adaptive star-fill normals for sm_100a.
//
// Reference: adaptive.py:177-268 (estimate_normals_adaptive), the paper's
// edge-aware estimator.  Per pixel, rays in M directions (ray_offsets,
// adaptive.py:60-77 -- computed on the host with numpy so the rounding of
// rint(i cos), rint(i sin) is the reference's own) walk up to s steps and
// stop (excluding the triggering pixel)
//   ST  where the depth Laplacian is invalid or exceeds t -- exactly the
//       passable bit mask of passable_bits_kernel at threshold t;
//   CD  where the covered depth range (per ray, or shared by all rays of the
//       pixel with shared_range) exceeds t * z_c, or the depth is invalid.
// The support is the union of the visited offsets; the least-squares
// gradient uses the moment sums over it, then the closed-form normal of
// geometry.py:175-216.  Every decision and sum is evaluated in fp64 with the
// reference's operation order and no contraction (__d*_rn), and the moment
// sums run over the support in the reference's member order (first
// occurrence over rays and steps), so masks are bit-exact and normals differ
// from the reference only by the final fp32 rounding.
//
// Kernels: depth_kernel (z = fx*b/d in fp64, 8 B/px, read by CD walks and
// for z_c), then adaptive_kernel<stop> with one thread per pixel; the walks
// read the depth map or the bit mask through L1 (neighbouring threads share
// their supports).

#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "sn_internal.h"

namespace sn {

// depth map for the CD walks: RN32 of the reference's fp64 depth
// z = fx*b/d (pred_depth: NaN unless d is finite and > 0).  Rounding is
// monotonic, so running maxima / minima of these values are the roundings of
// the fp64 ones -- the fp32 filter below relies on that.
template <typename T>
__global__ void depth_kernel(const T* __restrict__ disp, int64_t n, double fxb,
                             float* __restrict__ z) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    z[i] = (float)pred_depth(disp[i], fxb);
}

// CD walk, exact: the reference's fp64 running range (adaptive.py:214-234)
// over depths recomputed from the disparities, for the lanes the fp32 filter
// cannot decide.  Sets this lane's bit in the warp's key masks.
template <typename T>
__device__ __noinline__ void cd_walk_exact(const T* __restrict__ fd, int x, int y, int W, int H,
                                           double zc, const AdaptiveParams& ap,
                                           const StarTable& tab, uint32_t* km, uint32_t bit) {
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  const double limit = __dmul_rn(ap.threshold, zc);
  double rmax = zc, rmin = zc;
  for (int j = 0; j < tab.n_rays; ++j) {
    if (!ap.shared_range) rmax = rmin = zc;
    for (int st = tab.ray_start[j]; st < tab.ray_start[j + 1]; ++st) {
      const int k = tab.step_key[st];
      const int sxy = tab.step_xy[st];
      const int xx = x + (int)(int16_t)(sxy & 0xffff), yy = y + (sxy >> 16);
      const bool inside = (unsigned)xx < (unsigned)W && (unsigned)yy < (unsigned)H;
      // fmax/fmin ignore a NaN sample; while the ray is alive the shared-range
      // update (adaptive.py:226-228) is the same as the per-ray one, and it
      // still happens on the step that stops it
      const double zs = inside ? pred_depth(fd[yy * W + xx], ap.fp.fxb) : qnan;
      const double nmax = fmax(rmax, zs), nmin = fmin(rmin, zs);
      const bool ok = (zs == zs) && __dsub_rn(nmax, nmin) <= limit;
      rmax = nmax;
      rmin = nmin;
      if (!ok) break;
      atomicOr(&km[k], bit);
    }
  }
}

constexpr int kAdaptiveThreads = 128;

__host__ __device__ inline size_t star_smem_tables(int n_steps, int n_keys) {
  return ((size_t)n_steps * 10 + (size_t)n_keys * 8 + 15) / 16 * 16;
}
static size_t star_smem(int n_steps, int n_keys) {
  return star_smem_tables(n_steps, n_keys) + (size_t)(kAdaptiveThreads / 32) * n_keys * 4;
}
constexpr uint32_t kFull = 0xffffffffu;

// One lane per pixel, a warp walks the rays in lockstep: the step (offset,
// key) is warp-uniform, lanes whose ray has stopped idle until the whole warp
// has stopped, and the support is recorded per key as a ballot of the lanes
// that visited it (warp-private shared-memory masks) -- no per-lane member
// bitmaps, no divergent table reads.
template <int STOP, typename T>  // STOP 0 = ST, 1 = CD; T = fp32 / fp64 disparities
__global__ void __launch_bounds__(kAdaptiveThreads)
    adaptive_kernel(const T* __restrict__ disp, const float* __restrict__ depth,
                    const uint32_t* __restrict__ pbits, const __grid_constant__ AdaptiveParams ap,
                    const __grid_constant__ StarTable tab, float* __restrict__ out6,
                    uint8_t* __restrict__ mask, unsigned* __restrict__ next_span) {
  // dynamic shared memory: the step / key tables (read warp-uniformly every
  // step: shared-memory broadcasts instead of constant-cache misses once
  // the tables outgrow it) and the warps' key masks
  extern __shared__ __align__(16) uint8_t adyn[];
  const int n_steps = tab.ray_start[tab.n_rays];
  int32_t* s_xy = reinterpret_cast<int32_t*>(adyn);
  int32_t* s_lin = s_xy + n_steps;
  int32_t* k_xy = s_lin + n_steps;
  int32_t* k_lin = k_xy + tab.n_keys;
  int16_t* s_key = reinterpret_cast<int16_t*>(k_lin + tab.n_keys);
  uint32_t* kmask = reinterpret_cast<uint32_t*>(adyn + star_smem_tables(n_steps, tab.n_keys));
  for (int i = threadIdx.x; i < n_steps; i += blockDim.x) {
    s_xy[i] = tab.step_xy[i];
    s_lin[i] = tab.step_lin[i];
    s_key[i] = tab.step_key[i];
  }
  for (int i = threadIdx.x; i < tab.n_keys; i += blockDim.x) {
    k_xy[i] = tab.key_xy[i];
    k_lin[i] = tab.key_lin[i];
  }
  __syncthreads();
  const FixedParams& p = ap.fp;
  const int W = (int)p.W, H = (int)p.H;
  const int64_t HW = p.H * p.W;
  const int64_t n = p.B * HW;
  const int lane = threadIdx.x & 31;
  uint32_t* km = kmask + (threadIdx.x >> 5) * tab.n_keys;
  const uint32_t lbit = 1u << lane;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  const float fnan = __int_as_float(0x7fc00000);
  // 32-pixel spans handed out dynamically (a span's walks vary a lot in
  // length): a warp's first span by its global warp index, the next ones
  // from a counter, the next value fetched while the current span runs
  const int64_t n_spans = (n + 31) / 32;
  const int64_t n_static = (int64_t)gridDim.x * blockDim.x / 32;
  unsigned nraw = lane == 0 ? atomicAdd(next_span, 1u) : 0u;
  for (int64_t span = ((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / 32; span < n_spans;
       span = n_static + __shfl_sync(0xffffffffu, nraw, 0),
               nraw = (lane == 0 && span < n_spans) ? atomicAdd(next_span, 1u) : nraw) {
    const int64_t wbase = span * 32;
    const int64_t idx = wbase + lane;
    const bool have = idx < n;
    const int64_t f = have ? idx / HW : 0;
    const int pix = have ? (int)(idx - f * HW) : 0;
    const int y = pix / W, x = pix - y * W;
    const T* fd = disp + f * HW;
    const double zc = have ? pred_depth(fd[pix], p.fxb) : qnan;
    const bool center_ok = zc == zc;
    for (int k = lane; k < tab.n_keys; k += 32) km[k] = 0u;
    __syncwarp();
    bool undecided = false;
    if (STOP == 0) {
      const uint32_t* fb = pbits + f * p.H * p.bits_ww;
      for (int j = 0; j < tab.n_rays; ++j) {
        bool alive = center_ok;
        for (int st = tab.ray_start[j]; st < tab.ray_start[j + 1]; ++st) {
          if (!__any_sync(kFull, alive)) break;
          const int k = s_key[st];
          const int sxy = s_xy[st];
          const int xx = x + (int)(int16_t)(sxy & 0xffff), yy = y + (sxy >> 16);
          alive = alive && (unsigned)xx < (unsigned)W && (unsigned)yy < (unsigned)H &&
                  ((fb[yy * p.bits_ww + (xx >> 5)] >> (xx & 31)) & 1u) != 0u;
          const uint32_t b = __ballot_sync(kFull, alive);
          if (lane == 0 && b) km[k] |= b;
        }
      }
    } else {
      // fp32 filter of the CD decisions.  With z32 = RN32(z) (u = 2^-24),
      // the running extremes are RN32 of the fp64 ones (rounding is
      // monotonic), so the fp32 range r is within 3.02 u M of max - min, and
      // the reference's RN64 subtraction and RN64(t z_c) add 2^-53 M and
      // u L.  A keep decision (r < l - m0) implies M <= (z_c + L)(1 + 4u),
      // so the per-pixel margin m0 = 2^-19 (z_c + 2 L) covers it with room to
      // spare; a stop decision (r > l + m0) is safe for any M (large M only
      // widens r - L).  Undecided steps, or depths outside [2^-100, 2^100],
      // send the lane to the exact fp64 walk.
      const double limit = __dmul_rn(ap.threshold, zc);
      const float lim32 = (float)limit, zc32 = (float)zc;
      undecided = center_ok && !(zc32 >= 7.888609052210118e-31f && zc32 <= 1.2676506002282294e30f &&
                                 lim32 >= 7.888609052210118e-31f && lim32 <= 1.2676506002282294e30f);
      const float m0 = (zc32 + 2.0f * lim32) * 1.9073486328125e-06f;  // 2^-19
      const float lo = lim32 - m0, hi = lim32 + m0;
      const float* fzp = depth + f * HW + pix;  // this lane's pixel
      // warps whose pixels all lie at least `reach` from the border skip the
      // per-step bounds test
      const bool interior = __all_sync(kFull, !have || (x >= tab.reach && x < W - tab.reach &&
                                                        y >= tab.reach && y < H - tab.reach));
      float rmax = zc32, rmin = zc32;
      for (int j = 0; j < tab.n_rays; ++j) {
        if (!ap.shared_range) rmax = rmin = zc32;
        bool alive = center_ok && !undecided;
        for (int st = tab.ray_start[j]; st < tab.ray_start[j + 1]; ++st) {
          if (!__any_sync(kFull, alive)) break;
          const int k = s_key[st];
          bool inside = true;
          if (!interior) {
            const int sxy = s_xy[st];
            const int xx = x + (int)(int16_t)(sxy & 0xffff), yy = y + (sxy >> 16);
            inside = (unsigned)xx < (unsigned)W && (unsigned)yy < (unsigned)H;
          }
          const float zs = (alive && inside) ? fzp[s_lin[st]] : fnan;
          // NaN / outside: stop with the extremes unchanged; otherwise the
          // extremes take the sample (also on the step that stops the ray)
          const bool fin = zs == zs;
          const bool inr = zs >= 7.888609052210118e-31f && zs <= 1.2676506002282294e30f;
          const float nmax = fmaxf(rmax, zs), nmin = fminf(rmin, zs);
          const float range = nmax - nmin;
          const bool keep = range < lo;
          if (alive && fin) {
            rmax = nmax;
            rmin = nmin;
            if (!inr || !(keep || range > hi)) undecided = true;
          }
          alive = alive && inr && keep;
          const uint32_t b = __ballot_sync(kFull, alive);
          if (lane == 0 && b) km[k] |= b;
        }
        if (__all_sync(kFull, !center_ok || undecided)) break;
      }
      __syncwarp();
      if (__any_sync(kFull, undecided)) {  // rare: exact walk for those lanes
        if (undecided) {
          for (int k = 0; k < tab.n_keys; ++k) atomicAnd(&km[k], ~lbit);
          cd_walk_exact(fd, x, y, W, H, zc, ap, tab, km, lbit);
        }
      }
    }
    __syncwarp();
    // moments over the support in member order (adaptive.py:240-255): keys
    // are numbered by first occurrence, so ascending key order IS member
    // order.  alpha, beta, gamma are integer sums (exact, as the reference's
    // fp64 sums are); v * (d_k - d_c) is exact for fp32 disparities, so one
    // FMA per term rounds like the reference's multiply-then-add; fp64
    // disparities round the product first (adaptive.py:251-252: b1 += vx * dd).
    // 32-bit sums unless the table's sums could overflow them (tab.wide)
    long long ia = 0, ib = 0, ig = 0;
    int ja = 0, jb = 0, jg = 0;
    double b1 = 0.0, b2 = 0.0;
    const double dc = (double)fd[pix];
    const T* fdp = fd + pix;
    for (int k = 0; k < tab.n_keys; ++k) {
      const uint32_t mk = km[k];
      if (mk == 0u) continue;  // warp-uniform
      if (mk & lbit) {
        const int kxy = k_xy[k];
        const int kx = (int)(int16_t)(kxy & 0xffff), ky = kxy >> 16;
        if (tab.wide) {
          ia += (long long)kx * kx;
          ib += (long long)kx * ky;
          ig += (long long)ky * ky;
        } else {
          ja += kx * kx;
          jb += kx * ky;
          jg += ky * ky;
        }
        const double dd = __dsub_rn((double)fdp[k_lin[k]], dc);
        if constexpr (sizeof(T) == 4) {
          b1 = __fma_rn((double)kx, dd, b1);
          b2 = __fma_rn((double)ky, dd, b2);
        } else {
          b1 = __dadd_rn(b1, __dmul_rn((double)kx, dd));
          b2 = __dadd_rn(b2, __dmul_rn((double)ky, dd));
        }
      }
    }
    if (!tab.wide) {
      ia = ja;
      ib = jb;
      ig = jg;
    }
    __syncwarp();  // the masks are cleared for the next pixels
    if (!have) continue;
    const double alpha = (double)ia, beta = (double)ib, gamma = (double)ig;
    const double det = __dsub_rn(__dmul_rn(alpha, gamma), __dmul_rn(beta, beta));
    bool ok = center_ok && det > 0.5;
    float n32[3] = {__int_as_float(0x7fc00000), __int_as_float(0x7fc00000),
                    __int_as_float(0x7fc00000)};
    if (ok) {
      const double g1 = __ddiv_rn(__dsub_rn(__dmul_rn(gamma, b1), __dmul_rn(beta, b2)), det);
      const double g2 = __ddiv_rn(__dadd_rn(__dmul_rn(-beta, b1), __dmul_rn(alpha, b2)), det);
      const double a1 = __dadd_rn(1.0, g1);  // adaptive.py:261 passes 1 + g1 ...
      // ... geometry.py:192-211, same order
      const double du = __dsub_rn((double)x, p.u0);
      const double dv = __dsub_rn((double)(y + p.row0), p.v0);
      const double wgt = dc > 0.0 ? __ddiv_rn(ap.baseline, dc) : qnan;
      const double g = __dsub_rn(1.0, a1);
      const double nx = __dmul_rn(__dmul_rn(g, wgt), ap.fxfx);
      const double ny = __dmul_rn(__dmul_rn(g2, wgt), ap.nfxfy);
      double nz = __dmul_rn(g2, dv);
      nz = __dsub_rn(nz, __dmul_rn(g, du));
      nz = __dmul_rn(nz, wgt);
      nz = __dsub_rn(nz, ap.baseline);
      nz = __dmul_rn(nz, p.fx);
      const double nrm = __dsqrt_rn(
          __dadd_rn(__dadd_rn(__dmul_rn(nx, nx), __dmul_rn(ny, ny)), __dmul_rn(nz, nz)));
      const double ux = __ddiv_rn(nx, nrm), uy = __ddiv_rn(ny, nrm), uz = __ddiv_rn(nz, nrm);
      ok = finite_d(ux) && finite_d(uy) && finite_d(uz);
      if (ok) {
        n32[0] = (float)ux;
        n32[1] = (float)uy;
        n32[2] = (float)uz;
      }
    }
    // point: the fused pass's formula (geometry.py:39-64; fp32, or fp64 for
    // fp64 disparities)
    float px, py, pz;
    if constexpr (sizeof(T) == 8) {
      point_from_disparity_f64(dc, (double)x - p.u0, (double)(y + p.row0) - p.v0, p, px, py, pz);
    } else {
      const float d32 = fd[pix];
      const float du_f = ((float)x - p.u0_hi) - p.u0_lo;
      const float dv_f = ((float)(y + p.row0) - p.v0_hi) - p.v0_lo;
      point_from_disparity(d32, du_f, dv_f, p.fxb_f, p.inv_fx_f, p.inv_fy_f, px, py, pz);
      if (d32 > 0.0f && d32 < 1.175494351e-38f) {  // subnormal: rcp.approx flushes
        pz = (float)(p.fxb / (double)d32);
        px = du_f * pz * p.inv_fx_f;
        py = pz * (dv_f * p.inv_fy_f);
      }
    }
    float2* o = reinterpret_cast<float2*>(out6 + idx * 6);
    o[0] = make_float2(px, py);
    o[1] = make_float2(pz, n32[0]);
    o[2] = make_float2(n32[1], n32[2]);
    if (mask) mask[idx] = ok ? 1 : 0;
  }
}

size_t adaptive_workspace_bytes(int64_t B, int64_t H, int64_t W) {
  const int64_t WW = (W + 31) / 32;
  return (size_t)(B * H * W) * 4 + 256 + (size_t)(B * H * WW) * 4;
}

template <typename T>
int run_adaptive(const LaunchCtx& ctx, const T* disp, const AdaptiveParams& ap,
                 const StarTable& tab, int stop, float* out6, uint8_t* mask, void* workspace,
                 size_t ws_bytes) {
  const FixedParams& p = ap.fp;
  const int64_t n = p.B * p.H * p.W;
  if (n == 0) return SN_OK;
  if (p.H * p.W > 0x7fffffffLL) return set_error(SN_EINVAL, "frame too large");
  if (!workspace || ws_bytes < adaptive_workspace_bytes(p.B, p.H, p.W))
    return set_error(SN_EINVAL, "adaptive workspace too small");
  float* depth = static_cast<float*>(workspace);
  uint32_t* bits = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(workspace) +
                                               ((size_t)n * 4 + 255) / 256 * 256);
  int rc = SN_OK;
  if (stop == 1) {
    int64_t g = (n + 255) / 256;
    if (g > (int64_t)ctx.num_sms * 32) g = (int64_t)ctx.num_sms * 32;
    depth_kernel<T><<<(unsigned)g, 256, 0, ctx.stream>>>(disp, n, p.fxb, depth);
    if ((rc = check_launch("depth_kernel"))) return rc;
  }
  AdaptiveParams a = ap;
  if (stop == 0) {
    FixedParams fp = p;
    fill_predicate(fp, p.fxb, ap.threshold, bits);
    if ((rc = run_passable_bits<T>(ctx, disp, fp, bits))) return rc;
    a.fp.bits = bits;
    a.fp.bits_ww = fp.bits_ww;
  }
  int64_t ga = (n + kAdaptiveThreads - 1) / kAdaptiveThreads;
  if (ga > (int64_t)ctx.num_sms * 64) ga = (int64_t)ctx.num_sms * 64;
  const size_t sm = star_smem(tab.ray_start[tab.n_rays], tab.n_keys);
  const int smax = (int)star_smem(kStarMaxSteps, kStarMaxKeys);
  if ((rc = ensure_dyn_smem(reinterpret_cast<const void*>(adaptive_kernel<0, T>), smax, ctx.device,
                            "adaptive_kernel<st>")) ||
      (rc = ensure_dyn_smem(reinterpret_cast<const void*>(adaptive_kernel<1, T>), smax, ctx.device,
                            "adaptive_kernel<cd>")))
    return rc;
  // the span counter: stream-ordered scratch (concurrent calls on other
  // streams get their own)
  unsigned* next_span = nullptr;
  if ((rc = scratch_alloc(ctx, sizeof(unsigned), reinterpret_cast<void**>(&next_span)))) return rc;
  if (cudaMemsetAsync(next_span, 0, sizeof(unsigned), ctx.stream) != cudaSuccess) {
    scratch_free(ctx, next_span);
    return set_cuda_error("cudaMemsetAsync(span counter)");
  }
  if (stop == 0)
    adaptive_kernel<0, T><<<(unsigned)ga, kAdaptiveThreads, sm, ctx.stream>>>(
        disp, depth, a.fp.bits, a, tab, out6, mask, next_span);
  else
    adaptive_kernel<1, T><<<(unsigned)ga, kAdaptiveThreads, sm, ctx.stream>>>(
        disp, depth, nullptr, a, tab, out6, mask, next_span);
  rc = check_launch("adaptive_kernel");
  scratch_free(ctx, next_span);
  return rc;
}
template int run_adaptive<float>(const LaunchCtx&, const float*, const AdaptiveParams&,
                                 const StarTable&, int, float*, uint8_t*, void*, size_t);
template int run_adaptive<double>(const LaunchCtx&, const double*, const AdaptiveParams&,
                                  const StarTable&, int, float*, uint8_t*, void*, size_t);

}  // namespace sn
