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

__global__ void depth_kernel(const float* __restrict__ disp, int64_t n, double fxb,
                             double* __restrict__ z) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    z[i] = pred_depth(disp[i], fxb);
}

template <int STOP>  // 0 = ST, 1 = CD
__global__ void __launch_bounds__(128)
    adaptive_kernel(const float* __restrict__ disp, const double* __restrict__ depth,
                    const uint32_t* __restrict__ pbits, const AdaptiveParams ap,
                    const __grid_constant__ StarTable tab, float* __restrict__ out6,
                    uint8_t* __restrict__ mask) {
  const FixedParams& p = ap.fp;
  const int W = (int)p.W, H = (int)p.H;
  const int64_t HW = p.H * p.W;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < p.B * HW;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = idx / HW;
    const int pix = (int)(idx - f * HW);
    const int y = pix / W, x = pix - y * W;
    const float* fd = disp + f * HW;
    const double* fz = depth + f * HW;
    const double zc = fz[pix];
    const bool center_ok = zc == zc;
    uint32_t mem[kStarKeyWords];
#pragma unroll
    for (int i = 0; i < kStarKeyWords; ++i) mem[i] = 0u;
    if (center_ok) {
      const double limit = __dmul_rn(ap.threshold, zc);
      double rmax = zc, rmin = zc;
      for (int j = 0; j < tab.n_rays; ++j) {
        if (STOP == 1 && !ap.shared_range) rmax = rmin = zc;
        for (int st = tab.ray_start[j]; st < tab.ray_start[j + 1]; ++st) {
          const int k = tab.step_key[st];
          const int xx = x + tab.key_x[k], yy = y + tab.key_y[k];
          const bool inside = (unsigned)xx < (unsigned)W && (unsigned)yy < (unsigned)H;
          bool ok;
          if (STOP == 0) {
            ok = inside &&
                 ((pbits[(f * p.H + yy) * p.bits_ww + (xx >> 5)] >> (xx & 31)) & 1u) != 0u;
          } else {
            // fmax/fmin ignore a NaN sample; while the ray is alive the
            // shared-range update (adaptive.py:226-228) is the same as the
            // per-ray one, and it still happens on the step that stops it
            const double zs = inside ? fz[yy * W + xx] : qnan;
            const double nmax = fmax(rmax, zs), nmin = fmin(rmin, zs);
            ok = (zs == zs) && __dsub_rn(nmax, nmin) <= limit;
            rmax = nmax;
            rmin = nmin;
          }
          if (!ok) break;  // alive stays false for the rest of the ray
          mem[k >> 5] |= 1u << (k & 31);
        }
      }
    }
    // moments over the support in member order (adaptive.py:240-255)
    double alpha = 0.0, beta = 0.0, gamma = 0.0, b1 = 0.0, b2 = 0.0;
    const double dc = (double)fd[pix];
    if (center_ok) {
      for (int w = 0; w < kStarKeyWords; ++w) {
        for (uint32_t m = mem[w]; m; m &= m - 1u) {
          const int k = w * 32 + __ffs(m) - 1;
          const double vx = (double)tab.key_x[k], vy = (double)tab.key_y[k];
          alpha = __dadd_rn(alpha, __dmul_rn(vx, vx));
          beta = __dadd_rn(beta, __dmul_rn(vx, vy));
          gamma = __dadd_rn(gamma, __dmul_rn(vy, vy));
          const double dd = __dsub_rn((double)fd[(y + tab.key_y[k]) * W + x + tab.key_x[k]], dc);
          b1 = __dadd_rn(b1, __dmul_rn(vx, dd));
          b2 = __dadd_rn(b2, __dmul_rn(vy, dd));
        }
      }
    }
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
    // point: the fused pass's formula (geometry.py:39-64, fp32)
    float px, py, pz;
    {
      const float d32 = fd[pix];
      const float du_f = ((float)x - p.u0_hi) - p.u0_lo;
      const float dv_f = ((float)(y + p.row0) - p.v0_hi) - p.v0_lo;
      point_from_disparity(d32, du_f, dv_f, p.fxb_f, p.inv_fx_f, p.inv_fy_f, px, py, pz);
      if (d32 > 0.0f && d32 < 1.175494351e-38f) {  // subnormal: rcp.approx flushes
        pz = (float)(p.fxb / (double)d32);
        px = du_f * pz * p.inv_fx_f;
        py = dv_f * pz * p.inv_fy_f;
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
  return (size_t)(B * H * W) * 8 + 256 + (size_t)(B * H * WW) * 4;
}

int run_adaptive(const LaunchCtx& ctx, const float* disp, const AdaptiveParams& ap,
                 const StarTable& tab, int stop, float* out6, uint8_t* mask, void* workspace,
                 size_t ws_bytes) {
  const FixedParams& p = ap.fp;
  const int64_t n = p.B * p.H * p.W;
  if (n == 0) return SN_OK;
  if (p.H * p.W > 0x7fffffffLL) return set_error(SN_EINVAL, "frame too large");
  if (!workspace || ws_bytes < adaptive_workspace_bytes(p.B, p.H, p.W))
    return set_error(SN_EINVAL, "adaptive workspace too small");
  double* depth = static_cast<double*>(workspace);
  uint32_t* bits = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(workspace) +
                                               ((size_t)n * 8 + 255) / 256 * 256);
  int64_t g = (n + 255) / 256;
  if (g > (int64_t)ctx.num_sms * 32) g = (int64_t)ctx.num_sms * 32;
  depth_kernel<<<(unsigned)g, 256, 0, ctx.stream>>>(disp, n, p.fxb, depth);
  int rc = check_launch("depth_kernel");
  if (rc) return rc;
  AdaptiveParams a = ap;
  if (stop == 0) {
    FixedParams fp = p;
    fill_predicate(fp, p.fxb, ap.threshold, bits);
    if ((rc = run_passable_bits(ctx, disp, fp, bits))) return rc;
    a.fp.bits = bits;
    a.fp.bits_ww = fp.bits_ww;
  }
  int64_t ga = (n + 127) / 128;
  if (ga > (int64_t)ctx.num_sms * 64) ga = (int64_t)ctx.num_sms * 64;
  if (stop == 0)
    adaptive_kernel<0><<<(unsigned)ga, 128, 0, ctx.stream>>>(disp, depth, a.fp.bits, a, tab, out6,
                                                             mask);
  else
    adaptive_kernel<1><<<(unsigned)ga, 128, 0, ctx.stream>>>(disp, depth, nullptr, a, tab, out6,
                                                             mask);
  return check_launch("adaptive_kernel");
}

}  // namespace sn
