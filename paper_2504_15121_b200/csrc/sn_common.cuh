// Shared device helpers for the sm_100a kernels: TMA / mbarrier / bulk-copy
// PTX wrappers and the closed-form normal epilogue.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#ifdef SN_CHECK
#include <cstdio>
#endif

#include "sn_b200.h"

namespace sn {

// ---------------------------------------------------------------------------
// kernel parameters shared by the fixed-pass kernels

// Bounds checks of the checked build (make check: -DSN_CHECK): a failed check
// prints its site and traps, which fails the calling test.  No code at all in
// the product build.
#ifdef SN_CHECK
#define SN_ASSERT(cond)                                                              \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      printf("SN_ASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
             #cond, (int)blockIdx.x, (int)threadIdx.x);                              \
      __trap();                                                                      \
    }                                                                                \
  } while (0)
#else
#define SN_ASSERT(cond) \
  do {                  \
  } while (0)
#endif

struct FixedParams {
  int64_t B, H, W;
  // rig, pre-combined on the host in Python's double order
  double fx, fy, u0, v0;
  double fxb;      // fx * b (Python double product, geometry.py:43)
  float fxb_f;     // fp32(fx * b)       point path
  float inv_fx_f;  // fp32(1 / fx)
  float nfx_f, nfy_f, nal_f;  // -fp32(fx), -fp32(fy), -fp32(alpha): the fp32 normal's factors
  float inv_fy_f;  // fp32(1 / fy)
  float u0_hi, u0_lo, v0_hi, v0_lo;  // two-float split of u0, v0
  // integer moments of the offset pattern (exact in double)
  double alpha, beta, gamma, det, sx, sy;
  int R;     // square radius (fast path)
  int row0;  // image row of the block's first row (strips of a larger frame)
  // optional ST-passable bit mask emitted by the fused pass ([B][H][bits_ww]
  // uint32, bit u%32 of word u/32 = pixel u of the row); NULL = not wanted
  uint32_t* bits;
  int bits_ww;
  int pred_exact;  // every predicate decision on the fp64 path (filter out of range)
  double t;        // ST threshold
  float t_f, fxb_pf;  // fp32 threshold / fx*b for the predicate filter
  // 16-bit PNG disparity input (formats.py:133-150): d = (raw - 1) / scale,
  // raw == invalid -> NaN
  double png_scale, png_rcp;  // png_rcp = RN(1 / scale), 0 = divide
  float png_rcp_f;            // (float)RN(1 / scale)
  int png_invalid, png_sign;  // png_sign = sign(scale)
};

// (raw - 1) / scale correctly rounded (the reference's fp64 division,
// formats.py:148).  With rcp = RN(1/scale): q = RN(a rcp) is within 1 ulp of
// a/scale, r = a - q scale is exact (fma), and q + r rcp rounds to RN(a/scale)
// (Markstein's theorem) as long as nothing over/underflows -- guaranteed for
// |a| <= 65535 and 2^-100 <= |scale| <= 2^100 (the host passes rcp = 0
// outside that range: plain division).  4 fp64 ops instead of a DDIV sequence.
__device__ __forceinline__ double png16_value(uint32_t raw, int invalid, double scale,
                                              double rcp) {
  if ((int)raw == invalid) return __longlong_as_double(0x7ff8000000000000ll);
  const double a = (double)raw - 1.0;
  if (rcp == 0.0) return __ddiv_rn(a, scale);
  const double q = __dmul_rn(a, rcp);
  const double r = __fma_rn(-q, scale, a);
  return __fma_rn(r, rcp, q);
}

// a 16-bit quantised disparity sample (the fused pass's third input type)
struct Png16 {
  uint16_t raw;
};

__device__ __forceinline__ float rcp_ftz(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// ---------------------------------------------------------------------------
// ST-passable predicate (adaptive.py:80-97,130-132) from raw disparities
//
// exact: z_i = fl64(fxb / d_i) (geometry.py:39-45), e = |((((4 z_c - z_l) -
// z_r) - z_u) - z_d)| with correctly rounded fp64 operations in numpy's
// order, passable iff all five d finite and > 0 and e <= t.

__device__ __forceinline__ double pred_depth(float d, double fxb) {
  double z = __longlong_as_double(0x7ff8000000000000ll);
  if (d > 0.0f && d <= 3.402823466e38f) {
    const double q = __ddiv_rn(fxb, (double)d);
    if (fabs(q) <= 1.7976931348623157e308) z = q;
  }
  return z;
}

static __device__ __noinline__ uint32_t pred_exact_d(float a, float b, float c, float e, float f,
                                             double fxb, double t) {
  // invalid neighbourhoods (a sample not finite and > 0) first, without dividing
  const uint32_t lim = 0x7f7fffffu;
  if (!(((__float_as_uint(a) - 1u) < lim) & ((__float_as_uint(b) - 1u) < lim) &
        ((__float_as_uint(c) - 1u) < lim) & ((__float_as_uint(e) - 1u) < lim) &
        ((__float_as_uint(f) - 1u) < lim)))
    return 0u;
  const double zc = pred_depth(a, fxb), zl = pred_depth(b, fxb), zr = pred_depth(c, fxb),
               zu = pred_depth(e, fxb), zd = pred_depth(f, fxb);
  if (!(zc == zc && zl == zl && zr == zr && zu == zu && zd == zd)) return 0u;
  const double ev =
      fabs(__dsub_rn(__dsub_rn(__dsub_rn(__dsub_rn(__dmul_rn(4.0, zc), zl), zr), zu), zd));
  return ev <= t ? 1u : 0u;
}

// fp64 disparities (the reference's own ScalarField values, fields.py:37-40):
// the same predicate on the unrounded samples
__device__ __forceinline__ double pred_depth(double d, double fxb) {
  double z = __longlong_as_double(0x7ff8000000000000ll);
  if (d > 0.0 && d <= 1.7976931348623157e308) {
    const double q = __ddiv_rn(fxb, d);
    if (fabs(q) <= 1.7976931348623157e308) z = q;
  }
  return z;
}

static __device__ __noinline__ uint32_t pred_exact_d(double a, double b, double c, double e,
                                                     double f, double fxb, double t) {
  const double zc = pred_depth(a, fxb), zl = pred_depth(b, fxb), zr = pred_depth(c, fxb),
               zu = pred_depth(e, fxb), zd = pred_depth(f, fxb);
  if (!(zc == zc && zl == zl && zr == zr && zu == zu && zd == zd)) return 0u;
  const double ev =
      fabs(__dsub_rn(__dsub_rn(__dsub_rn(__dsub_rn(__dmul_rn(4.0, zc), zl), zr), zu), zd));
  return ev <= t ? 1u : 0u;
}

// fp32 view of a disparity sample for the predicate filters.  For fp64
// samples the extra rounding adds 2^-24 to the depth's relative error (the
// filter bound below grows from 2^-21 S to 0.5625 * 2^-20 S, still inside its
// 2^-20 S margin); samples outside fp32's normal range become 0 or inf and
// force the exact path.
__device__ __forceinline__ float disp_f32(float d) { return d; }
__device__ __forceinline__ float disp_f32(double d) { return __double2float_rn(d); }

// fp32 filter on depths (passable_bits_kernel).  zf = fl(fxb_f * rcp.approx(d))
// has relative error <= 2^-24 (fxb_f) + 2^-23 (rcp.approx, 1 ulp) + 2^-24
// (product) = 2^-22 while zf stays a normal float.  With S = 4c + l + r + u + dn
// (all depths > 0) the fp32 edge value is within 2^-22 S (inputs) + 4 * 2^-24 S
// (four roundings of partial sums bounded by S) = 2^-21 S of the exact one, the
// fp64 edge value within 2^-50 S, and t_f = fl(t) within 2^-24 t.  So when
// |e32 - t_f| > 2^-20 S_f + 2^-21 t_f (twice the bound) both agree on e <= t;
// otherwise the pixel takes pred_exact_d.  Invalid samples (non-finite or
// <= 0) and depths outside [2^-100, 2^100] force the exact path.  Valid for
// fx*b and t in [2^-40, 2^40] (host-checked, fill_predicate).

// ---------------------------------------------------------------------------
// PTX wrappers (sm_90+ async proxy; all used on sm_100a)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity), "r"(1000000u)  // suspend up to 1 ms per try: waiting warps stop issuing
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// L2 cache policy for the bulk row copies (createpolicy)
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// non-tensor bulk copy shared -> global (16-B aligned addresses, size % 16
// == 0) with an L2 cache policy
__device__ __forceinline__ void bulk_store_1d_hint(void* gdst, const void* src, uint32_t bytes,
                                                   uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_u32(src)), "r"(bytes), "l"(policy)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// three-input NaN-propagating min / max (FMNMX3.NAN on sm_100a), the |x|
// forms with free absolute-value operands
__device__ __forceinline__ float max3_nan(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float min3_nan(float a, float b, float c) {
  float r;
  asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

// ---------------------------------------------------------------------------
// closed-form normal (geometry.py:175-216, rescaled)
//
// The reference computes, for d > 0 and w = b/d, g = -dd/du:
//   n ~ (g w fx^2, -a2 w fx fy, ((a2 dv - g du) w - b) fx)
// Dividing by w*fx > 0 and multiplying by det > 0 (neither changes the
// direction) gives, with P1 = det*dd/du, P2 = det*dd/dv:
//   n ~ (-P1 fx, -P2 fy, P2 dv + P1 du - det d)
// which needs no division before the normalisation and cannot overflow for
// fp32-representable inputs.  The camera-facing flip never fires
// (n . X = -b fx z < 0, geometry.py:181-184), so none is applied.

__device__ __forceinline__ void normal_from_moments(double P1, double P2, double det, double d,
                                                    double du, double dv, double fx, double fy,
                                                    float& nx, float& ny, float& nz) {
  const double ax = -P1 * fx;
  const double ay = -P2 * fy;
  const double az = fma(P2, dv, fma(P1, du, -det * d));  // the cancelling component, in fp64
  // fp32 normalisation of the fp64-rounded components: the direction keeps
  // ~1e-7 relative accuracy (~6e-6 deg); out-of-range magnitudes take the
  // fp64 path so no input can overflow or underflow the fp32 squares
  const float fxv = (float)ax, fyv = (float)ay, fzv = (float)az;
  const float s = fmaf(fxv, fxv, fmaf(fyv, fyv, fzv * fzv));
  if (s > 1e-30f && s < 1e30f) {
    float r = rsqrtf(s);
    r = r * fmaf(-0.5f * s * r, r, 1.5f);  // one Newton step: ~1 ulp
    nx = fxv * r;
    ny = fyv * r;
    nz = fzv * r;
  } else {
    const double s64 = fma(ax, ax, fma(ay, ay, az * az));
    double inv;
    asm("rsqrt.approx.f64 %0, %1;" : "=d"(inv) : "d"(s64));
    inv = inv * fma(-0.5 * s64 * inv, inv, 1.5);
    nx = static_cast<float>(ax * inv);
    ny = static_cast<float>(ay * inv);
    nz = static_cast<float>(az * inv);
  }
}

// z = (fx b)/d; x = (u - u0) z / fx; y = (v - v0) z / fy  (geometry.py:39-64),
// fp32 with <= ~4 ulp relative error; NaN unless d is finite and > 0.
__device__ __forceinline__ void point_from_disparity(float d, float du, float dv, float fxb,
                                                     float inv_fx, float inv_fy, float& x,
                                                     float& y, float& z) {
  const bool ok = (d > 0.0f) && (d <= 3.402823466e38f);
  float r;
  asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(d));  // <= 1 ulp; z error <= ~3 ulp
  const float zz = ok ? fxb * r : __int_as_float(0x7fc00000);
  z = zz;
  x = du * zz * inv_fx;
  y = zz * (dv * inv_fy);  // = the fused pass (dv / fy hoisted per row)
}

// fp64-input variant (geometry.py:39-64 in double, then rounded to fp32).
__device__ __forceinline__ void point_from_disparity_f64(double d, double du, double dv,
                                                         const FixedParams& p, float& x, float& y,
                                                         float& z) {
  const bool ok = (d > 0.0) && (d <= 1.7976931348623157e308);
  if (ok) {
    const double zz = p.fxb / d;
    z = static_cast<float>(zz);
    x = static_cast<float>(du * zz / p.fx);
    y = static_cast<float>(dv * zz / p.fy);
  } else {
    x = y = z = __int_as_float(0x7fc00000);
  }
}

__device__ __forceinline__ bool finite_f(float v) { return fabsf(v) <= 3.402823466e38f; }
__device__ __forceinline__ bool finite_d(double v) { return fabs(v) <= 1.7976931348623157e308; }

}  // namespace sn
