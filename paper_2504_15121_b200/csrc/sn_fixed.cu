// Fused fixed-kernel oriented-point pass for sm_100a.
//
// Reference path (pkg/src/stereonorm): kernels.py:135-179 (_affine_pass:
// masked correlation with the precomputed LSQ weights, centre correction,
// support/border invalidation), kernels.py:237-261 (estimate_normals_fixed),
// geometry.py:175-216 (fused normal epilogue) and geometry.py:39-64,85-89
// (triangulation).  The reference never materialises the denoised map; nor
// does this pass: one launch reads the fp32 disparity once and writes the
// 24-byte (x, y, z, nx, ny, nz) record per pixel.
//
// Arithmetic: the weights s1 = vx/alpha, s2 = vy/alpha of a
// square pattern are integer offsets over an integer moment, so the device
// accumulates U = sum vx*d and V = sum vy*d EXACTLY in fp64 (fp32 inputs
// times small integers need < 53 bits) and divides by the moments once, in
// the rescaled normal formula of sn_common.cuh.  The square pattern is
// separable, so the sums are two sliding-window passes:
//   pass V (lane <-> column): C = sum_dy d,   Rr = sum_dy dy*d
//   pass H (lane <-> row):    U = sum_dx dx*C, V = sum_dx Rr
// each O(1) per pixel.  Every intermediate is an exact sum of the current
// window whenever the window's dynamic range fits 53 bits; columns/runs that
// hold |d| > 2^40 take a direct (non-sliding) path so no rounding can leak
// past the window.  Validity is tracked exactly with bit masks: a pixel is
// valid iff every support sample is inside the image and finite and the
// centre disparity is > 0; samples outside the image are
// masked by coordinate, which reproduces kernels.py:166-176.
//
// Data movement (B200): the input tile + halo is one 3D TMA load
// (cp.async.bulk.tensor) per item, prefetched while the previous item's
// pass H runs; the AoS-6 output tile is staged in row-major shared memory
// (pitch 3072 + 16 B: conflict-free float4 writes from lanes that own
// different rows) and leaves as one contiguous 3 KB bulk copy
// (cp.async.bulk, L2 evict_first) per output row, 16 per item, so HBM sees
// full-line writes only; the store lanes hand the staging tile back through
// an mbarrier that pass H waits on only after its sliding sums.  Persistent
// grid, two CTAs per SM.

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>

#include "sn_common.cuh"
#include "sn_internal.h"

namespace sn {

constexpr int kTW = 128;           // output columns per item
constexpr int kG = 16;             // output rows per item
constexpr int kCP = kG + 1;        // pitch of the column-major C/Rr/Dc arrays (odd)
constexpr int kHalfUnits = 160;    // pass-V units per half: 5 warps, 32-column aligned
constexpr int kFastThreads = 2 * kHalfUnits;  // 10 warps; pass H uses the first 8
constexpr int kRun = 8;            // output columns per pass-H lane
constexpr int kStoreTid = 8 * 32;  // warp 8 issues the output bulk stores
constexpr uint32_t kBigBits = 0x53800000u;  // fp32 bit pattern of 2^40
// row-major staging: one output row of an item (128
// records, 3072 B) per bulk copy; the 16-B pad makes the pitch 4 banks off,
// so the 8 lanes (= 8 rows) of each quarter-warp phase of pass H's 16-byte
// stores hit distinct banks
constexpr int kRowPitch = kTW * 24 + 16;
constexpr size_t kRowStageBytes = (size_t)kG * kRowPitch;

__host__ __device__ constexpr size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// accumulator of the sliding sums (see sval below): fp64, int32 for PNG16
template <typename T> struct AccOf { using type = double; using pair = double2; };
template <> struct AccOf<Png16> { using type = int; using pair = int2; };
template <typename T> using Acc = typename AccOf<T>::type;
template <typename T> using AccPair = typename AccOf<T>::pair;
template <typename T> constexpr bool kIntAcc = sizeof(Acc<T>) == 4;

template <int R, typename T>
struct FastCfg {
  static constexpr int NC = kTW + 2 * R;  // C/Rr columns (output columns + halo)
  static constexpr int NR = kG + 2 * R;   // input rows per item
  static constexpr int AE = 16 / (int)sizeof(T);
  // the box starts at (x0 - R) rounded down to 16 B, so it spans up to AE-1 extra columns
  static constexpr int BW = (NC + AE - 1 + AE - 1) / AE * AE;
  static constexpr size_t STAGE_BYTES = kRowStageBytes;
  static constexpr size_t IN_BYTES = (size_t)NR * BW * sizeof(T);
  static constexpr size_t CS_BYTES = (size_t)NC * kCP * sizeof(AccPair<T>);  // (C, Rr) [NC][kCP]
  // column flags (NC words) + 8-column block ORs of them (NB words)
  static constexpr int NB = (NC + 7) / 8;
  static constexpr size_t FL_BYTES = align_up((size_t)(NC + NB) * 4, 16);
  // shared-memory layout: 1 staging tile, 2 input tiles, 1 (C, Rr) array
  static constexpr size_t STAGE = 0;
  static constexpr size_t IN0 = STAGE + STAGE_BYTES;
  static constexpr size_t IN1 = align_up(IN0 + IN_BYTES, 128);
  static constexpr size_t CS = align_up(IN1 + IN_BYTES, 128);
  static constexpr size_t FL = align_up(CS + CS_BYTES, 16);
  static constexpr size_t BAR = align_up(FL + FL_BYTES, 16);
  // + slack for the 128-B base alignment
  static constexpr size_t TOTAL = BAR + 24 + 128;  // 3 mbarriers
  static_assert(NC <= kHalfUnits, "pass V: one unit per thread");
  static_assert(NR <= 32, "row validity bits must fit 32 bits");
};

template <typename T>
__device__ __forceinline__ bool finite_t(T v) {
  return fabs((double)v) <= 1.7976931348623157e308;
}
template <>
__device__ __forceinline__ bool finite_t<float>(float v) {
  return fabsf(v) <= 3.402823466e38f;
}

// |v| <= 2^40 (and finite): the sliding sums stay exact
template <typename T>
__device__ __forceinline__ bool small_t(T v) {
  return fabs((double)v) <= 1099511627776.0;
}
template <>
__device__ __forceinline__ bool small_t<float>(float v) {
  return (__float_as_uint(v) & 0x7fffffffu) <= kBigBits;
}

// disparity value of an input sample in fp64 (PNG16: the reference's
// (raw - 1.0) / scale, formats.py:147-149, invalid raw -> NaN)
template <typename T>
__device__ __forceinline__ double dval(T x, const FixedParams&) {
  return (double)x;
}
template <>
__device__ __forceinline__ double dval<Png16>(Png16 x, const FixedParams& p) {
  return png16_value(x.raw, p.png_invalid, p.png_scale, p.png_rcp);
}

// Accumulator of the sliding sums.  fp32/fp64 inputs: fp64, exact for the
// window's dynamic range.  PNG16: the integers raw - 1 in
// int32 -- |raw - 1| < 2^16, so C < 2^20, Rr < 2^23, U, V < 2^28 for R <= 8:
// exact, on the full-rate integer pipe instead of the fp64 one, and 8-byte
// (C, Rr) pairs in shared memory.  The 1/scale of d = (raw - 1)/scale is
// never applied to the sums: the normal is homogeneous of degree 1 in
// (U, V, d), so the integer sums with d_int = raw - 1 give the same direction
// (times sign(scale)).
// (AccOf: the accumulator types, defined above FastCfg)

__device__ __forceinline__ double2 make_pair(double a, double b) { return make_double2(a, b); }
// pairwise (tree) sum of N values: every partial sum here is exact (see the
// file header), so the association does not change the result -- only the
// length of the dependent chain (log2 N instead of N)
template <int N, typename A>
__device__ __forceinline__ A tree_sum(const A* x) {
  if constexpr (N == 1) return x[0];
  else return tree_sum<N / 2>(x) + tree_sum<N - N / 2>(x + N / 2);
}
__device__ __forceinline__ int2 make_pair(int a, int b) { return make_int2(a, b); }
// a + w * x: one FMA in fp64 (exact here), one IMAD in int32
__device__ __forceinline__ double mac(double w, double x, double a) { return fma(w, x, a); }
__device__ __forceinline__ int mac(int w, int x, int a) { return a + w * x; }

template <typename T>
__device__ __forceinline__ Acc<T> sval(T x, const FixedParams& p) {
  return dval(x, p);
}
template <>
__device__ __forceinline__ int sval<Png16>(Png16 x, const FixedParams&) {
  // Invalid samples keep their (finite, exact) value: pass V flags them from
  // the integer, and only windows that hold one -- invalid anyway -- see it
  // in their sums
  return (int)x.raw - 1;
}

// the fp32 epilogue's view of the centre sample: d rounded to fp32 and the
// exact "valid and d > 0" test.  PNG16: (raw - 1) * RN32(1/scale) (within ~1
// fp32 ulp of d; exact for power-of-two scales), and d > 0 decided on the
// integer: raw != invalid and sign(raw - 1) == sign(scale)
template <typename T>
__device__ __forceinline__ float dflt(T x, const FixedParams& p) {
  return (float)dval(x, p);
}
template <>
__device__ __forceinline__ float dflt<Png16>(Png16 x, const FixedParams& p) {
  // raw - 1 exactly: (2^23 + raw) - (2^23 + 1), an FADD instead of an I2F
  const float a = __fsub_rn(__int_as_float(0x4b000000 | (int)x.raw), 8388609.0f);
  const float v = __fmul_rn(a, p.png_rcp_f);
  return (int)x.raw == p.png_invalid ? __int_as_float(0x7fc00000) : v;
}
template <typename T>
__device__ __forceinline__ bool dpos(T x, const FixedParams& p) {
  return dval(x, p) > 0.0;
}
template <>
__device__ __forceinline__ bool dpos<float>(float x, const FixedParams&) {
  return x > 0.0f;  // = (double)x > 0, without the conversion
}
template <>
__device__ __forceinline__ float dflt<float>(float x, const FixedParams&) {
  return x;
}
template <>
__device__ __forceinline__ bool dpos<Png16>(Png16 x, const FixedParams& p) {
  // the caller's window test already excludes raw == invalid (the centre is
  // in its own support): only the sign of (raw - 1) / scale is left
  return ((int)x.raw - 1) * p.png_sign > 0;
}

// the centre value the normal's alpha*d term uses: d itself, or for PNG16
// (integer sums) raw - 1 exactly
template <typename T>
__device__ __forceinline__ float dnorm(T, float d) {
  return d;
}
template <>
__device__ __forceinline__ float dnorm<Png16>(Png16 x, float) {
  return __fsub_rn(__int_as_float(0x4b000000 | (int)x.raw), 8388609.0f);
}

// inputs whose records take the fp32 epilogue: fp32 disparities, and PNG16
// ones (the host admits only scales that keep every nonzero value in the
// fp32 normal range; d is rounded to fp32 once, ~6e-8 relative)
template <typename T>
constexpr bool kF32Epi = sizeof(T) <= 4;

// normal from the exact sums, fp32 after one rounding of U and V: the
// components are U fx, V fy and V dv + U du - alpha d, each bounded by ~|n|
// (n . (du, dv, fx) = -alpha d fx for a camera-facing normal), so fp32 adds
// only a few ulp of angle (~1e-5 deg); out-of-range magnitudes take the fp64
// path of normal_from_moments
__device__ __forceinline__ void normal_square(double U, double V, float alpha_f, float d,
                                              float du, float dv, float fx_f, float fy_f,
                                              const FixedParams& p, float& nx, float& ny,
                                              float& nz) {
  const float Uf = (float)U, Vf = (float)V;
  const float ax = -Uf * fx_f, ay = -Vf * fy_f;
  const float az = fmaf(Vf, dv, fmaf(Uf, du, -alpha_f * d));
  const float s = fmaf(ax, ax, fmaf(ay, ay, az * az));
  if (s > 1e-30f && s < 1e30f) {
    float r = rsqrtf(s);
    r = r * fmaf(-0.5f * s * r, r, 1.5f);  // one Newton step: ~1 ulp
    nx = ax * r;
    ny = ay * r;
    nz = az * r;
  } else {
    normal_from_moments(U, V, p.alpha, (double)d, (double)du, (double)dv, p.fx, p.fy, nx, ny, nz);
  }
}

// rare paths of the epilogue, kept out of line so the hot loop stays small
// (eight inlined copies of the fp64 normal and four of the fp64 division per
// pass-H lane otherwise)
__device__ __noinline__ float3 normal_rare(double U, double V, double alpha, double d, double du,
                                           double dv, double fx, double fy) {
  float3 n;
  normal_from_moments(U, V, alpha, d, du, dv, fx, fy, n.x, n.y, n.z);
  return n;
}
__device__ __noinline__ float depth_rare(double fxb, float d) { return (float)(fxb / (double)d); }

// Oriented-point records of two neighbouring pixels (same row) with packed
// f32x2 arithmetic (FFMA2/FMUL2 on sm_100a).  Point: z = fxb/d (rcp.approx,
// <= ~3 ulp), x = du z / fx, y = dv z / fy, NaN unless d is finite and > 0;
// subnormal d takes an fp64 division (flush-to-zero would turn a finite z
// into inf).  Normal: normal_square's formula for both pixels; a pixel whose
// |n|^2 leaves fp32's comfortable range takes the fp64 path.  A = int: PNG16
// sums of raw - 1 with dn = raw - 1 (the normal is homogeneous in (U, V, d):
// same direction as with d = (raw - 1)/scale, up to sign(scale)); else
// dn = d.
//
// NANOK (fp32 input): the validity test folds into the arithmetic -- the
// fixed depth zz is NaN exactly when d is not a positive value, so r + (zz -
// zz) is r or NaN; pixels whose window holds an invalid sample or whose depth
// overflowed to inf (rare2, bit e for pixel e; usually 0) take the explicit
// test.  Otherwise ok0 / ok1 are the pixels' validity.
template <typename A, bool NANOK = false>
__device__ __forceinline__ void records_pair(A U0, A V0, A U1, A V1, float d0, float d1, float dn0,
                                             float dn1, float2 zz, bool ok0, bool ok1, float duh,
                                             float dv, const FixedParams& p, float* o,
                                             uint32_t wb2 = 0u, uint32_t rare2 = 0u,
                                             float2* s_out = nullptr) {
  constexpr bool kInt = sizeof(A) == 4;
  // points; zz = the depths as fixed by the caller (pass_h: fxb_f * rcp(d),
  // or NaN / an fp64 division where that leaves (0, FLT_MAX)); duh = (x -
  // u0_hi) exactly, du = duh - u0_lo
  const float2 dd = make_float2(dn0, dn1);
  // (duh, duh + 1) exactly, then one packed subtraction: the same roundings
  const float2 du = __fadd2_rn(make_float2(duh, duh + 1.0f), make_float2(-p.u0_lo, -p.u0_lo));
  const float2 px = __fmul2_rn(__fmul2_rn(du, zz), make_float2(p.inv_fx_f, p.inv_fx_f));
  // dv / fy is a per-row constant (hoisted out of the run): one product per pixel
  const float dvy = dv * p.inv_fy_f;
  const float2 py = __fmul2_rn(zz, make_float2(dvy, dvy));
  o[0] = px.x;
  o[1] = py.x;
  o[2] = zz.x;
  o[6] = px.y;
  o[7] = py.y;
  o[8] = zz.y;
  // normals
  const float2 Uf = make_float2((float)U0, (float)U1), Vf = make_float2((float)V0, (float)V1);
  const float nfx = p.nfx_f, nfy = p.nfy_f, nal = p.nal_f;
  const float2 ax = __fmul2_rn(Uf, make_float2(nfx, nfx));
  const float2 ay = __fmul2_rn(Vf, make_float2(nfy, nfy));
  const float2 az = __ffma2_rn(Vf, make_float2(dv, dv),
                               __ffma2_rn(Uf, du, __fmul2_rn(make_float2(nal, nal), dd)));
  const float2 s = __ffma2_rn(ax, ax, __ffma2_rn(ay, ay, __fmul2_rn(az, az)));
  // rsqrt.approx (relative error <= 2^-22.9): the common scale of the three
  // components leaves the direction untouched; |n| - 1 stays below ~3e-7
  float2 r = make_float2(rsqrt_ftz(s.x), rsqrt_ftz(s.y));
  if constexpr (kInt) {
    if (p.png_sign < 0) r = make_float2(-r.x, -r.y);
  }
  // an invalid pixel's normal is NaN: one select on r instead of three on n
  if constexpr (NANOK) {
    const float2 r_in = r;
    r = __fadd2_rn(r, __fadd2_rn(zz, make_float2(-zz.x, -zz.y)));
    if (rare2) {  // ok = dpos and support clear
      ok0 = !(wb2 & 1u) && d0 > 0.0f;
      ok1 = !(wb2 & 2u) && d1 > 0.0f;
      r.x = ok0 ? r_in.x : __int_as_float(0x7fc00000);
      r.y = ok1 ? r_in.y : __int_as_float(0x7fc00000);
    } else if (s_out == nullptr) {
      ok0 = !(wb2 & 1u) && d0 > 0.0f;
      ok1 = !(wb2 & 2u) && d1 > 0.0f;
    }
  } else {
    if (!ok0) r.x = __int_as_float(0x7fc00000);
    if (!ok1) r.y = __int_as_float(0x7fc00000);
  }
  const float2 nx = __fmul2_rn(ax, r), ny = __fmul2_rn(ay, r), nz = __fmul2_rn(az, r);
  o[3] = nx.x;
  o[4] = ny.x;
  o[5] = nz.x;
  o[9] = nx.y;
  o[10] = ny.y;
  o[11] = nz.y;
  if (s_out != nullptr) {  // the caller tests the range once for its whole run
    *s_out = s;
    return;
  }
  // both |n|^2 in fp32's comfortable range (NaN-propagating min/max: a NaN
  // fails the test) -- else the per-pixel checks below
  float smin, smax;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(smin) : "f"(s.x), "f"(s.y));
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(smax) : "f"(s.x), "f"(s.y));
  if (smin > 1e-30f && smax < 1e30f) return;
  const bool in0 = s.x > 1e-30f && s.x < 1e30f, in1 = s.y > 1e-30f && s.y < 1e30f;
  // the rare fp64 path works on the disparity sums: integer sums / scale
  auto dsum = [&](A u) -> double {
    if constexpr (kInt) return __ddiv_rn((double)u, p.png_scale);
    else return u;
  };
  if (ok0 && !in0) {
    const float3 n = normal_rare(dsum(U0), dsum(V0), p.alpha, (double)d0, (double)du.x,
                                 (double)dv, p.fx, p.fy);
    o[3] = n.x;
    o[4] = n.y;
    o[5] = n.z;
  }
  if (ok1 && !in1) {
    const float3 n = normal_rare(dsum(U1), dsum(V1), p.alpha, (double)d1, (double)du.y,
                                 (double)dv, p.fx, p.fy);
    o[9] = n.x;
    o[10] = n.y;
    o[11] = n.z;
  }
}

// ---------------------------------------------------------------------------
// fast path: centred square pattern, radius R
//
// Per item (128 columns x 16 rows of one frame):
//   pass V  unit = (half h, column c), 5 warps per half, lane <-> column, so
//           each warp covers 32 aligned columns.  C, Rr for the 8 output rows
//           of the half as a sliding chain -> smem, column-major (pitch 17
//           doubles: conflict-free for both passes), validity bits per column
//           (bit 8 of a half's flags: a sample too large for exact sliding).
//           With a threshold, the same registers give the ST-passable bits:
//           depths of the unit's rows, left/right depths by shuffle, one
//           ballot per row.
//   pass H  8 warps, lane <-> (output row, run of 8 columns): U, V as a
//           sliding chain, closed-form normal + point (packed f32x2), 6 floats
//           per pixel into the staging tile, bulk row stores.
// fixed_square_kernel runs the passes (2 CTAs/SM, separated by CTA barriers,
// any R <= 8, fp32/fp64/PNG16 input).

struct ItemDecoder {
  int tiles_x, tiles_y;
  double inv_tx, inv_ty;
  __device__ ItemDecoder(int tx, int ty)
      : tiles_x(tx), tiles_y(ty), inv_tx(1.0 / (double)tx), inv_ty(1.0 / (double)ty) {}
  __device__ static unsigned udiv(unsigned u, unsigned d, double inv) {  // exact for u < 2^31
    unsigned q = (unsigned)((double)u * inv);
    if (q * d > u) --q;
    else if ((q + 1) * d <= u) ++q;
    return q;
  }
  __device__ void operator()(int it, int& x0, int& y0, int& bz) const {
    const unsigned u = (unsigned)it;
    const unsigned r = udiv(u, (unsigned)tiles_x, inv_tx);
    x0 = (int)(u - r * (unsigned)tiles_x) * kTW;
    const unsigned f = udiv(r, (unsigned)tiles_y, inv_ty);
    y0 = (int)(r - f * (unsigned)tiles_y) * kG;
    bz = (int)f;
  }
};

// the persistent loop's item coordinates, advanced by gridDim.x items per
// step as a mixed-radix addition (one decode per CTA instead of one per item
// and thread); the step's digits are each below their radix, so one carry
// per digit at most
struct ItemWalk {
  int tx, ty, bz, dtx, dty, dbz, tiles_x, tiles_y;
  __device__ ItemWalk(const ItemDecoder& dec, int item, int step)
      : tiles_x(dec.tiles_x), tiles_y(dec.tiles_y) {
    dec(item, tx, ty, bz);
    dec(step, dtx, dty, dbz);
    tx /= kTW;
    ty /= kG;
    dtx /= kTW;
    dty /= kG;
  }
  __device__ void advance() {
    tx += dtx;
    int cy = 0;
    if (tx >= tiles_x) {
      tx -= tiles_x;
      cy = 1;
    }
    ty += dty + cy;
    int cz = 0;
    if (ty >= tiles_y) {
      ty -= tiles_y;
      cz = 1;
    }
    bz += dbz + cz;
  }
  __device__ int x0() const { return tx * kTW; }
  __device__ int y0() const { return ty * kG; }
};

// TMA tile origin: the halo origin with its innermost coordinate rounded
// down to a 16-byte multiple (an unaligned innermost TMA coordinate raises
// an illegal-instruction fault on this part -- measured with
// tools/ubench/tma_probe.cu).  Negative aligned coordinates are fine; the
// samples outside the image are masked by coordinate in pass V, which
// reproduces the no-padding border rule kernels.py:166-176 (and arrive as
// zeros, i.e. invalid depths, for the passable predicate).
// OR of x >> j for j in [0, N): bit i = any of bits i .. i+N-1.  Doubling
// spans up to the largest power of two P <= N, then the remaining N - P
// (2 log N shift-ors instead of N)
__host__ __device__ constexpr int pow2_floor(int n) { return n >= 2 ? 2 * pow2_floor(n / 2) : 1; }
template <int N>
__device__ __forceinline__ uint32_t window_or(uint32_t x) {
  if constexpr (N <= 1) {
    return x;
  } else {
    constexpr int P = pow2_floor(N);
    uint32_t a = x;
#pragma unroll
    for (int span = 1; span < P; span *= 2) a |= a >> span;
    if constexpr (P < N) a |= window_or<N - P>(x >> P);
    return a;
  }
}

template <int R, int AE>
__device__ __forceinline__ int tile_x0(int x0) {
  return (x0 - R) & ~(AE - 1);
}

// pass V for unit (h, c) of one item.  Every thread of the 10 pass-V warps
// calls it (the shuffles/ballots need full warps); `unit` is false for the
// idle lanes beyond NC.
template <int R, typename T>
__device__ __forceinline__ void pass_v(const T* in, int sh, int x0, int y0, int H, int W, int h,
                                       int c, bool unit, AccPair<T>* CR, uint32_t* fl,
                                       const FixedParams& p) {
  using Cfg = FastCfg<R, T>;
  using A = Acc<T>;
  constexpr int BW = Cfg::BW;
  constexpr int NC = Cfg::NC;
  // all operands live in shared memory: let the compiler emit LDS/STS
  __builtin_assume(__isShared(in));
  __builtin_assume(__isShared(CR));
  __builtin_assume(__isShared(fl));
  constexpr int NWIN = 2 * R + 1;
  constexpr int HG = kG / 2;      // rows per pass-V unit
  constexpr int NV = HG + 2 * R;  // input rows read per pass-V unit
  const int gx = x0 - R + c;
  const int r0 = h * HG;  // first input row of the unit (item-relative, incl. halo)
  const T* col = in + r0 * BW + c + sh;
  // the unit's column of the input tile and its (C, Rr) entries stay inside
  // their shared-memory arrays
  SN_ASSERT(!unit || (c + sh >= 0 && c + sh < BW && r0 + NV <= Cfg::NR && c < NC &&
                      r0 + HG <= kCP));
  T raw[NV];
  bool all_small = true;  // every sample finite with |v| <= 2^40 (sliding sums exact)
  uint32_t png_inv = 0;   // PNG16: bit i = sample i is the invalid value
  uint32_t f16 = 0;       // this unit's column flags (0 for idle lanes)
  if (unit) {
    if constexpr (sizeof(T) == 4) {
      // |v| <= 2^40 for every sample (NaN fails): a chain of three-input
      // NaN-propagating maxima of |v|, one compare
#pragma unroll
      for (int i = 0; i < NV; ++i) raw[i] = col[i * BW];
      float m = fabsf(raw[0]);
      int i = 1;
#pragma unroll
      for (; i + 1 < NV; i += 2) m = max3_nan(m, fabsf(raw[i]), fabsf(raw[i + 1]));
      if (i < NV) m = max3_nan(m, fabsf(raw[i]), fabsf(raw[i]));
      all_small = m <= 1099511627776.0f;
    } else if constexpr (sizeof(T) == 2) {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        raw[i] = col[i * BW];
        png_inv |= ((int)raw[i].raw == p.png_invalid ? 1u : 0u) << i;
      }
    } else {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        raw[i] = col[i * BW];
        all_small &= fabs(sval(raw[i], p)) <= 1099511627776.0;  // 2^40, NaN fails
      }
    }
  }
  if (unit) {
    // rows of the unit inside the image
    const int lo = max(0, R - y0 - r0), hi = min(NV, H - y0 + R - r0);
    uint32_t inside = 0;
    if ((unsigned)gx < (unsigned)W && hi > lo) inside = (uint32_t)(((1ull << (hi - lo)) - 1ull) << lo);
    A v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = sval(raw[i], p);
    constexpr uint32_t kAll = (NV >= 32) ? 0xffffffffu : ((1u << NV) - 1u);
    uint32_t fin = kAll & ~png_inv;
    bool big = false;
    if constexpr (!kIntAcc<T>) if (!all_small) {
      // rare: non-finite (zeroed so the sliding sums stay finite) or huge samples
      fin = 0;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const bool f = finite_d(v[i]);
        fin |= (f ? 1u : 0u) << i;
        big |= f && !(fabs(v[i]) <= 1099511627776.0);
        if (!f) v[i] = 0.0;
      }
    }
    const uint32_t invb = ~(fin & inside);
    AccPair<T>* cr = CR + c * kCP + r0;
    if (!big) {
      // first window as trees (exact sums: any association gives the same)
      A C = tree_sum<NWIN>(v);
      A wd[R];
#pragma unroll
      for (int k = 1; k <= R; ++k) wd[k - 1] = (A)k * (v[R + k] - v[R - k]);
      A Rr = tree_sum<R>(wd);
      cr[0] = make_pair(C, Rr);
#pragma unroll
      for (int g = 1; g < HG; ++g) {
        const A vin = v[g + 2 * R], vout = v[g - 1];
        const A tin = mac((A)R, vout, (A)(R + 1) * vin);  // off the chain
        C += vin - vout;
        Rr = (Rr - C) + tin;
        cr[g] = make_pair(C, Rr);
      }
    } else {
      // rare (fp inputs, a sample above 2^40): direct sums per output row,
      // re-read from the tile (non-finite samples as 0) in a rolled loop to
      // keep the kernel's code small
#pragma unroll 1
      for (int g = 0; g < HG; ++g) {
        A C = 0, Rr = 0;
#pragma unroll
        for (int j = 0; j < NWIN; ++j) {
          A x = sval(col[(g + j) * BW], p);
          if constexpr (!kIntAcc<T>) x = finite_d(x) ? x : 0.0;
          C += x;
          Rr = mac((A)(j - R), x, Rr);
        }
        cr[g] = make_pair(C, Rr);
      }
    }
    const uint32_t acc = window_or<NWIN>(invb);
    // flags of column c, half h: bits 0-7 = support of output row 8h+i holds
    // an invalid sample, bit 8 = the half's sums were computed directly
    f16 = (acc & 0xFFu) | (big ? 0x100u : 0u);
    reinterpret_cast<uint16_t*>(fl + c)[h] = (uint16_t)f16;
  }
  // OR of the flags of the 8-column block of c (the warp's lanes are 32
  // aligned columns of one half): pass H reads 2-3 block words per run
  // instead of every column's flags
  f16 |= __shfl_xor_sync(0xffffffffu, f16, 1);
  f16 |= __shfl_xor_sync(0xffffffffu, f16, 2);
  f16 |= __shfl_xor_sync(0xffffffffu, f16, 4);
  if ((c & 7) == 0 && (c >> 3) < Cfg::NB) reinterpret_cast<uint16_t*>(fl + NC + (c >> 3))[h] = (uint16_t)f16;
}

// pass H + epilogue for lane hl (< 256) of one item; records into the
// row-major padded staging tile (kRowPitch)
template <int R, typename T>
__device__ __forceinline__ void pass_h(int hl, const T* in, int sh, int x0, int y0, int bz, int H,
                                       int W, const AccPair<T>* CR, const uint32_t* fl,
                                       uint32_t stage_base, const FixedParams& p,
                                       uint8_t* mask_out, uint64_t* sfree, uint32_t sparity) {
  using Cfg = FastCfg<R, T>;
  using A = Acc<T>;
  __builtin_assume(__isShared(in));
  __builtin_assume(__isShared(CR));
  __builtin_assume(__isShared(fl));
  constexpr int BW = Cfg::BW;
  constexpr int NWIN = 2 * R + 1;
  constexpr int NH = kRun + 2 * R;  // C/Rr columns read per pass-H lane
  const int g = hl & 15;
  const int q = hl >> 4;  // run of kRun output columns
  const int colbase = q * kRun;
  A cc[NH], rr[NH];
#pragma unroll
  for (int i = 0; i < NH; ++i) {
    const AccPair<T> v = CR[(colbase + i) * kCP + g];
    cc[i] = v.x;
    rr[i] = v.y;
  }
  // flags of the run's NH columns: the ORs of its 8-column blocks (pass V)
  uint32_t any = 0;
#pragma unroll
  for (int b = 0; b < (NH + 7) / 8; ++b) any |= fl[Cfg::NC + (colbase >> 3) + b];
  const uint32_t hshift = (uint32_t)(g & 8) * 2;  // 0 or 16: the half of row g
  const bool big = ((any >> (hshift + 8)) & 1u) != 0u;
  uint32_t win = 0;  // bit j: support of output j holds an invalid sample
  if (((any >> hshift) & 0xFFu) != 0u) {
    uint32_t colinv = 0;
#pragma unroll
    for (int i = 0; i < NH; ++i) colinv |= ((fl[colbase + i] >> (hshift + (g & 7))) & 1u) << i;
    win = window_or<NWIN>(colinv);
  }

  const int yg = y0 + g;
  const int xb = x0 + colbase;
  const int yv = p.row0 + yg;  // image row (strips: block row + offset)
  const double dv = (double)yv - p.v0;
  const float dv_f = ((float)yv - p.v0_hi) - p.v0_lo;
  const float du_hi = (float)xb - p.u0_hi;  // exact; + j stays exact
  const T* drow = in + (g + R) * BW + colbase + R + sh;  // centre disparities of the run
  SN_ASSERT(colbase + NH <= Cfg::NC && colbase + R + sh + kRun <= BW && sh >= 0 && g + R < Cfg::NR);
  // staging address of chunk c (0..11, 16 B) of this run: row g, 192 B per run
  const uint32_t row_a = stage_base + (uint32_t)g * (uint32_t)kRowPitch + (uint32_t)q * 192u;
  auto stg_addr = [&](int c) { return row_a + (uint32_t)c * 16u; };

  // sliding sums first (short dependent chain), then independent epilogues
  A Us[kRun], Vs[kRun];
  if (!big) {
    // first window as trees: U = sum_k k (c[R+k] - c[R-k])
    A Bx = tree_sum<NWIN>(cc), V = tree_sum<NWIN>(rr);
    A wd[R];
#pragma unroll
    for (int k = 1; k <= R; ++k) wd[k - 1] = (A)k * (cc[R + k] - cc[R - k]);
    A U = tree_sum<R>(wd);
    Us[0] = U;
    Vs[0] = V;
#pragma unroll
    for (int j = 1; j < kRun; ++j) {
      const A cin = cc[j + 2 * R], cout = cc[j - 1];
      const A tin = mac((A)R, cout, (A)(R + 1) * cin);  // independent of the chain
      Bx += cin - cout;
      U = (U - Bx) + tin;
      V += rr[j + 2 * R] - rr[j - 1];
      Us[j] = U;
      Vs[j] = V;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kRun; ++j) {
      A U = 0, V = 0;
#pragma unroll
      for (int i = 0; i < NWIN; ++i) {
        U = mac((A)(i - R), cc[j + i], U);
        V += rr[j + i];
      }
      Us[j] = U;
      Vs[j] = V;
    }
  }
  // depths zf = fxb * rcp(d) of the run's pixels (zc[1 .. kRun])
  float zc[kRun + 2], df[kRun];
  uint32_t zinf = 0;  // bit j: pixel j's depth overflowed fp32 (fp64 division > FLT_MAX)
#pragma unroll
  for (int j = 0; j < kRun; ++j) {
    df[j] = dflt(drow[j], p);
    zc[j + 1] = __fmul_rn(p.fxb_f, rcp_ftz(df[j]));
  }
  // zf is finite and > 0 exactly when d is a normal positive disparity whose
  // reciprocal does not flush; anything else -- d invalid (NaN, <= 0, +inf:
  // the point is NaN), subnormal, or so large or small that rcp or the
  // product leaves the normal range -- is fixed here, once for the run
  // (NaN-propagating min / max: one test for its 8 depths)
  {
    float lo = zc[1], hi = zc[1];
    static_assert(kRun % 2 == 0, "depth test: pairs after the first");
#pragma unroll
    for (int j = 2; j + 1 <= kRun; j += 2) {
      lo = min3_nan(lo, zc[j], zc[j + 1]);
      hi = max3_nan(hi, zc[j], zc[j + 1]);
    }
    lo = min3_nan(lo, zc[kRun], zc[kRun]);
    hi = max3_nan(hi, zc[kRun], zc[kRun]);
    if (!(lo > 0.0f && hi < 3.402823466e38f)) {
#pragma unroll
      for (int j = 0; j < kRun; ++j)
        if (!(zc[j + 1] > 0.0f && zc[j + 1] < 3.402823466e38f)) {
          zc[j + 1] = (df[j] > 0.0f && df[j] <= 3.402823466e38f) ? depth_rare(p.fxb, df[j])
                                                                : __int_as_float(0x7fc00000);
          if (zc[j + 1] == __int_as_float(0x7f800000)) zinf |= 1u << j;  // z beyond fp32
        }
    }
  }
  // the staging tile is free once the previous item's bulk stores have read it
  mbar_wait(sfree, sparity);
  float o[12];
  float2 srun[kRun / 2];  // fp32 input: |n|^2 of the run's pixels
#pragma unroll
  for (int j = 0; j < kRun; j += 2) {
    const bool ok0 = (((win >> j) & 1u) == 0u) && dpos(drow[j], p);
    const bool ok1 = (((win >> (j + 1)) & 1u) == 0u) && dpos(drow[j + 1], p);
    // fp64 inputs take the fp32 epilogue too when both centre samples are
    // invalid or within [2^-100, 2^100] (d rounded once to fp32: ~6e-8
    // relative); others -- fp32-subnormal or huge disparities -- the fp64 one
    bool f32_epi = kF32Epi<T>;
    if constexpr (sizeof(T) == 8) {
      auto safe = [](double d) {
        return !(d > 0.0 && d <= 1.7976931348623157e308) ||
               (d >= 7.888609052210118e-31 && d <= 1.2676506002282294e30);
      };
      f32_epi = safe((double)drow[j]) && safe((double)drow[j + 1]);
    }
    if constexpr (sizeof(T) == 4 && !kIntAcc<T>) {
      // fp32 input: validity from the fixed depths and the support bits
      records_pair<A, true>(Us[j], Vs[j], Us[j + 1], Vs[j + 1], df[j], df[j + 1], df[j],
                            df[j + 1], make_float2(zc[j + 1], zc[j + 2]), false, false,
                            du_hi + (float)j, dv_f, p, o, (win >> j) & 3u,
                            ((win | zinf) >> j) & 3u, &srun[j >> 1]);
    } else if (f32_epi) {
      records_pair(Us[j], Vs[j], Us[j + 1], Vs[j + 1], df[j], df[j + 1], dnorm(drow[j], df[j]),
                   dnorm(drow[j + 1], df[j + 1]), make_float2(zc[j + 1], zc[j + 2]), ok0, ok1,
                   du_hi + (float)j, dv_f, p, o);
    } else {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double dcv = dval(drow[j + e], p);
        const double du = (double)(xb + j + e) - p.u0;
        float* r = o + 6 * e;
        point_from_disparity_f64(dcv, du, dv, p, r[0], r[1], r[2]);
        if (e ? ok1 : ok0) {
          const float3 n = normal_rare(Us[j + e], Vs[j + e], p.alpha, dcv, du, dv, p.fx, p.fy);
          r[3] = n.x;
          r[4] = n.y;
          r[5] = n.z;
        } else
          r[3] = r[4] = r[5] = __int_as_float(0x7fc00000);
      }
    }
    // pixels (j, j+1) = 12 floats = chunks c .. c+2 of the run (stg_addr)
#pragma unroll
    for (int t = 0; t < 3; ++t)
      st_shared_v4(stg_addr((j >> 1) * 3 + t), o[4 * t], o[4 * t + 1], o[4 * t + 2], o[4 * t + 3]);
  }
  if constexpr (sizeof(T) == 4 && !kIntAcc<T>) {
    // |n|^2 of the whole run in fp32's comfortable range (NaN-skipping: a NaN
    // comes from an invalid sample, whose normal is NaN anyway) -- else the
    // fp64 normal of every valid pixel out of range, over its staged record
    float smin = srun[0].x, smax = srun[0].x;
#pragma unroll
    for (int k = 0; k < kRun / 2; ++k) {
      smin = fminf(fminf(smin, srun[k].x), srun[k].y);
      smax = fmaxf(fmaxf(smax, srun[k].x), srun[k].y);
    }
    if (!(smin > 1e-30f && smax < 1e30f)) {
#pragma unroll
      for (int k = 0; k < kRun; ++k) {
        const float sk = (k & 1) ? srun[k >> 1].y : srun[k >> 1].x;
        const bool ok = !((win >> k) & 1u) && df[k] > 0.0f;
        if (ok && !(sk > 1e-30f && sk < 1e30f)) {
          const float du = __fsub_rn(du_hi + (float)k, p.u0_lo);
          const float3 n = normal_rare(Us[k], Vs[k], p.alpha, (double)df[k], (double)du,
                                       (double)dv_f, p.fx, p.fy);
          const uint32_t a = row_a + (uint32_t)k * 24u + 12u;
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(n.x) : "memory");
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(a + 4u), "f"(n.y) : "memory");
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(a + 8u), "f"(n.z) : "memory");
        }
      }
    }
  }
  if (mask_out != nullptr && yg < H) {
    // the validity bits, recomputed here so the hot loop does not carry them
    uint32_t validbits = 0;
#pragma unroll
    for (int j = 0; j < kRun; ++j)
      validbits |= ((((win >> j) & 1u) == 0u && dpos(drow[j], p)) ? 1u : 0u) << j;
    uint8_t* mrow = mask_out + ((int64_t)bz * H + yg) * W + xb;
    if (xb + kRun <= W && (reinterpret_cast<uintptr_t>(mrow) & 7u) == 0) {
      // one 8-byte store: bit j -> byte j
      const uint32_t lo = (validbits & 1u) | ((validbits & 2u) << 7) | ((validbits & 4u) << 14) |
                          ((validbits & 8u) << 21);
      const uint32_t hb = validbits >> 4;
      const uint32_t hi = (hb & 1u) | ((hb & 2u) << 7) | ((hb & 4u) << 14) | ((hb & 8u) << 21);
      *reinterpret_cast<uint2*>(mrow) = make_uint2(lo, hi);
    } else {
#pragma unroll 1
      for (int j = 0; j < kRun && xb + j < W; ++j) mrow[j] = (uint8_t)((validbits >> j) & 1u);
    }
  }
}

// ---------------------------------------------------------------------------
// classic kernel: persistent, 2 CTAs/SM, the passes of one item separated by
// CTA barriers; the next item's input is prefetched during the current item

template <int R, typename T>
__global__ void __launch_bounds__(kFastThreads, 2)
    fixed_square_kernel(const __grid_constant__ CUtensorMap in_map, const FixedParams p,
                        uint8_t* __restrict__ mask_out, float* __restrict__ out6,
                        const int64_t out_pitch, const int n_items, const int tiles_x,
                        const int tiles_y) {
  using Cfg = FastCfg<R, T>;
  constexpr int NC = Cfg::NC, AE = Cfg::AE;
  constexpr int kStoreLanes = kG;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  // 128-B aligned base; offset arithmetic on the __shared__ array keeps the
  // shared address space (LDS/STS, not generic LD/ST)
  constexpr uint32_t kAlign = 128u;
  uint8_t* smem = smem_raw + ((kAlign - (smem_u32(smem_raw) & (kAlign - 1u))) & (kAlign - 1u));
  AccPair<T>* CR = reinterpret_cast<AccPair<T>*>(smem + Cfg::CS);
  uint32_t* fl = reinterpret_cast<uint32_t*>(smem + Cfg::FL);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::BAR);
  const uint32_t stage_base = smem_u32(smem + Cfg::STAGE);
  const int tid = threadIdx.x;
  const int W = (int)p.W, H = (int)p.H;

  int item = blockIdx.x;
  if (item >= n_items) return;
  const ItemDecoder decode(tiles_x, tiles_y);
  ItemWalk cur(decode, item, (int)gridDim.x), nxt = cur;
  nxt.advance();
  auto load_tile = [&](const ItemWalk& w, int buf) {
    T* dst = reinterpret_cast<T*>(smem + (buf ? Cfg::IN1 : Cfg::IN0));
    mbar_arrive_expect_tx(bar + buf, (uint32_t)Cfg::IN_BYTES);
    tma_load_3d(dst, &in_map, bar + buf, tile_x0<R, AE>(w.x0()), w.y0() - R, w.bz);
  };

  if (tid == 0) {
    tma_prefetch_desc(&in_map);
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_init(bar + 2, kStoreLanes);  // staging free (the store lanes' bulk reads done)
    fence_mbar_init();
    load_tile(cur, 0);
  }
  __syncthreads();

  const int h = tid >= kHalfUnits ? 1 : 0;  // pass-V unit of this thread
  const int c = tid - h * kHalfUnits;
  const bool unit = c < NC;

  for (int it = 0; item < n_items; ++it, item += gridDim.x, cur = nxt, nxt.advance()) {
    const int buf = it & 1;
    if (tid == 0 && item + (int)gridDim.x < n_items) load_tile(nxt, buf ^ 1);
    const int x0 = cur.x0(), y0 = cur.y0(), bz = cur.bz;
    const int sh = (x0 - R) - tile_x0<R, AE>(x0);  // logical column c <-> smem column c + sh
    const T* in = reinterpret_cast<const T*>(smem + (buf ? Cfg::IN1 : Cfg::IN0));
    mbar_wait(bar + buf, (uint32_t)(it >> 1) & 1u);

    pass_v<R, T>(in, sh, x0, y0, H, W, h, c, unit, CR, fl, p);
    __syncthreads();

    if (tid < kStoreTid) {
      pass_h<R, T>(tid, in, sh, x0, y0, bz, H, W, CR, fl, stage_base, p, mask_out, bar + 2,
                   (uint32_t)it & 1u);
    } else if (tid >= kStoreTid && tid < kStoreTid + kStoreLanes) {
      // the store lanes (idle in pass H): the previous item's bulk stores have
      // read the staging tile -> pass H may write it (waited for there, after
      // its sliding sums, instead of before the barrier above)
      bulk_wait_read0();
      mbar_arrive(bar + 2);
    }
    fence_proxy_async_smem();
    __syncthreads();
    // output stores from a warp that is idle in pass H -- warp 0 goes
    // straight on to the next item
    if (tid >= kStoreTid && tid < kStoreTid + kStoreLanes) {
      const int b = tid - kStoreTid;
      // one contiguous bulk copy per output row (3072 B, less at the right
      // edge).  The pitch is even, so rows start 16-B aligned and a row
      // ends on a 16-B multiple; an odd width writes into a pitched buffer
      // (dispatch_square_staged), whose pad column takes the extra record
      if (y0 + b < H) {
        const int n = min(kTW, (int)out_pitch - x0);
        // the row's records stay inside the [B][H][out_pitch] output
        SN_ASSERT(n > 0 && x0 + n <= out_pitch && bz < p.B && y0 + b < H);
        // L2 evict_first: the 24 B/px of records stream through L2 without
        // pushing out the input rows the vertically adjacent item reads as
        // its halo (DRAM reads 1.08x -> 1.00x of the 4 B/px, DESIGN 4.1)
        bulk_store_1d_hint(out6 + (((int64_t)bz * H + y0 + b) * out_pitch + x0) * 6,
                           smem + Cfg::STAGE + (size_t)b * kRowPitch, (uint32_t)n * 24u,
                           policy_evict_first());
      }
      bulk_commit();
    }
  }
  if (tid >= kStoreTid && tid < kStoreTid + kStoreLanes) bulk_wait0();
}

// ---------------------------------------------------------------------------
// generic path: any offset pattern, any shape (direct sums U = sum vx d,
// V = sum vy d in fp64, in the pattern's order)

// the record / affine output of one pixel from its sums (shared by both
// generic kernels)
template <typename T, bool AFFINE>
__device__ __forceinline__ void generic_out(int64_t idx, int64_t x, int64_t y, T dc, bool ok,
                                            double U, double V, const FixedParams& p,
                                            float* __restrict__ out6, uint8_t* __restrict__ mask,
                                            double* __restrict__ a1, double* __restrict__ a2) {
  const double dcd = (double)dc;
  const double Up = U - p.sx * dcd;
  const double Vp = V - p.sy * dcd;
  const double P1 = p.gamma * Up - p.beta * Vp;  // det * dd/du
  const double P2 = p.alpha * Vp - p.beta * Up;  // det * dd/dv
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  if (AFFINE) {
    a1[idx] = ok ? 1.0 + P1 / p.det : qnan;
    a2[idx] = ok ? P2 / p.det : qnan;
    if (mask) mask[idx] = ok ? 1 : 0;
  } else {
    const bool valid = ok && (dc > (T)0);
    float px, py, pz, nx, ny, nz;
    if constexpr (sizeof(T) == 4) {
      const float du_f = ((float)x - p.u0_hi) - p.u0_lo;
      const float dv_f = ((float)(y + p.row0) - p.v0_hi) - p.v0_lo;
      point_from_disparity((float)dc, du_f, dv_f, p.fxb_f, p.inv_fx_f, p.inv_fy_f, px, py, pz);
    } else {
      point_from_disparity_f64(dcd, (double)x - p.u0, (double)(y + p.row0) - p.v0, p, px, py, pz);
    }
    if (valid) {
      normal_from_moments(P1, P2, p.det, dcd, (double)x - p.u0, (double)(y + p.row0) - p.v0, p.fx,
                          p.fy, nx, ny, nz);
    } else {
      nx = ny = nz = __int_as_float(0x7fc00000);
    }
    float* o6 = out6 + idx * 6;
    reinterpret_cast<float2*>(o6)[0] = make_float2(px, py);
    reinterpret_cast<float2*>(o6)[1] = make_float2(pz, nx);
    reinterpret_cast<float2*>(o6)[2] = make_float2(ny, nz);
    if (mask) mask[idx] = valid ? 1 : 0;
  }
}

// thread per pixel, samples straight from global memory (patterns whose
// bounding box does not fit the tiled kernel's shared memory)
template <typename T, bool AFFINE>
__global__ void __launch_bounds__(256)
    fixed_generic_kernel(const T* __restrict__ disp, const FixedParams p,
                         const __grid_constant__ OffsetTable tab, float* __restrict__ out6,
                         uint8_t* __restrict__ mask, double* __restrict__ a1,
                         double* __restrict__ a2) {
  const int n_off = tab.n;
  const int2* soff = tab.v;
  const int64_t total = p.B * p.H * p.W;
  const int64_t W = p.W, H = p.H;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = idx % W;
    const int64_t r = idx / W;
    const int64_t y = r % H;
    const T* frame = disp + (r / H) * H * W;
    const T dc = frame[y * W + x];
    bool ok = finite_t(dc);
    double U = 0.0, V = 0.0;
    for (int i = 0; i < n_off && ok; ++i) {
      const int2 o = soff[i];
      const int64_t xx = x + o.x, yy = y + o.y;
      if (xx < 0 || xx >= W || yy < 0 || yy >= H) {
        ok = false;
        break;
      }
      const T v = frame[yy * W + xx];
      if (!finite_t(v)) {
        ok = false;
        break;
      }
      U = fma((double)o.x, (double)v, U);
      V = fma((double)o.y, (double)v, V);
    }
    generic_out<T, AFFINE>(idx, x, y, dc, ok, U, V, p, out6, mask, a1, a2);
  }
}

// Tiled generic kernel: one 32 x 16 block of a frame per CTA, the block plus
// the pattern's bounding box staged in shared memory as fp64 (coalesced
// loads, each sample read once from global memory), the pattern as (weights,
// linear shared-memory offsets) in shared memory; a thread sums its two
// pixels' supports from shared memory in the pattern's order.  A pixel is
// valid iff its support box lies in the frame and every sample (and the
// centre) is finite: for fp32 samples the fp64 sums carry any non-finite
// sample (NaN, or inf times any weight) and never overflow, so finite sums
// are the test; fp64 samples are tested one by one.
constexpr int kGTW = 32, kGTH = 16;

struct GenericGeom {
  int minx, maxx, miny, maxy;  // pattern extents (validity)
  int bx, by, bw, bh;          // staged box: origin offset (<= 0) and size, pattern + centre
};

// staged box rounded up to whole 16-byte units: the weight pairs follow it
__host__ __device__ inline int generic_box(const GenericGeom& g) {
  return ((kGTW + g.bw) * (kGTH + g.bh) + 1) & ~1;
}
__host__ __device__ inline size_t generic_smem(const GenericGeom& g, int n) {
  return (size_t)generic_box(g) * 8 + (size_t)n * 20;
}

template <typename T, bool AFFINE>
__global__ void __launch_bounds__(256)
    fixed_generic_tiled_kernel(const T* __restrict__ disp, const FixedParams p,
                               const __grid_constant__ OffsetTable tab, const GenericGeom g,
                               float* __restrict__ out6, uint8_t* __restrict__ mask,
                               double* __restrict__ a1, double* __restrict__ a2) {
  extern __shared__ __align__(16) unsigned char gsm[];
  const int SW = kGTW + g.bw, SH = kGTH + g.bh;  // staged box
  double* tile = reinterpret_cast<double*>(gsm);
  double2* wt = reinterpret_cast<double2*>(tile + generic_box(g));
  int* lin = reinterpret_cast<int*>(wt + tab.n);
  const int tid = threadIdx.x;
  const int W = (int)p.W, H = (int)p.H;
  const int tiles_x = (W + kGTW - 1) / kGTW, tiles_y = (H + kGTH - 1) / kGTH;
  const int64_t bt = blockIdx.x;
  const int tx = (int)(bt % tiles_x);
  const int64_t rest = bt / tiles_x;
  const int ty = (int)(rest % tiles_y);
  const int64_t f = rest / tiles_y;
  const int x0 = tx * kGTW, y0 = ty * kGTH;
  const T* frame = disp + f * p.H * p.W;
  for (int i = tid; i < tab.n; i += 256) {
    const int2 o = tab.v[i];
    wt[i] = make_double2((double)o.x, (double)o.y);
    lin[i] = o.y * SW + o.x;
  }
  // the staged box, rows / columns clamped into the frame (samples of
  // out-of-frame positions only ever feed invalid pixels)
  for (int i = tid; i < SW * SH; i += 256) {
    const int r = i / SW, c = i - r * SW;
    const int yy = min(max(y0 + g.by + r, 0), H - 1), xx = min(max(x0 + g.bx + c, 0), W - 1);
    tile[i] = (double)frame[(int64_t)yy * W + xx];
  }
  __syncthreads();
  const int cx = tid & (kGTW - 1);
#pragma unroll 1
  for (int cy = tid / kGTW; cy < kGTH; cy += 256 / kGTW) {
    const int x = x0 + cx, y = y0 + cy;
    if (x >= W || y >= H) continue;
    const double* c = tile + (cy - g.by) * SW + (cx - g.bx);  // the centre sample
    const T dc = (T)c[0];
    bool ok = finite_t(dc) && x + g.minx >= 0 && x + g.maxx < W && y + g.miny >= 0 &&
              y + g.maxy < H;
    double U = 0.0, V = 0.0;
    bool fin = true;
    for (int i = 0; i < tab.n; ++i) {
      const double v = c[lin[i]];
      const double2 w2 = wt[i];
      if constexpr (sizeof(T) == 8) fin &= fabs(v) <= 1.7976931348623157e308;
      U = fma(w2.x, v, U);
      V = fma(w2.y, v, V);
    }
    if constexpr (sizeof(T) == 8) ok = ok && fin;
    else ok = ok && fabs(U) <= 1.7976931348623157e308 && fabs(V) <= 1.7976931348623157e308;
    generic_out<T, AFFINE>(f * p.H * p.W + (int64_t)y * W + x, x, y, dc, ok, U, V, p, out6, mask,
                           a1, a2);
  }
}

// ---------------------------------------------------------------------------
// host-side launchers

template <int R, typename T>
static int launch_square(const LaunchCtx& ctx, const T* disp, const FixedParams& p, float* out6,
                         uint8_t* mask, int64_t in_pitch, int64_t out_pitch) {
  using Cfg = FastCfg<R, T>;
  CUtensorMap in_map;
  const CUtensorMapDataType dt =
      sizeof(T) == 4   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
      : sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                       : CU_TENSOR_MAP_DATA_TYPE_UINT16;
  {
    cuuint64_t dims[3] = {(cuuint64_t)p.W, (cuuint64_t)p.H, (cuuint64_t)p.B};
    cuuint64_t strides[2] = {(cuuint64_t)(in_pitch * sizeof(T)),
                             (cuuint64_t)(in_pitch * p.H * sizeof(T))};
    cuuint32_t box[3] = {(cuuint32_t)Cfg::BW, (cuuint32_t)Cfg::NR, 1};
    cuuint32_t es[3] = {1, 1, 1};
    if (encode_tiled(&in_map, dt, 3, (void*)disp, dims, strides, box, es,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != 0)
      return SN_ECUDA;
  }
  const int tiles_x = (int)((p.W + kTW - 1) / kTW);
  const int tiles_y = (int)((p.H + kG - 1) / kG);
  const int64_t n_items64 = (int64_t)tiles_x * tiles_y * p.B;
  if (n_items64 >= 0x7fffffffLL) return -1;  // generic path handles absurd batches
  const int n_items = (int)n_items64;
  auto kern = fixed_square_kernel<R, T>;
  if (ensure_dyn_smem(reinterpret_cast<const void*>(kern), (int)Cfg::TOTAL, ctx.device,
                      "fixed_square_kernel"))
    return SN_ECUDA;
  const int per_sm =
      occupancy_per_sm(reinterpret_cast<const void*>(kern), kFastThreads, Cfg::TOTAL, ctx.device);
  int64_t grid = (int64_t)per_sm * ctx.num_sms;
  if (grid > n_items) grid = n_items;
  kern<<<(unsigned)grid, kFastThreads, Cfg::TOTAL, ctx.stream>>>(in_map, p, mask, out6, out_pitch,
                                                                 n_items, tiles_x, tiles_y);
  return check_launch("fixed_square_kernel");
}

template <typename T>
static int dispatch_square(int R, const LaunchCtx& ctx, const T* disp, const FixedParams& p,
                           float* out6, uint8_t* mask, int64_t in_pitch = -1,
                           int64_t out_pitch = -1) {
  if (in_pitch < 0) in_pitch = p.W;
  if (out_pitch < 0) out_pitch = p.W;
  switch (R) {
    case 1: return launch_square<1, T>(ctx, disp, p, out6, mask, in_pitch, out_pitch);
    case 2: return launch_square<2, T>(ctx, disp, p, out6, mask, in_pitch, out_pitch);
    case 3: return launch_square<3, T>(ctx, disp, p, out6, mask, in_pitch, out_pitch);
    case 4: return launch_square<4, T>(ctx, disp, p, out6, mask, in_pitch, out_pitch);
    case 5: return launch_square<5, T>(ctx, disp, p, out6, mask, in_pitch, out_pitch);
    case 6: return launch_square<6, T>(ctx, disp, p, out6, mask, in_pitch, out_pitch);
    case 7: return launch_square<7, T>(ctx, disp, p, out6, mask, in_pitch, out_pitch);
    case 8: return launch_square<8, T>(ctx, disp, p, out6, mask, in_pitch, out_pitch);
    default: return -1;
  }
}

// rows of `words` 4-byte words from src (pitch sp words) to dst (pitch dp
// words): one thread per word, a 2D grid of (row chunk, word chunk)
template <typename U>
__global__ void __launch_bounds__(256)
    pitch_copy_kernel(const U* __restrict__ src, int64_t sp, U* __restrict__ dst, int64_t dp,
                      int64_t words, int64_t rows) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= words) return;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) dst[r * dp + w] = __ldcs(src + r * sp + w);
}

// 4-byte words when every width and pitch allows it, else 2-byte ones
static int pitch_copy(const LaunchCtx& ctx, const void* src, int64_t sp_bytes, void* dst,
                      int64_t dp_bytes, int64_t width_bytes, int64_t rows) {
  const int64_t ws = (width_bytes % 4 == 0 && sp_bytes % 4 == 0 && dp_bytes % 4 == 0) ? 4 : 2;
  const int64_t words = width_bytes / ws;
  const unsigned gx = (unsigned)((words + 255) / 256);
  int64_t gy = (int64_t)ctx.num_sms * 16 / std::max<int64_t>(1, (int64_t)gx);
  gy = std::max<int64_t>(1, std::min<int64_t>(gy, std::min<int64_t>(rows, 65535)));
  if (ws == 4)
    pitch_copy_kernel<uint32_t><<<dim3(gx, (unsigned)gy), 256, 0, ctx.stream>>>(
        static_cast<const uint32_t*>(src), sp_bytes / 4, static_cast<uint32_t*>(dst),
        dp_bytes / 4, words, rows);
  else
    pitch_copy_kernel<uint16_t><<<dim3(gx, (unsigned)gy), 256, 0, ctx.stream>>>(
        static_cast<const uint16_t*>(src), sp_bytes / 2, static_cast<uint16_t*>(dst),
        dp_bytes / 2, words, rows);
  return check_launch("pitch_copy_kernel");
}

// The fast kernel on widths (or pointers) TMA cannot address directly: the
// disparities are copied into a row-pitched buffer (pitch rounded up to 16
// bytes; +8 B/px of traffic), and for odd widths the records go through a
// pitched buffer too (+48 B/px).  Stream-ordered allocations from the
// library's private pool (scratch_alloc), so concurrent calls on different
// streams do not share scratch.  Returns -1 to fall back
// to the generic kernel if the scratch cannot be had.
template <typename T>
static int dispatch_square_staged(int R, const LaunchCtx& ctx, const T* disp, const FixedParams& p,
                                  float* out6, uint8_t* mask) {
  constexpr int64_t AE = 16 / (int64_t)sizeof(T);
  const int64_t Wp = (p.W + AE - 1) / AE * AE;  // even (AE >= 2)
  const bool out_direct = p.W % 2 == 0 && reinterpret_cast<uintptr_t>(out6) % 16 == 0;
  T* in_tmp = nullptr;
  float* out_tmp = nullptr;
  const size_t in_bytes = (size_t)(p.B * p.H * Wp) * sizeof(T);
  const size_t out_bytes = out_direct ? 0 : (size_t)(p.B * p.H * Wp) * 24;
  if (scratch_alloc(ctx, in_bytes, reinterpret_cast<void**>(&in_tmp)) != SN_OK) return -1;
  if (!out_direct && scratch_alloc(ctx, out_bytes, reinterpret_cast<void**>(&out_tmp)) != SN_OK) {
    scratch_free(ctx, in_tmp);
    return -1;
  }
  int rc = pitch_copy(ctx, disp, p.W * (int64_t)sizeof(T), in_tmp, Wp * (int64_t)sizeof(T),
                      p.W * (int64_t)sizeof(T), p.B * p.H);
  if (rc == SN_OK)
    rc = dispatch_square<T>(R, ctx, in_tmp, p, out_direct ? out6 : out_tmp, mask, Wp,
                            out_direct ? p.W : Wp);
  if (rc == SN_OK && !out_direct)
    rc = pitch_copy(ctx, out_tmp, Wp * 24, out6, p.W * 24, p.W * 24, p.B * p.H);
  scratch_free(ctx, in_tmp);
  if (out_tmp) scratch_free(ctx, out_tmp);
  return rc;
}

template <typename T>
static int launch_generic(const LaunchCtx& ctx, const T* disp, const FixedParams& p,
                          const OffsetTable& tab, float* out6, uint8_t* mask, double* a1,
                          double* a2, bool affine) {
  const int64_t total = p.B * p.H * p.W;
  if (total == 0) return SN_OK;
  // the tiled kernel when the staged box fits 96 KB of shared memory
  GenericGeom g{0, 0, 0, 0, 0, 0, 0, 0};
  if (tab.n > 0) {  // extents of the pattern itself (validity); the box also holds the centre
    g.minx = g.maxx = tab.v[0].x;
    g.miny = g.maxy = tab.v[0].y;
    for (int i = 1; i < tab.n; ++i) {
      g.minx = std::min(g.minx, tab.v[i].x);
      g.maxx = std::max(g.maxx, tab.v[i].x);
      g.miny = std::min(g.miny, tab.v[i].y);
      g.maxy = std::max(g.maxy, tab.v[i].y);
    }
  }
  g.bx = std::min(g.minx, 0);
  g.by = std::min(g.miny, 0);
  g.bw = std::max(g.maxx, 0) - g.bx;
  g.bh = std::max(g.maxy, 0) - g.by;
  const size_t sm = (g.bw < 4096 && g.bh < 4096) ? generic_smem(g, tab.n) : SIZE_MAX;
  const int64_t tiles = p.B * ((p.H + kGTH - 1) / kGTH) * ((p.W + kGTW - 1) / kGTW);
  if (sm <= 96 * 1024 && tiles < 0x7fffffffLL) {
    auto kern = affine ? fixed_generic_tiled_kernel<T, true> : fixed_generic_tiled_kernel<T, false>;
    if (ensure_dyn_smem(reinterpret_cast<const void*>(kern), 96 * 1024, ctx.device,
                        "fixed_generic_tiled_kernel"))
      return SN_ECUDA;
    kern<<<(unsigned)tiles, 256, sm, ctx.stream>>>(disp, p, tab, g, out6, mask, a1, a2);
    return check_launch("fixed_generic_tiled_kernel");
  }
  int64_t grid = (total + 255) / 256;
  const int64_t cap = (int64_t)ctx.num_sms * 8;
  if (grid > cap) grid = cap;
  if (affine)
    fixed_generic_kernel<T, true><<<(unsigned)grid, 256, 0, ctx.stream>>>(disp, p, tab, out6, mask,
                                                                        a1, a2);
  else
    fixed_generic_kernel<T, false><<<(unsigned)grid, 256, 0, ctx.stream>>>(disp, p, tab, out6, mask,
                                                                         a1, a2);
  return check_launch("fixed_generic_kernel");
}

template <typename T>
int run_fixed(const LaunchCtx& ctx, const T* disp, const FixedParams& p, const sn_moments_t& m,
              const OffsetTable& tab, float* out6, uint8_t* mask, double* a1, double* a2,
              bool affine, int force_generic) {
  if (p.B * p.H * p.W == 0) return SN_OK;
  const bool aligned = (reinterpret_cast<uintptr_t>(disp) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(out6) % 16 == 0) &&
                       (p.W % (16 / (int64_t)sizeof(T)) == 0) && (p.W % 2 == 0) &&
                       p.W <= (int64_t)0x7fffffff / 6 && p.H <= 0x7fffffff && p.B <= 0x7fffffff;
  const bool sized = p.W <= (int64_t)0x7fffffff / 6 && p.H <= 0x7fffffff && p.B <= 0x7fffffff;
  if (!affine && !force_generic && m.square_r >= 1 && m.square_r <= 8 && sized) {
    int rc = aligned ? dispatch_square<T>(m.square_r, ctx, disp, p, out6, mask)
                     : dispatch_square_staged<T>(m.square_r, ctx, disp, p, out6, mask);
    if (rc == SN_OK && p.bits != nullptr) {
      if constexpr (sizeof(T) >= 4) rc = run_passable_bits<T>(ctx, disp, p, p.bits);
    }
    if (rc >= 0) return rc;
  }
  int rc = launch_generic<T>(ctx, disp, p, tab, out6, mask, a1, a2, affine);
  if (rc == SN_OK && !affine && p.bits != nullptr) {
    if constexpr (sizeof(T) >= 4) rc = run_passable_bits<T>(ctx, disp, p, p.bits);
  }
  return rc;
}

// Row-pitched input (ld >= W elements between rows, ld * H between frames):
// the TMA tensor map takes the pitch directly when the rows are 16-byte
// aligned and the pattern is a centred square; otherwise the rows are packed
// into stream-ordered scratch first and the contiguous path runs on it.
template <typename T>
int run_fixed_strided(const LaunchCtx& ctx, const T* disp, int64_t ld, const FixedParams& p,
                      const sn_moments_t& m, const OffsetTable& tab, float* out6, uint8_t* mask) {
  if (p.B * p.H * p.W == 0) return SN_OK;
  if (ld == p.W) return run_fixed<T>(ctx, disp, p, m, tab, out6, mask, nullptr, nullptr, false, 0);
  const bool sized = p.W <= (int64_t)0x7fffffff / 6 && p.H <= 0x7fffffff && p.B <= 0x7fffffff;
  if (m.square_r >= 1 && m.square_r <= 8 && sized && reinterpret_cast<uintptr_t>(disp) % 16 == 0 &&
      (ld * (int64_t)sizeof(T)) % 16 == 0 && reinterpret_cast<uintptr_t>(out6) % 16 == 0 &&
      p.W % 2 == 0) {
    const int rc = dispatch_square<T>(m.square_r, ctx, disp, p, out6, mask, ld, p.W);
    if (rc >= 0) return rc;
  }
  T* packed = nullptr;
  int rc = scratch_alloc(ctx, (size_t)(p.B * p.H * p.W) * sizeof(T), reinterpret_cast<void**>(&packed));
  if (rc) return rc;
  rc = pitch_copy(ctx, disp, ld * (int64_t)sizeof(T), packed, p.W * (int64_t)sizeof(T),
                  p.W * (int64_t)sizeof(T), p.B * p.H);
  if (rc == SN_OK)
    rc = run_fixed<T>(ctx, packed, p, m, tab, out6, mask, nullptr, nullptr, false, 0);
  scratch_free(ctx, packed);
  return rc;
}
template int run_fixed_strided<float>(const LaunchCtx&, const float*, int64_t, const FixedParams&,
                                      const sn_moments_t&, const OffsetTable&, float*, uint8_t*);
template int run_fixed_strided<double>(const LaunchCtx&, const double*, int64_t,
                                       const FixedParams&, const sn_moments_t&, const OffsetTable&,
                                       float*, uint8_t*);

template int run_fixed<float>(const LaunchCtx&, const float*, const FixedParams&,
                              const sn_moments_t&, const OffsetTable&, float*, uint8_t*, double*,
                              double*, bool, int);
// 16-bit PNG input: the fast (square, aligned) kernel only
int run_fixed_png16(const LaunchCtx& ctx, const uint16_t* raw, const FixedParams& p,
                    const sn_moments_t& m, float* out6, uint8_t* mask) {
  if (p.B * p.H * p.W == 0) return SN_OK;
  const bool sized = p.W <= (int64_t)0x7fffffff / 6 && p.H <= 0x7fffffff && p.B <= 0x7fffffff;
  const bool aligned = (reinterpret_cast<uintptr_t>(raw) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(out6) % 16 == 0) && (p.W % 8 == 0);
  if (m.square_r < 1 || m.square_r > 8 || !sized)
    return set_error(SN_EINVAL,
                     "16-bit input needs a centred square kernel (3..17); dequantise with "
                     "sn_dequant_png16 otherwise");
  const Png16* in = reinterpret_cast<const Png16*>(raw);
  const int rc = aligned ? dispatch_square<Png16>(m.square_r, ctx, in, p, out6, mask)
                         : dispatch_square_staged<Png16>(m.square_r, ctx, in, p, out6, mask);
  return rc >= 0 ? rc : set_error(SN_EINVAL, "batch too large or scratch unavailable");
}

template int run_fixed<double>(const LaunchCtx&, const double*, const FixedParams&,
                               const sn_moments_t&, const OffsetTable&, float*, uint8_t*, double*,
                               double*, bool, int);

}  // namespace sn
