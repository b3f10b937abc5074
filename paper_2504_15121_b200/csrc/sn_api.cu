// C ABI (include/sn_b200.h): argument validation, kernel-pattern moments,
// rig pre-combination, dispatch, the host-buffer pipeline and the strip
// seam merge.

#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <numeric>
#include <map>
#include <set>
#include <tuple>
#include <thread>
#include <unordered_map>
#include <vector>

#include "sn_b200.h"
#include "sn_internal.h"

namespace sn {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int set_cuda_error(const char* what) {
  const cudaError_t e = cudaGetLastError();
  return set_error(SN_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(SN_ECUDA, "%s launch: %s", what, cudaGetErrorString(e));
  return SN_OK;
}

int ensure_dyn_smem(const void* func, int bytes, int device, const char* name) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;  // (kernel, device) pairs
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({func, device})) return SN_OK;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return set_error(SN_ECUDA, "cudaFuncSetAttribute(%s): %s", name,
                     cudaGetErrorString(cudaGetLastError()));
  done.insert({func, device});
  return SN_OK;
}

int occupancy_per_sm(const void* func, int threads, size_t smem, int device) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t, int>, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(func, threads, smem, device);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 1;
  }
  if (per_sm < 1) per_sm = 1;
  cache.emplace(key, per_sm);
  return per_sm;
}

// A private stream-ordered pool per device: its release threshold keeps the
// memory between calls without touching the device's default pool (which
// other cudaMallocAsync users in the process own).
static cudaMemPool_t scratch_pool(int device) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  if (device < 0 || device >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[device]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[device] = pool;
  }
  return pools[device];
}

int scratch_alloc(const LaunchCtx& ctx, size_t bytes, void** ptr) {
  *ptr = nullptr;
  cudaMemPool_t pool = scratch_pool(ctx.device);
  if (!pool) return set_error(SN_ECUDA, "cannot create the scratch memory pool");
  if (cudaMallocFromPoolAsync(ptr, bytes ? bytes : 1, pool, ctx.stream) != cudaSuccess) {
    *ptr = nullptr;
    return set_cuda_error("cudaMallocFromPoolAsync(scratch)");
  }
  return SN_OK;
}

void scratch_free(const LaunchCtx& ctx, void* ptr) {
  if (ptr) cudaFreeAsync(ptr, ctx.stream);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

int encode_tiled(CUtensorMap* map, CUtensorMapDataType dt, int rank, void* gaddr,
                 const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                 const cuuint32_t* elem_strides, CUtensorMapSwizzle swizzle,
                 CUtensorMapFloatOOBfill oob) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return set_error(SN_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
  const CUresult r = fn(map, dt, (cuuint32_t)rank, gaddr, dims, strides, box, elem_strides,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        oob);
  if (r != CUDA_SUCCESS) return set_error(SN_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SN_OK;
}

}  // namespace sn

using namespace sn;

// ---------------------------------------------------------------------------
// plan

struct sn_plan {
  int device;
  int num_sms;
  // host-path workspace (sn_*_host): three streams, double-buffered device
  // staging, and pinned host staging used when the caller's buffers are
  // pageable.  Guarded by mu: host-path calls on one plan run one at a time.
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr},
              ev_out[2] = {nullptr, nullptr};
  void* d_in[2] = {nullptr, nullptr};  // input chunk (fp32 or fp64)
  float* d_out[2] = {nullptr, nullptr};
  uint8_t* d_mask[2] = {nullptr, nullptr};
  int32_t* d_lab[2] = {nullptr, nullptr};
  void* d_ws[2] = {nullptr, nullptr};
  size_t cap_in = 0, cap_px = 0, ws_cap = 0;
  void* h_in[2] = {nullptr, nullptr};  // pinned staging (pageable callers only)
  void* h_out[2] = {nullptr, nullptr};
  size_t h_in_cap = 0, h_out_cap = 0;
  std::mutex mu;
  // second stream for the labeller's half batches (ccl_labels_ws_impl);
  // its own lock, held while the halves are enqueued
  cudaStream_t s_aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  std::mutex aux_mu;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int check_shape(int64_t B, int64_t H, int64_t W) {
  if (B < 0 || H < 0 || W < 0) return set_error(SN_EINVAL, "negative shape (%lld, %lld, %lld)",
                                               (long long)B, (long long)H, (long long)W);
  if (H > 0x7fffffffLL || W > 0x7fffffffLL || B > 0x7fffffffLL)
    return set_error(SN_EINVAL, "dimension exceeds int32 range");
  return SN_OK;
}

int check_rig(const sn_rig_t* rig) {
  if (!rig) return set_error(SN_EINVAL, "rig is NULL");
  // geometry.py:32-36
  if (!(rig->fx > 0.0 && rig->fy > 0.0)) return set_error(SN_EINVAL, "focal lengths must be positive");
  if (!(rig->baseline > 0.0)) return set_error(SN_EINVAL, "baseline must be positive");
  if (!isfinite(rig->u0) || !isfinite(rig->v0) || !isfinite(rig->fx) || !isfinite(rig->fy) ||
      !isfinite(rig->baseline))
    return set_error(SN_EINVAL, "rig parameters must be finite");
  return SN_OK;
}

void fill_rig(FixedParams& p, const sn_rig_t* rig) {
  p.fx = rig->fx;
  p.fy = rig->fy;
  p.u0 = rig->u0;
  p.v0 = rig->v0;
  p.fxb = rig->fx * rig->baseline;  // geometry.py:43 evaluates fx * b first
  p.fxb_f = (float)p.fxb;
  p.inv_fx_f = (float)(1.0 / rig->fx);
  p.nfx_f = -(float)rig->fx;
  p.nfy_f = -(float)rig->fy;
  p.inv_fy_f = (float)(1.0 / rig->fy);
  p.u0_hi = (float)rig->u0;
  p.u0_lo = (float)(rig->u0 - (double)p.u0_hi);
  p.v0_hi = (float)rig->v0;
  p.v0_lo = (float)(rig->v0 - (double)p.v0_hi);
}

}  // namespace

void sn::fill_predicate(FixedParams& p, double fxb, double t, uint32_t* bits) {
  p.bits = bits;
  p.bits_ww = (int)((p.W + 31) / 32);
  p.t = t;
  p.t_f = (float)t;
  p.fxb_pf = (float)fxb;
  // the filter's ranges (sn_common.cuh pred_bit): K and t in [2^-40, 2^40]
  const double lo = 9.094947017729282e-13, hi = 1099511627776.0;
  p.pred_exact = !(fxb >= lo && fxb <= hi && t >= lo && t <= hi);
}

namespace {

int prepare(const int32_t* offsets_xy, int32_t n_off, sn_moments_t& m, OffsetTable& tab) {
  int rc = sn_kernel_moments(offsets_xy, n_off, &m);
  if (rc) return rc;
  if (n_off > kMaxOffsets)
    return set_error(SN_EINVAL, "at most %d offsets are supported (got %d)", kMaxOffsets, n_off);
  tab.n = n_off;
  for (int i = 0; i < n_off; ++i) tab.v[i] = make_int2(offsets_xy[2 * i], offsets_xy[2 * i + 1]);
  return SN_OK;
}

void fill_moments(FixedParams& p, const sn_moments_t& m) {
  p.alpha = (double)m.alpha;
  p.nal_f = -(float)p.alpha;
  p.beta = (double)m.beta;
  p.gamma = (double)m.gamma;
  p.det = (double)m.det;
  p.sx = (double)m.sx;
  p.sy = (double)m.sy;
  p.R = m.square_r;
}

LaunchCtx make_ctx(sn_plan_t* plan, void* stream) {
  LaunchCtx c;
  c.stream = reinterpret_cast<cudaStream_t>(stream);
  c.device = plan->device;
  c.num_sms = plan->num_sms;
  return c;
}

template <typename T>
int oriented_points_impl(sn_plan_t* plan, const T* disp, int64_t B, int64_t H, int64_t W,
                         const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off,
                         float* out6, uint8_t* mask, void* stream, int force_generic,
                         int64_t row0 = 0, uint32_t* bits = nullptr, double t = 0.0) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  if (row0 < 0 || row0 + H > 0x7fffffffLL) return set_error(SN_EINVAL, "row offset out of range");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if ((rc = check_rig(rig))) return rc;
  sn_moments_t m;
  static thread_local OffsetTable tab;
  if ((rc = prepare(offsets_xy, n_off, m, tab))) return rc;
  if (B * H * W > 0 && (!disp || !out6)) return set_error(SN_EINVAL, "NULL buffer");
  FixedParams p{};
  p.B = B;
  p.H = H;
  p.W = W;
  fill_rig(p, rig);
  fill_moments(p, m);
  p.row0 = (int)row0;
  if (bits) {
    if (!(t > 0.0)) return set_error(SN_EINVAL, "threshold must be positive");
    fill_predicate(p, p.fxb, t, bits);
  }
  DeviceGuard g(plan->device);
  return run_fixed<T>(make_ctx(plan, stream), disp, p, m, tab, out6, mask, nullptr, nullptr, false,
                      force_generic);
}

template <typename T>
int affine_impl(sn_plan_t* plan, const T* disp, int64_t B, int64_t H, int64_t W,
                const int32_t* offsets_xy, int32_t n_off, double* a1, double* a2, uint8_t* mask,
                void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  sn_moments_t m;
  static thread_local OffsetTable tab;
  if ((rc = prepare(offsets_xy, n_off, m, tab))) return rc;
  if (B * H * W > 0 && (!disp || !a1 || !a2)) return set_error(SN_EINVAL, "NULL buffer");
  FixedParams p{};
  p.B = B;
  p.H = H;
  p.W = W;
  fill_moments(p, m);
  DeviceGuard g(plan->device);
  return run_fixed<T>(make_ctx(plan, stream), disp, p, m, tab, nullptr, mask, a1, a2, true, 1);
}

}  // namespace

extern "C" {

int sn_abi_version(void) { return SN_ABI_VERSION; }

const char* sn_last_error(void) { return g_err; }

int sn_plan_create(int device, sn_plan_t** plan) {
  if (!plan) return set_error(SN_EINVAL, "plan out-pointer is NULL");
  *plan = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    return set_error(SN_ECUDA, "no CUDA device available");
  if (device < 0 || device >= n) return set_error(SN_EINVAL, "device %d out of range [0, %d)", device, n);
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (major != 10)
    return set_error(SN_ECUDA, "device %d has compute capability %d.x; this build targets sm_100a",
                     device, major);
  sn_plan* p = new sn_plan();
  p->device = device;
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device);
  *plan = p;
  return SN_OK;
}

int sn_plan_destroy(sn_plan_t* plan) {
  if (!plan) return SN_OK;
  {
    DeviceGuard g(plan->device);
    for (int i = 0; i < 2; ++i) {
      if (plan->h_in[i]) cudaFreeHost(plan->h_in[i]);
      if (plan->h_out[i]) cudaFreeHost(plan->h_out[i]);
      if (plan->d_in[i]) cudaFree(plan->d_in[i]);
      if (plan->d_out[i]) cudaFree(plan->d_out[i]);
      if (plan->d_mask[i]) cudaFree(plan->d_mask[i]);
      if (plan->d_lab[i]) cudaFree(plan->d_lab[i]);
      if (plan->d_ws[i]) cudaFree(plan->d_ws[i]);
      if (plan->ev_in[i]) cudaEventDestroy(plan->ev_in[i]);
      if (plan->ev_done[i]) cudaEventDestroy(plan->ev_done[i]);
      if (plan->ev_out[i]) cudaEventDestroy(plan->ev_out[i]);
    }
    if (plan->s_h2d) cudaStreamDestroy(plan->s_h2d);
    if (plan->s_comp) cudaStreamDestroy(plan->s_comp);
    if (plan->s_d2h) cudaStreamDestroy(plan->s_d2h);
    if (plan->s_aux) cudaStreamDestroy(plan->s_aux);
    if (plan->ev_fork) cudaEventDestroy(plan->ev_fork);
    if (plan->ev_join) cudaEventDestroy(plan->ev_join);
  }
  delete plan;
  return SN_OK;
}

int sn_kernel_moments(const int32_t* offsets_xy, int32_t n_off, sn_moments_t* out) {
  if (!out) return set_error(SN_EINVAL, "moments out-pointer is NULL");
  // kernels.py:38-43
  if (!offsets_xy || n_off <= 0) return set_error(SN_EINVAL, "offsets must have shape (N, 2)");
  std::vector<int64_t> keys(n_off);
  for (int i = 0; i < n_off; ++i)
    keys[i] = ((int64_t)offsets_xy[2 * i] << 32) ^ (uint32_t)offsets_xy[2 * i + 1];
  std::sort(keys.begin(), keys.end());
  if (std::adjacent_find(keys.begin(), keys.end()) != keys.end())
    return set_error(SN_EINVAL, "offsets must be distinct");
  sn_moments_t m{};
  int32_t minx = 0, maxx = 0, miny = 0, maxy = 0;
  for (int i = 0; i < n_off; ++i) {
    const int64_t vx = offsets_xy[2 * i], vy = offsets_xy[2 * i + 1];
    m.alpha += vx * vx;
    m.beta += vx * vy;
    m.gamma += vy * vy;
    m.sx += vx;
    m.sy += vy;
    minx = std::min<int32_t>(minx, (int32_t)vx);
    maxx = std::max<int32_t>(maxx, (int32_t)vx);
    miny = std::min<int32_t>(miny, (int32_t)vy);
    maxy = std::max<int32_t>(maxy, (int32_t)vy);
  }
  m.det = m.alpha * m.gamma - m.beta * m.beta;
  m.hx = std::max(maxx, -minx);
  m.hy = std::max(maxy, -miny);
  // centred (2R+1)^2 square?
  m.square_r = -1;
  if (minx == -maxx && miny == -maxy && maxx == maxy) {
    const int64_t side = 2 * (int64_t)maxx + 1;
    if (side * side == n_off) m.square_r = maxx;  // distinct + inside the box => full square
  }
  *out = m;
  // kernels.py:91-93: det is an exact integer, so det <= 0.5 <=> det <= 0
  if (m.det <= 0) return set_error(SN_EDEGENERATE, "offset pattern is rank deficient (det=%lld)",
                                   (long long)m.det);
  return SN_OK;
}

int sn_oriented_points(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                       const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off, float* out6,
                       uint8_t* mask, void* stream) {
  return oriented_points_impl<float>(plan, disp, B, H, W, rig, offsets_xy, n_off, out6, mask,
                                     stream, 0);
}

}  // extern "C"

namespace {

template <typename T>
int strided_impl(sn_plan_t* plan, const T* disp, int64_t B, int64_t H, int64_t W, int64_t ld,
                 const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off, float* out6,
                 uint8_t* mask, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (ld < W) return set_error(SN_EINVAL, "row pitch ld=%lld is smaller than W=%lld",
                               (long long)ld, (long long)W);
  if ((rc = check_rig(rig))) return rc;
  sn_moments_t m;
  static thread_local OffsetTable tab;
  if ((rc = prepare(offsets_xy, n_off, m, tab))) return rc;
  if (B * H * W > 0 && (!disp || !out6)) return set_error(SN_EINVAL, "NULL buffer");
  FixedParams p{};
  p.B = B;
  p.H = H;
  p.W = W;
  fill_rig(p, rig);
  fill_moments(p, m);
  DeviceGuard g(plan->device);
  return run_fixed_strided<T>(make_ctx(plan, stream), disp, ld, p, m, tab, out6, mask);
}

}  // namespace

extern "C" {

int sn_oriented_points_strided(sn_plan_t* plan, const float* disp, int64_t B, int64_t H,
                               int64_t W, int64_t ld, const sn_rig_t* rig,
                               const int32_t* offsets_xy, int32_t n_off, float* out6,
                               uint8_t* mask, void* stream) {
  return strided_impl<float>(plan, disp, B, H, W, ld, rig, offsets_xy, n_off, out6, mask, stream);
}

int sn_oriented_points_strided_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H,
                                   int64_t W, int64_t ld, const sn_rig_t* rig,
                                   const int32_t* offsets_xy, int32_t n_off, float* out6,
                                   uint8_t* mask, void* stream) {
  return strided_impl<double>(plan, disp, B, H, W, ld, rig, offsets_xy, n_off, out6, mask, stream);
}

int sn_oriented_points_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H, int64_t W,
                           const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off,
                           float* out6, uint8_t* mask, void* stream) {
  return oriented_points_impl<double>(plan, disp, B, H, W, rig, offsets_xy, n_off, out6, mask,
                                      stream, 0);
}

int sn_oriented_points_rows(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                            int64_t row0, const sn_rig_t* rig, const int32_t* offsets_xy,
                            int32_t n_off, float* out6, uint8_t* mask, void* stream) {
  return oriented_points_impl<float>(plan, disp, B, H, W, rig, offsets_xy, n_off, out6, mask,
                                     stream, 0, row0);
}

int sn_oriented_points_bits(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                            int64_t row0, const sn_rig_t* rig, const int32_t* offsets_xy,
                            int32_t n_off, double t, float* out6, uint8_t* mask, uint32_t* bits,
                            void* stream) {
  if (B * H * W > 0 && !bits) return set_error(SN_EINVAL, "NULL bit-mask buffer");
  return oriented_points_impl<float>(plan, disp, B, H, W, rig, offsets_xy, n_off, out6, mask,
                                     stream, 0, row0, bits, t);
}

int sn_oriented_points_bits_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H,
                                int64_t W, int64_t row0, const sn_rig_t* rig,
                                const int32_t* offsets_xy, int32_t n_off, double t, float* out6,
                                uint8_t* mask, uint32_t* bits, void* stream) {
  if (B * H * W > 0 && !bits) return set_error(SN_EINVAL, "NULL bit-mask buffer");
  return oriented_points_impl<double>(plan, disp, B, H, W, rig, offsets_xy, n_off, out6, mask,
                                      stream, 0, row0, bits, t);
}

int sn_oriented_points_rows_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H,
                                int64_t W, int64_t row0, const sn_rig_t* rig,
                                const int32_t* offsets_xy, int32_t n_off, float* out6,
                                uint8_t* mask, void* stream) {
  return oriented_points_impl<double>(plan, disp, B, H, W, rig, offsets_xy, n_off, out6, mask,
                                      stream, 0, row0);
}

}  // extern "C"

namespace {

template <typename T>
int passable_bits_impl(sn_plan_t* plan, const T* disp, int64_t B, int64_t H, int64_t W,
                       const sn_rig_t* rig, double t, uint32_t* bits, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if ((rc = check_rig(rig))) return rc;
  if (!(t > 0.0)) return set_error(SN_EINVAL, "threshold must be positive");
  if (B * H * W == 0) return SN_OK;
  if (!disp || !bits) return set_error(SN_EINVAL, "NULL buffer");
  FixedParams p{};
  p.B = B;
  p.H = H;
  p.W = W;
  fill_rig(p, rig);
  fill_predicate(p, p.fxb, t, bits);
  DeviceGuard g(plan->device);
  return run_passable_bits<T>(make_ctx(plan, stream), disp, p, bits);
}

}  // namespace

extern "C" {

int sn_passable_bits(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                     const sn_rig_t* rig, double t, uint32_t* bits, void* stream) {
  return passable_bits_impl<float>(plan, disp, B, H, W, rig, t, bits, stream);
}

int sn_passable_bits_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H, int64_t W,
                         const sn_rig_t* rig, double t, uint32_t* bits, void* stream) {
  return passable_bits_impl<double>(plan, disp, B, H, W, rig, t, bits, stream);
}

static int check_png16(double scale, int32_t invalid) {
  // nonzero values (raw - 1) / scale, |raw - 1| <= 65535, stay normal fp32
  const double a = fabs(scale);
  if (!(a >= 7.888609052210118e-31 && a <= 1.2676506002282294e30))  // 2^-100 .. 2^100
    return set_error(SN_EINVAL, "PNG16 scale must be finite with 2^-100 <= |scale| <= 2^100");
  if (invalid < -1 || invalid > 0xFFFF)
    return set_error(SN_EINVAL, "invalid_value must be a 16-bit sample or -1 (none)");
  return SN_OK;
}

int sn_oriented_points_png16(sn_plan_t* plan, const uint16_t* raw, int64_t B, int64_t H,
                             int64_t W, double scale, int32_t invalid, const sn_rig_t* rig,
                             const int32_t* offsets_xy, int32_t n_off, float* out6,
                             uint8_t* mask, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if ((rc = check_rig(rig))) return rc;
  if ((rc = check_png16(scale, invalid))) return rc;
  sn_moments_t m;
  static thread_local OffsetTable tab;
  if ((rc = prepare(offsets_xy, n_off, m, tab))) return rc;
  if (B * H * W > 0 && (!raw || !out6)) return set_error(SN_EINVAL, "NULL buffer");
  FixedParams p{};
  p.B = B;
  p.H = H;
  p.W = W;
  fill_rig(p, rig);
  fill_moments(p, m);
  p.png_scale = scale;
  p.png_rcp = png16_rcp(scale);
  p.png_rcp_f = (float)(1.0 / scale);
  p.png_sign = scale > 0 ? 1 : -1;
  p.png_invalid = invalid;
  DeviceGuard g(plan->device);
  return run_fixed_png16(make_ctx(plan, stream), raw, p, m, out6, mask);
}

int sn_dequant_png16(sn_plan_t* plan, const uint16_t* raw, int64_t B, int64_t H, int64_t W,
                     double scale, int32_t invalid, float* out_f32, double* out_f64,
                     void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (!(scale == scale) || scale == 0.0 || fabs(scale) > 1.7976931348623157e308)
    return set_error(SN_EINVAL, "PNG16 scale must be finite and nonzero");
  if (invalid < -1 || invalid > 0xFFFF)
    return set_error(SN_EINVAL, "invalid_value must be a 16-bit sample or -1 (none)");
  if (B * H * W > 0 && (!raw || (!out_f32 && !out_f64)))
    return set_error(SN_EINVAL, "NULL buffer");
  DeviceGuard g(plan->device);
  return run_dequant_png16(make_ctx(plan, stream), raw, B * H * W, invalid, scale, out_f32,
                           out_f64);
}

int sn_decode_pfm(sn_plan_t* plan, const void* payload, int64_t B, int64_t H, int64_t W,
                  int32_t channels, int32_t big_endian, float* out, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (channels != 1 && channels != 3) return set_error(SN_EINVAL, "PFM has 1 or 3 channels");
  if (B * H * W > 0 && (!payload || !out)) return set_error(SN_EINVAL, "NULL buffer");
  if (reinterpret_cast<uintptr_t>(payload) % 4 || reinterpret_cast<uintptr_t>(out) % 4)
    return set_error(SN_EINVAL, "PFM buffers must be 4-byte aligned");
  DeviceGuard g(plan->device);
  return run_decode_pfm(make_ctx(plan, stream), payload, B, H, W * channels, big_endian != 0,
                        out);
}

int sn_cloud_workspace_bytes(int64_t B, int64_t H, int64_t W, size_t* bytes) {
  if (!bytes) return set_error(SN_EINVAL, "bytes out-pointer is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  *bytes = cloud_workspace_bytes(B, H, W);
  return SN_OK;
}

int sn_compact_cloud(sn_plan_t* plan, const float* out6, const uint8_t* mask, int64_t B,
                     int64_t H, int64_t W, float* cloud, int64_t capacity, int64_t* frame_offsets,
                     void* workspace, size_t ws_bytes, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (capacity < 0) return set_error(SN_EINVAL, "negative capacity");
  if (!frame_offsets || (B * H * W > 0 && (!out6 || !mask || (capacity > 0 && !cloud))))
    return set_error(SN_EINVAL, "NULL buffer");
  DeviceGuard g(plan->device);
  return run_compact_cloud(make_ctx(plan, stream), out6, mask, B, H, W, cloud, capacity,
                           frame_offsets, workspace, ws_bytes);
}

int sn_cloud_count(sn_plan_t* plan, const uint8_t* mask, int64_t B, int64_t H, int64_t W,
                   int64_t* frame_offsets, void* workspace, size_t ws_bytes, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (!frame_offsets || (B * H * W > 0 && !mask)) return set_error(SN_EINVAL, "NULL buffer");
  DeviceGuard g(plan->device);
  return run_cloud_count(make_ctx(plan, stream), mask, B, H, W, frame_offsets, workspace,
                         ws_bytes);
}

int sn_cloud_scatter(sn_plan_t* plan, const float* out6, const uint8_t* mask, int64_t B,
                     int64_t H, int64_t W, float* cloud, int64_t capacity, void* workspace,
                     size_t ws_bytes, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (capacity < 0) return set_error(SN_EINVAL, "negative capacity");
  if (B * H * W > 0 && capacity > 0 && (!out6 || !mask || !cloud))
    return set_error(SN_EINVAL, "NULL buffer");
  DeviceGuard g(plan->device);
  return run_cloud_scatter(make_ctx(plan, stream), out6, mask, B, H, W, cloud, capacity, workspace,
                           ws_bytes);
}

int sn_adaptive_workspace_bytes(int64_t B, int64_t H, int64_t W, size_t* bytes) {
  if (!bytes) return set_error(SN_EINVAL, "bytes out-pointer is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  *bytes = adaptive_workspace_bytes(B, H, W);
  return SN_OK;
}

}  // extern "C"

namespace {

template <typename T>
int adaptive_impl(sn_plan_t* plan, const T* disp, int64_t B, int64_t H, int64_t W,
                  const sn_rig_t* rig, int32_t n_rays, const int32_t* ray_len,
                  const int32_t* ray_xy, int32_t stop, int32_t shared_range, double threshold,
                  float* out6, uint8_t* mask, void* workspace, size_t ws_bytes, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if ((rc = check_rig(rig))) return rc;
  // adaptive.py:49-57
  if (stop != 0 && stop != 1) return set_error(SN_EINVAL, "stop must be 0 (st) or 1 (cd)");
  if (!(threshold > 0.0)) return set_error(SN_EINVAL, "threshold must be positive");
  if (n_rays < 3) return set_error(SN_EINVAL, "need at least 3 ray directions");
  if (n_rays > kStarMaxRays) return set_error(SN_EINVAL, "at most %d directions", kStarMaxRays);
  if (!ray_len || !ray_xy) return set_error(SN_EINVAL, "NULL ray table");
  static thread_local StarTable tab;
  tab.n_rays = n_rays;
  tab.n_keys = 0;
  int steps = 0;
  std::unordered_map<int64_t, int> key_of;
  for (int j = 0; j < n_rays; ++j) {
    tab.ray_start[j] = steps;
    if (ray_len[j] < 0) return set_error(SN_EINVAL, "negative ray length");
    for (int i = 0; i < ray_len[j]; ++i, ++steps) {
      if (steps >= kStarMaxSteps) return set_error(SN_EINVAL, "at most %d ray steps", kStarMaxSteps);
      const int vx = ray_xy[2 * steps], vy = ray_xy[2 * steps + 1];
      if (vx < -32767 || vx > 32767 || vy < -32767 || vy > 32767)
        return set_error(SN_EINVAL, "ray offset out of range");
      const int64_t kk = ((int64_t)vx << 32) ^ (uint32_t)vy;
      auto it = key_of.find(kk);
      int k;
      if (it == key_of.end()) {
        if (tab.n_keys >= kStarMaxKeys)
          return set_error(SN_EINVAL, "at most %d distinct ray offsets", kStarMaxKeys);
        k = tab.n_keys++;
        key_of.emplace(kk, k);
        tab.key_xy[k] = (int32_t)(((uint32_t)(uint16_t)vx) | ((uint32_t)(uint16_t)vy << 16));
        tab.key_lin[k] = (int32_t)((int64_t)vy * W + vx);
      } else {
        k = it->second;
      }
      tab.step_key[steps] = (int16_t)k;
      tab.step_xy[steps] = tab.key_xy[k];
      tab.step_lin[steps] = tab.key_lin[k];
    }
  }
  tab.ray_start[n_rays] = steps;
  // y * W + x must fit int32 for every offset; moment sums (sum of x^2 etc.
  // over all keys) pick 32- or 64-bit accumulation
  {
    int64_t sxx = 0, sxy = 0, syy = 0;
    tab.reach = 0;
    for (int k = 0; k < tab.n_keys; ++k) {
      const int64_t vx = (int16_t)(tab.key_xy[k] & 0xffff), vy = (int16_t)(tab.key_xy[k] >> 16);
      tab.reach = (int)std::max<int64_t>(tab.reach, std::max(std::llabs(vx), std::llabs(vy)));
      if (std::llabs(vy) * W + std::llabs(vx) > 0x7fffffffLL)
        return set_error(SN_EINVAL, "ray offsets too large for the frame width");
      sxx += vx * vx;
      sxy += std::llabs(vx * vy);
      syy += vy * vy;
    }
    tab.wide = (sxx > 0x7fffffffLL || sxy > 0x7fffffffLL || syy > 0x7fffffffLL) ? 1 : 0;
  }
  if (B * H * W == 0) return SN_OK;
  if (!disp || !out6) return set_error(SN_EINVAL, "NULL buffer");
  AdaptiveParams ap{};
  ap.fp.B = B;
  ap.fp.H = H;
  ap.fp.W = W;
  fill_rig(ap.fp, rig);
  ap.threshold = threshold;
  ap.baseline = rig->baseline;
  ap.fxfx = rig->fx * rig->fx;
  ap.nfxfy = -rig->fx * rig->fy;
  ap.shared_range = shared_range != 0;
  DeviceGuard g(plan->device);
  return run_adaptive<T>(make_ctx(plan, stream), disp, ap, tab, stop, out6, mask, workspace,
                         ws_bytes);
}

}  // namespace

extern "C" {

int sn_adaptive_points(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                       const sn_rig_t* rig, int32_t n_rays, const int32_t* ray_len,
                       const int32_t* ray_xy, int32_t stop, int32_t shared_range,
                       double threshold, float* out6, uint8_t* mask, void* workspace,
                       size_t ws_bytes, void* stream) {
  return adaptive_impl<float>(plan, disp, B, H, W, rig, n_rays, ray_len, ray_xy, stop,
                              shared_range, threshold, out6, mask, workspace, ws_bytes, stream);
}

int sn_adaptive_points_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H, int64_t W,
                           const sn_rig_t* rig, int32_t n_rays, const int32_t* ray_len,
                           const int32_t* ray_xy, int32_t stop, int32_t shared_range,
                           double threshold, float* out6, uint8_t* mask, void* workspace,
                           size_t ws_bytes, void* stream) {
  return adaptive_impl<double>(plan, disp, B, H, W, rig, n_rays, ray_len, ray_xy, stop,
                               shared_range, threshold, out6, mask, workspace, ws_bytes, stream);
}

int sn_eval_workspace_bytes(int64_t B, int64_t H, int64_t W, size_t* bytes) {
  if (!bytes) return set_error(SN_EINVAL, "bytes out-pointer is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  *bytes = eval_workspace_bytes(B, H, W);
  return SN_OK;
}

int sn_angular_error(sn_plan_t* plan, const float* est, int32_t est_stride, const double* gt,
                     const uint8_t* gt_mask, const uint8_t* extra_mask, int64_t B, int64_t H,
                     int64_t W, double* err_out, double* stats, void* workspace, size_t ws_bytes,
                     void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (est_stride < 3) return set_error(SN_EINVAL, "est_stride must be >= 3");
  if (H * W == 0) return set_error(SN_EINVAL, "cannot summarize an empty error map");
  if (B > 0 && (!est || !gt || !gt_mask || !stats)) return set_error(SN_EINVAL, "NULL buffer");
  DeviceGuard g(plan->device);
  return run_eval(make_ctx(plan, stream), est, nullptr, est_stride, gt, gt_mask, extra_mask, B, H,
                  W, err_out, stats, workspace, ws_bytes);
}

int sn_error_stats(sn_plan_t* plan, const double* values, int64_t B, int64_t H, int64_t W,
                   double* stats, void* workspace, size_t ws_bytes, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (H * W == 0) return set_error(SN_EINVAL, "cannot summarize an empty error map");
  if (B > 0 && (!values || !stats)) return set_error(SN_EINVAL, "NULL buffer");
  DeviceGuard g(plan->device);
  return run_eval(make_ctx(plan, stream), nullptr, nullptr, 3, nullptr, nullptr, nullptr, B, H, W,
                  const_cast<double*>(values), stats, workspace, ws_bytes);
}

int sn_angular_error_f64(sn_plan_t* plan, const double* est, int32_t est_stride, const double* gt,
                         const uint8_t* gt_mask, const uint8_t* extra_mask, int64_t B, int64_t H,
                         int64_t W, double* err_out, double* stats, void* workspace,
                         size_t ws_bytes, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (est_stride < 3) return set_error(SN_EINVAL, "est_stride must be >= 3");
  if (H * W == 0) return set_error(SN_EINVAL, "cannot summarize an empty error map");
  if (B > 0 && (!est || !gt || !gt_mask || !stats)) return set_error(SN_EINVAL, "NULL buffer");
  DeviceGuard g(plan->device);
  return run_eval(make_ctx(plan, stream), nullptr, est, est_stride, gt, gt_mask, extra_mask, B, H,
                  W, err_out, stats, workspace, ws_bytes);
}

/* test hook: force the generic (non-TMA) kernel, to cross-check the fast path */
int sn_oriented_points_generic(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                               const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off,
                               float* out6, uint8_t* mask, void* stream) {
  return oriented_points_impl<float>(plan, disp, B, H, W, rig, offsets_xy, n_off, out6, mask,
                                     stream, 1);
}

int sn_affine(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
              const int32_t* offsets_xy, int32_t n_off, double* a1, double* a2, uint8_t* mask,
              void* stream) {
  return affine_impl<float>(plan, disp, B, H, W, offsets_xy, n_off, a1, a2, mask, stream);
}

int sn_affine_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H, int64_t W,
                  const int32_t* offsets_xy, int32_t n_off, double* a1, double* a2, uint8_t* mask,
                  void* stream) {
  return affine_impl<double>(plan, disp, B, H, W, offsets_xy, n_off, a1, a2, mask, stream);
}

}  // extern "C"

namespace {

template <typename T>
int passable_impl(sn_plan_t* plan, const T* disp, int64_t B, int64_t H, int64_t W,
                  const sn_rig_t* rig, double t, uint8_t* passable, double* edges, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if ((rc = check_rig(rig))) return rc;
  if (!(t > 0.0)) return set_error(SN_EINVAL, "threshold must be positive");  // adaptive.py:56-57
  if (B * H * W > 0 && !disp) return set_error(SN_EINVAL, "NULL buffer");
  const CclParams p = make_ccl_params(B, H, W, rig->fx * rig->baseline, t);
  DeviceGuard g(plan->device);
  return run_passable<T>(make_ctx(plan, stream), disp, p, passable, edges);
}

}  // namespace

extern "C" {

int sn_passable(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                const sn_rig_t* rig, double t, uint8_t* passable, double* edges, void* stream) {
  return passable_impl<float>(plan, disp, B, H, W, rig, t, passable, edges, stream);
}

int sn_passable_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H, int64_t W,
                    const sn_rig_t* rig, double t, uint8_t* passable, double* edges,
                    void* stream) {
  return passable_impl<double>(plan, disp, B, H, W, rig, t, passable, edges, stream);
}

int sn_ccl_workspace_bytes(int64_t B, int64_t H, int64_t W, size_t* bytes) {
  if (!bytes) return set_error(SN_EINVAL, "bytes out-pointer is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  *bytes = ccl_workspace_bytes(B, H, W);
  return SN_OK;
}

}  // extern "C"

namespace {

int ccl_args(sn_plan_t* plan, int64_t B, int64_t H, int64_t W, int64_t row_base,
             const void* input, const int32_t* labels) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (B * H * W > 0 && (!input || !labels)) return set_error(SN_EINVAL, "NULL buffer");
  if (row_base < 0 || (row_base + H) * W > 0x7fffffffLL)
    return set_error(SN_EINVAL, "label index range exceeds int32");
  return SN_OK;
}

// Entry points without a caller workspace take one from the device's private
// stream-ordered pool on the caller's stream and free it there: concurrent
// calls on different streams never share scratch, and the pool keeps the
// memory between calls (no cudaMalloc in the steady state).
struct StreamScratch {
  LaunchCtx ctx;
  void* ptr = nullptr;
  size_t bytes = 0;
  int acquire(const LaunchCtx& c, size_t n) {
    ctx = c;
    bytes = n;
    return scratch_alloc(c, n, &ptr);
  }
  ~StreamScratch() {
    if (ptr) scratch_free(ctx, ptr);
  }
};

template <typename T>
int ccl_labels_ws_impl(sn_plan_t* plan, const T* disp, int64_t B, int64_t H, int64_t W,
                       const sn_rig_t* rig, double t, int64_t row_base, int32_t* labels,
                       void* workspace, size_t ws_bytes, void* stream) {
  int rc = ccl_args(plan, B, H, W, row_base, disp, labels);
  if (rc) return rc;
  if ((rc = check_rig(rig))) return rc;
  if (!(t > 0.0)) return set_error(SN_EINVAL, "threshold must be positive");
  const CclParams p = make_ccl_params(B, H, W, rig->fx * rig->baseline, t);
  DeviceGuard g(plan->device);
  const LaunchCtx ctx = make_ctx(plan, stream);
  const int64_t B0 = B / 2, B1 = B - B0;
  const size_t w0 = ccl_workspace_bytes_one(B0, H, W);
  if (B < kCclSplitFrames || !workspace || ws_bytes < ccl_workspace_bytes(B, H, W))
    return run_ccl<T>(ctx, disp, nullptr, p, row_base * W, labels, workspace, ws_bytes);
  // two half batches on two streams (the caller's and the plan's second):
  // one half's issue-bound tile pass runs beside the other's memory-bound
  // predicate and resolve kernels, and each launch's tail is filled
  // (DESIGN 4.3).  Each half has its own workspace; the caller's stream
  // waits for both.
  std::lock_guard<std::mutex> lock(plan->aux_mu);
  if (!plan->s_aux) {
    if (cudaStreamCreateWithFlags(&plan->s_aux, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&plan->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&plan->ev_join, cudaEventDisableTiming) != cudaSuccess)
      return set_cuda_error("cudaStreamCreate(labeller halves)");
  }
  if (cudaEventRecord(plan->ev_fork, ctx.stream) != cudaSuccess ||
      cudaStreamWaitEvent(plan->s_aux, plan->ev_fork, 0) != cudaSuccess)
    return set_cuda_error("labeller fork");
  LaunchCtx aux = ctx;
  aux.stream = plan->s_aux;
  const CclParams p0 = make_ccl_params(B0, H, W, rig->fx * rig->baseline, t);
  const CclParams p1 = make_ccl_params(B1, H, W, rig->fx * rig->baseline, t);
  const int64_t off = B0 * H * W;
  rc = run_ccl<T>(ctx, disp, nullptr, p0, row_base * W, labels, workspace, w0);
  const int rc1 = run_ccl<T>(aux, disp + off, nullptr, p1, row_base * W, labels + off,
                             static_cast<uint8_t*>(workspace) + w0, ws_bytes - w0);
  // the join is recorded whatever happened, so the caller's stream never
  // runs ahead of work still queued on the second stream
  if (cudaEventRecord(plan->ev_join, plan->s_aux) != cudaSuccess ||
      cudaStreamWaitEvent(ctx.stream, plan->ev_join, 0) != cudaSuccess)
    return set_cuda_error("labeller join");
  return rc ? rc : rc1;
}

template <typename T>
int ccl_labels_impl(sn_plan_t* plan, const T* disp, int64_t B, int64_t H, int64_t W,
                    const sn_rig_t* rig, double t, int64_t row_base, int32_t* labels,
                    void* stream) {
  int rc = ccl_args(plan, B, H, W, row_base, disp, labels);
  if (rc) return rc;
  if (B * H * W == 0) return ccl_labels_ws_impl<T>(plan, disp, B, H, W, rig, t, row_base, labels,
                                                   nullptr, 0, stream);
  DeviceGuard g(plan->device);
  StreamScratch ws;
  if ((rc = ws.acquire(make_ctx(plan, stream), ccl_workspace_bytes(B, H, W)))) return rc;
  return ccl_labels_ws_impl<T>(plan, disp, B, H, W, rig, t, row_base, labels, ws.ptr, ws.bytes,
                               stream);
}

template <typename T>
int pipeline_ws_impl(sn_plan_t* plan, const T* disp, int64_t B, int64_t H, int64_t W,
                     const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off, double t,
                     float* out6, uint8_t* mask, int32_t* labels, void* workspace,
                     size_t ws_bytes, void* stream) {
  int rc = ccl_args(plan, B, H, W, 0, disp, labels);
  if (rc) return rc;
  if (B * H * W == 0) return SN_OK;
  if (!workspace || ws_bytes < ccl_workspace_bytes(B, H, W))
    return set_error(SN_EINVAL, "pipeline workspace too small");
  // the bit mask lives at the head of the labeller workspace
  uint32_t* bits = static_cast<uint32_t*>(workspace);
  if ((rc = oriented_points_impl<T>(plan, disp, B, H, W, rig, offsets_xy, n_off, out6, mask,
                                    stream, 0, 0, bits, t)))
    return rc;
  return sn_ccl_from_bits_ws(plan, bits, B, H, W, 0, labels, workspace, ws_bytes, stream);
}

template <typename T>
int pipeline_impl(sn_plan_t* plan, const T* disp, int64_t B, int64_t H, int64_t W,
                  const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off, double t,
                  float* out6, uint8_t* mask, int32_t* labels, void* stream) {
  int rc = ccl_args(plan, B, H, W, 0, disp, labels);
  if (rc) return rc;
  if (B * H * W == 0) return SN_OK;
  DeviceGuard g(plan->device);
  StreamScratch ws;
  if ((rc = ws.acquire(make_ctx(plan, stream), ccl_workspace_bytes(B, H, W)))) return rc;
  return pipeline_ws_impl<T>(plan, disp, B, H, W, rig, offsets_xy, n_off, t, out6, mask, labels,
                             ws.ptr, ws.bytes, stream);
}

}  // namespace

extern "C" {

int sn_ccl_labels_ws(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                     const sn_rig_t* rig, double t, int64_t row_base, int32_t* labels,
                     void* workspace, size_t ws_bytes, void* stream) {
  return ccl_labels_ws_impl<float>(plan, disp, B, H, W, rig, t, row_base, labels, workspace,
                                   ws_bytes, stream);
}

int sn_ccl_labels_ws_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H, int64_t W,
                         const sn_rig_t* rig, double t, int64_t row_base, int32_t* labels,
                         void* workspace, size_t ws_bytes, void* stream) {
  return ccl_labels_ws_impl<double>(plan, disp, B, H, W, rig, t, row_base, labels, workspace,
                                    ws_bytes, stream);
}

int sn_ccl_labels(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                  const sn_rig_t* rig, double t, int64_t row_base, int32_t* labels, void* stream) {
  return ccl_labels_impl<float>(plan, disp, B, H, W, rig, t, row_base, labels, stream);
}

int sn_ccl_labels_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H, int64_t W,
                      const sn_rig_t* rig, double t, int64_t row_base, int32_t* labels,
                      void* stream) {
  return ccl_labels_impl<double>(plan, disp, B, H, W, rig, t, row_base, labels, stream);
}

int sn_ccl_from_passable_ws(sn_plan_t* plan, const uint8_t* passable, int64_t B, int64_t H,
                            int64_t W, int64_t row_base, int32_t* labels, void* workspace,
                            size_t ws_bytes, void* stream) {
  int rc = ccl_args(plan, B, H, W, row_base, passable, labels);
  if (rc) return rc;
  const CclParams p = make_ccl_params(B, H, W, 0.0, 1.0);
  DeviceGuard g(plan->device);
  return run_ccl<float>(make_ctx(plan, stream), nullptr, passable, p, row_base * W, labels,
                        workspace, ws_bytes);
}

int sn_ccl_from_passable(sn_plan_t* plan, const uint8_t* passable, int64_t B, int64_t H, int64_t W,
                         int64_t row_base, int32_t* labels, void* stream) {
  int rc = ccl_args(plan, B, H, W, row_base, passable, labels);
  if (rc) return rc;
  if (B * H * W == 0) return SN_OK;
  DeviceGuard g(plan->device);
  StreamScratch ws;
  if ((rc = ws.acquire(make_ctx(plan, stream), ccl_workspace_bytes(B, H, W)))) return rc;
  return sn_ccl_from_passable_ws(plan, passable, B, H, W, row_base, labels, ws.ptr, ws.bytes,
                                 stream);
}

int sn_ccl_from_bits_ws(sn_plan_t* plan, const uint32_t* bits, int64_t B, int64_t H, int64_t W,
                        int64_t row_base, int32_t* labels, void* workspace, size_t ws_bytes,
                        void* stream) {
  int rc = ccl_args(plan, B, H, W, row_base, bits, labels);
  if (rc) return rc;
  const CclParams p = make_ccl_params(B, H, W, 0.0, 1.0);
  DeviceGuard g(plan->device);
  return run_ccl<float>(make_ctx(plan, stream), nullptr, nullptr, p, row_base * W, labels,
                        workspace, ws_bytes, bits);
}

int sn_pipeline_ws(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                   const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off, double t,
                   float* out6, uint8_t* mask, int32_t* labels, void* workspace, size_t ws_bytes,
                   void* stream) {
  return pipeline_ws_impl<float>(plan, disp, B, H, W, rig, offsets_xy, n_off, t, out6, mask,
                                 labels, workspace, ws_bytes, stream);
}

int sn_pipeline_ws_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H, int64_t W,
                       const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off, double t,
                       float* out6, uint8_t* mask, int32_t* labels, void* workspace,
                       size_t ws_bytes, void* stream) {
  return pipeline_ws_impl<double>(plan, disp, B, H, W, rig, offsets_xy, n_off, t, out6, mask,
                                  labels, workspace, ws_bytes, stream);
}

int sn_pipeline(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off, double t,
                float* out6, uint8_t* mask, int32_t* labels, void* stream) {
  return pipeline_impl<float>(plan, disp, B, H, W, rig, offsets_xy, n_off, t, out6, mask, labels,
                              stream);
}

int sn_pipeline_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H, int64_t W,
                    const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off, double t,
                    float* out6, uint8_t* mask, int32_t* labels, void* stream) {
  return pipeline_impl<double>(plan, disp, B, H, W, rig, offsets_xy, n_off, t, out6, mask, labels,
                               stream);
}

}  // extern "C"

namespace {

template <typename T>
int depth_map_impl(sn_plan_t* plan, const T* disp, int64_t n, const sn_rig_t* rig, double* z,
                   void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  if (n < 0) return set_error(SN_EINVAL, "negative size");
  int rc = check_rig(rig);
  if (rc) return rc;
  if (n > 0 && (!disp || !z)) return set_error(SN_EINVAL, "NULL buffer");
  DeviceGuard g(plan->device);
  return run_depth_map<T>(make_ctx(plan, stream), disp, n, rig->fx * rig->baseline, z);
}

template <typename T>
int triangulate_grid_impl(sn_plan_t* plan, const T* disp, int64_t B, int64_t H, int64_t W,
                          const sn_rig_t* rig, double* xyz, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if ((rc = check_rig(rig))) return rc;
  if (B * H * W > 0 && (!disp || !xyz)) return set_error(SN_EINVAL, "NULL buffer");
  FixedParams p{};
  p.B = B;
  p.H = H;
  p.W = W;
  fill_rig(p, rig);
  DeviceGuard g(plan->device);
  return run_triangulate_grid<T>(make_ctx(plan, stream), disp, p, xyz);
}

}  // namespace

extern "C" {

int sn_depth_map(sn_plan_t* plan, const float* disp, int64_t n, const sn_rig_t* rig, double* z,
                 void* stream) {
  return depth_map_impl<float>(plan, disp, n, rig, z, stream);
}

int sn_depth_map_f64(sn_plan_t* plan, const double* disp, int64_t n, const sn_rig_t* rig,
                     double* z, void* stream) {
  return depth_map_impl<double>(plan, disp, n, rig, z, stream);
}

int sn_triangulate_f64(sn_plan_t* plan, const double* u, const double* v, const double* d,
                       int64_t n, const sn_rig_t* rig, double* x, double* y, double* z,
                       void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  if (n < 0) return set_error(SN_EINVAL, "negative size");
  int rc = check_rig(rig);
  if (rc) return rc;
  if (n > 0 && (!u || !v || !d || !x || !y || !z)) return set_error(SN_EINVAL, "NULL buffer");
  FixedParams p{};
  fill_rig(p, rig);
  DeviceGuard g(plan->device);
  return run_triangulate(make_ctx(plan, stream), u, v, d, n, p, x, y, z);
}

int sn_triangulate_grid(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                        const sn_rig_t* rig, double* xyz, void* stream) {
  return triangulate_grid_impl<float>(plan, disp, B, H, W, rig, xyz, stream);
}

int sn_triangulate_grid_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H, int64_t W,
                            const sn_rig_t* rig, double* xyz, void* stream) {
  return triangulate_grid_impl<double>(plan, disp, B, H, W, rig, xyz, stream);
}

int sn_depth_laplacian_f64(sn_plan_t* plan, const double* depth, const uint8_t* mask, int64_t B,
                           int64_t H, int64_t W, double* edges, uint8_t* ok, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if (B * H * W > 0 && (!depth || !mask || (!edges && !ok)))
    return set_error(SN_EINVAL, "NULL buffer");
  DeviceGuard g(plan->device);
  return run_laplacian(make_ctx(plan, stream), depth, mask, B, H, W, edges, ok);
}

int sn_relabel(sn_plan_t* plan, int32_t* labels, int64_t n, int64_t index_base,
               const int32_t* map_keys, const int32_t* map_vals, const int32_t* n_map,
               int32_t map_capacity, int32_t* scratch, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  if (n < 0 || map_capacity < 0) return set_error(SN_EINVAL, "negative size");
  if (n > 0 && (!labels || !scratch || !map_keys || !map_vals || !n_map))
    return set_error(SN_EINVAL, "NULL buffer");
  DeviceGuard g(plan->device);
  return run_relabel(make_ctx(plan, stream), labels, n, index_base, map_keys, map_vals, n_map,
                     map_capacity, scratch);
}

int sn_seam_merge(sn_plan_t* plan, const int32_t* seams, int32_t n_strips, int64_t W,
                  int32_t* table, int64_t table_n, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  if (n_strips < 0 || W < 0 || table_n < 0 || W > 0x7fffffffLL)
    return set_error(SN_EINVAL, "bad seam-merge arguments");
  if ((int64_t)n_strips * W > 0 && (!seams || !table)) return set_error(SN_EINVAL, "NULL buffer");
  DeviceGuard g(plan->device);
  return run_seam_merge(make_ctx(plan, stream), seams, n_strips, W, table, table_n);
}

int sn_relabel_table(sn_plan_t* plan, int32_t* labels, int64_t n, const int32_t* table,
                     int64_t table_n, void* stream) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  if (n < 0 || table_n < 0) return set_error(SN_EINVAL, "negative size");
  if (n > 0 && (!labels || !table)) return set_error(SN_EINVAL, "NULL buffer");
  DeviceGuard g(plan->device);
  return run_relabel_table(make_ctx(plan, stream), labels, n, table, table_n);
}

// Strip-seam merge on gathered boundary rows (host memory; tiny: 2 rows per
// strip).  Union-find over label values with min-root links, so the map is
// independent of gather order and identical on every rank.
int sn_seam_merge_host(const int32_t* seams, int32_t n_strips, int64_t W, int32_t* map_keys,
                       int32_t* map_vals, int32_t* n_map) {
  if (!seams || !map_keys || !map_vals || !n_map || n_strips < 0 || W < 0)
    return set_error(SN_EINVAL, "bad seam-merge arguments");
  std::unordered_map<int32_t, int32_t> parent;
  parent.reserve((size_t)n_strips * 2 * (size_t)W);
  auto find = [&](int32_t x) {
    int32_t r = x;
    while (true) {
      const int32_t p = parent[r];
      if (p == r) break;
      r = p;
    }
    while (parent[x] != r) {  // path compression
      const int32_t nx = parent[x];
      parent[x] = r;
      x = nx;
    }
    return r;
  };
  for (int64_t i = 0; i < (int64_t)n_strips * 2 * W; ++i)
    if (seams[i] >= 0) parent.emplace(seams[i], seams[i]);
  for (int32_t s = 0; s + 1 < n_strips; ++s) {
    const int32_t* a = seams + ((int64_t)s * 2 + 1) * W;   // last owned row of strip s
    const int32_t* b = seams + ((int64_t)(s + 1) * 2) * W;  // first owned row of strip s+1
    for (int64_t u = 0; u < W; ++u) {
      if (b[u] < 0) continue;
      for (int64_t du = -1; du <= 1; ++du) {
        const int64_t uu = u + du;
        if (uu < 0 || uu >= W || a[uu] < 0) continue;
        int32_t ra = find(a[uu]), rb = find(b[u]);
        if (ra == rb) continue;
        if (ra < rb) parent[rb] = ra;
        else parent[ra] = rb;
      }
    }
  }
  std::vector<int32_t> keys;
  keys.reserve(parent.size());
  for (auto& kv : parent) keys.push_back(kv.first);
  std::sort(keys.begin(), keys.end());
  int32_t n = 0;
  for (int32_t k : keys) {
    const int32_t r = find(k);
    if (r != k) {
      map_keys[n] = k;
      map_vals[n] = r;
      ++n;
    }
  }
  *n_map = n;
  return SN_OK;
}

// ---------------------------------------------------------------------------
// host-buffer path: frames in chunks, H2D / compute / D2H overlapped on three
// streams with double-buffered device staging.

}  // extern "C"

namespace {

bool is_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// host memcpy split over a few threads (a single core copies ~10 GB/s; the
// pageable staging would otherwise run below the PCIe rate)
void par_copy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kMinPart = 8u << 20;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t parts = std::min<size_t>(std::min<size_t>(hw, 8), std::max<size_t>(1, bytes / kMinPart));
  if (parts <= 1) {
    memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t step = (bytes / parts + 63) / 64 * 64;
  for (size_t off = 0; off < bytes; off += step) {
    const size_t n = std::min(step, bytes - off);
    th.emplace_back([=] { memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, n); });
  }
  for (auto& t : th) t.join();
}

int grow_pinned(void** buf, size_t& cap, size_t need) {
  if (cap >= need) return SN_OK;
  for (int i = 0; i < 2; ++i) {
    if (buf[i]) cudaFreeHost(buf[i]);
    buf[i] = nullptr;
  }
  cap = 0;
  for (int i = 0; i < 2; ++i)
    if (cudaHostAlloc(&buf[i], need, cudaHostAllocDefault) != cudaSuccess)
      return set_cuda_error("cudaHostAlloc(host-path staging)");
  cap = need;
  return SN_OK;
}

// host-buffer pipeline: frames in chunks, H2D / compute / D2H overlapped on
// three streams with double-buffered device staging; labels (and the passable
// bits they need) only when labels_host is non-NULL.  Pinned (page-locked)
// caller buffers are copied directly; pageable ones go through the plan's
// pinned staging slots, filled / drained by multi-threaded host copies while
// the device works on the other slot.
template <typename T>
int host_pipeline(sn_plan_t* plan, const T* disp_host, int64_t B, int64_t H, int64_t W,
                  const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off, double t,
                  float* out6_host, uint8_t* mask_host, int32_t* labels_host) {
  if (!plan) return set_error(SN_EINVAL, "plan is NULL");
  int rc = check_shape(B, H, W);
  if (rc) return rc;
  if ((rc = check_rig(rig))) return rc;
  sn_moments_t m;
  if ((rc = sn_kernel_moments(offsets_xy, n_off, &m))) return rc;
  if (labels_host && !(t > 0.0)) return set_error(SN_EINVAL, "threshold must be positive");
  const int64_t frame_px = H * W;
  if (B * frame_px == 0) return SN_OK;
  if (!disp_host || !out6_host) return set_error(SN_EINVAL, "NULL buffer");
  std::lock_guard<std::mutex> lock(plan->mu);
  DeviceGuard g(plan->device);
  // chunk: ~16 Mpx per step (64-128 MB in, 384 MB out), whole frames
  int64_t chunk = std::max<int64_t>(1, (int64_t)(16 << 20) / std::max<int64_t>(frame_px, 1));
  chunk = std::min<int64_t>(chunk, B);
  const size_t need = (size_t)(chunk * frame_px);
  const size_t ws_need = labels_host ? ccl_workspace_bytes(chunk, H, W) : 0;
  if (plan->cap_px < need || plan->cap_in < need * sizeof(T) ||
      (labels_host && (!plan->d_lab[0] || plan->ws_cap < ws_need))) {
    for (int i = 0; i < 2; ++i) {
      cudaFree(plan->d_in[i]);
      cudaFree(plan->d_out[i]);
      cudaFree(plan->d_mask[i]);
      cudaFree(plan->d_lab[i]);
      cudaFree(plan->d_ws[i]);
      plan->d_in[i] = nullptr;
      plan->d_out[i] = nullptr;
      plan->d_mask[i] = nullptr;
      plan->d_lab[i] = nullptr;
      plan->d_ws[i] = nullptr;
    }
    plan->cap_px = plan->cap_in = plan->ws_cap = 0;
    for (int i = 0; i < 2; ++i) {
      if (cudaMalloc(&plan->d_in[i], need * sizeof(double)) != cudaSuccess ||
          cudaMalloc(&plan->d_out[i], need * 24) != cudaSuccess ||
          cudaMalloc(&plan->d_mask[i], need) != cudaSuccess)
        return set_cuda_error("cudaMalloc(host-path staging)");
      if (labels_host && (cudaMalloc(&plan->d_lab[i], need * 4) != cudaSuccess ||
                          cudaMalloc(&plan->d_ws[i], ws_need) != cudaSuccess))
        return set_cuda_error("cudaMalloc(host-path labeller staging)");
    }
    plan->cap_px = need;
    plan->cap_in = need * sizeof(double);
    if (labels_host) plan->ws_cap = ws_need;
  }
  if (!plan->s_h2d) {
    if (cudaStreamCreateWithFlags(&plan->s_h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&plan->s_comp, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&plan->s_d2h, cudaStreamNonBlocking) != cudaSuccess)
      return set_cuda_error("cudaStreamCreate");
    for (int i = 0; i < 2; ++i) {
      if (cudaEventCreateWithFlags(&plan->ev_in[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&plan->ev_done[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&plan->ev_out[i], cudaEventDisableTiming) != cudaSuccess)
        return set_cuda_error("cudaEventCreate");
    }
  }
  // pageable buffers -> pinned staging slots; the output slot packs the
  // records, then the mask, then the labels of one chunk
  const bool pin_in = is_pinned(disp_host);
  const bool pin_out = is_pinned(out6_host) && is_pinned(mask_host) && is_pinned(labels_host);
  const size_t out_slot = need * 24 + (mask_host ? need : 0) + (labels_host ? need * 4 : 0);
  if (!pin_in && (rc = grow_pinned(plan->h_in, plan->h_in_cap, need * sizeof(T)))) return rc;
  if (!pin_out && (rc = grow_pinned(plan->h_out, plan->h_out_cap, out_slot))) return rc;

  // chunk c covers frames [cf0(c), cf0(c) + cnf(c)): a ramp of 1, 2, 4, ...
  // frames up to `chunk`, so the first D2H starts after one frame's H2D and
  // compute instead of a whole chunk's (the pipeline fill)
  int ramp = 0;  // ramp chunks: sizes 1, 2, .., 2^(ramp-1), all < chunk
  while (((int64_t)1 << ramp) < chunk) ++ramp;
  auto cf0 = [&](int64_t c) -> int64_t {
    return c <= ramp ? ((int64_t)1 << c) - 1 : (((int64_t)1 << ramp) - 1) + (c - ramp) * chunk;
  };
  auto cnf = [&](int64_t c) -> int64_t {
    return std::min<int64_t>(c < ramp ? (int64_t)1 << c : chunk, B - cf0(c));
  };
  int64_t n_chunks = 0;
  while (cf0(n_chunks) < B) ++n_chunks;
  // every exit waits for the queued work (it may still read or write the
  // caller's buffers or a staging slot)
  auto drain_all = [&] {
    cudaStreamSynchronize(plan->s_h2d);
    cudaStreamSynchronize(plan->s_comp);
    cudaStreamSynchronize(plan->s_d2h);
  };
  auto fail = [&](int code) {
    drain_all();
    cudaGetLastError();
    return code;
  };
  // copy chunk c's outputs out of its pinned slot (pageable callers)
  auto drain_out = [&](int64_t c) -> int {
    const int s = (int)(c & 1);
    const int64_t f0 = cf0(c), nf = cnf(c);
    const size_t px = (size_t)(nf * frame_px);
    if (cudaEventSynchronize(plan->ev_out[s]) != cudaSuccess) return set_cuda_error("D2H wait");
    const char* src = static_cast<const char*>(plan->h_out[s]);
    par_copy(out6_host + f0 * frame_px * 6, src, px * 24);
    src += need * 24;
    if (mask_host) {
      par_copy(mask_host + f0 * frame_px, src, px);
      src += need;
    }
    if (labels_host) par_copy(labels_host + f0 * frame_px, src, px * 4);
    return SN_OK;
  };
  for (int64_t c = 0; c < n_chunks; ++c) {
    const int s = (int)(c & 1);
    const int64_t f0 = cf0(c);
    const int64_t nf = cnf(c);
    const size_t px = (size_t)(nf * frame_px);
    if (!pin_out && c >= 2 && (rc = drain_out(c - 2))) return fail(rc);
    // buffers of slot s are free once chunk c-2's compute (inputs) and D2H (outputs) are done
    if (c >= 2) {
      cudaStreamWaitEvent(plan->s_h2d, plan->ev_done[s], 0);
      cudaStreamWaitEvent(plan->s_comp, plan->ev_out[s], 0);
    }
    const T* src = disp_host + f0 * frame_px;
    if (!pin_in) {
      // chunk c-2's H2D read this slot: its compute has started after it, so
      // ev_in[s] (recorded after that copy) marks the slot free
      if (c >= 2 && cudaEventSynchronize(plan->ev_in[s]) != cudaSuccess)
        return fail(set_cuda_error("H2D wait"));
      par_copy(plan->h_in[s], src, px * sizeof(T));
      src = static_cast<const T*>(plan->h_in[s]);
    }
    if (cudaMemcpyAsync(plan->d_in[s], src, px * sizeof(T), cudaMemcpyHostToDevice,
                        plan->s_h2d) != cudaSuccess)
      return fail(set_cuda_error("H2D copy"));
    cudaEventRecord(plan->ev_in[s], plan->s_h2d);
    cudaStreamWaitEvent(plan->s_comp, plan->ev_in[s], 0);
    uint8_t* dmask = mask_host ? plan->d_mask[s] : nullptr;
    const T* din = static_cast<const T*>(plan->d_in[s]);
    if (labels_host)
      rc = pipeline_ws_impl<T>(plan, din, nf, H, W, rig, offsets_xy, n_off, t, plan->d_out[s],
                               dmask, plan->d_lab[s], plan->d_ws[s], plan->ws_cap, plan->s_comp);
    else
      rc = oriented_points_impl<T>(plan, din, nf, H, W, rig, offsets_xy, n_off, plan->d_out[s],
                                   dmask, plan->s_comp, 0);
    if (rc) return fail(rc);
    cudaEventRecord(plan->ev_done[s], plan->s_comp);
    cudaStreamWaitEvent(plan->s_d2h, plan->ev_done[s], 0);
    char* hout = pin_out ? nullptr : static_cast<char*>(plan->h_out[s]);
    float* o6 = pin_out ? out6_host + f0 * frame_px * 6 : reinterpret_cast<float*>(hout);
    if (cudaMemcpyAsync(o6, plan->d_out[s], px * 24, cudaMemcpyDeviceToHost, plan->s_d2h) !=
        cudaSuccess)
      return fail(set_cuda_error("D2H copy"));
    if (mask_host) {
      uint8_t* mo = pin_out ? mask_host + f0 * frame_px : reinterpret_cast<uint8_t*>(hout + need * 24);
      if (cudaMemcpyAsync(mo, plan->d_mask[s], px, cudaMemcpyDeviceToHost, plan->s_d2h) !=
          cudaSuccess)
        return fail(set_cuda_error("D2H mask copy"));
    }
    if (labels_host) {
      int32_t* lo = pin_out ? labels_host + f0 * frame_px
                            : reinterpret_cast<int32_t*>(hout + need * 24 + (mask_host ? need : 0));
      if (cudaMemcpyAsync(lo, plan->d_lab[s], px * 4, cudaMemcpyDeviceToHost, plan->s_d2h) !=
          cudaSuccess)
        return fail(set_cuda_error("D2H label copy"));
    }
    cudaEventRecord(plan->ev_out[s], plan->s_d2h);
  }
  if (!pin_out)
    for (int64_t c = std::max<int64_t>(0, n_chunks - 2); c < n_chunks; ++c)
      if ((rc = drain_out(c))) return fail(rc);
  if (cudaStreamSynchronize(plan->s_d2h) != cudaSuccess) return fail(set_cuda_error("host-path sync"));
  if (cudaStreamSynchronize(plan->s_comp) != cudaSuccess) return fail(set_cuda_error("host-path sync"));
  return SN_OK;
}

}  // namespace

extern "C" {

int sn_oriented_points_host(sn_plan_t* plan, const float* disp_host, int64_t B, int64_t H,
                            int64_t W, const sn_rig_t* rig, const int32_t* offsets_xy,
                            int32_t n_off, float* out6_host, uint8_t* mask_host) {
  return host_pipeline<float>(plan, disp_host, B, H, W, rig, offsets_xy, n_off, 0.0, out6_host,
                              mask_host, nullptr);
}

int sn_oriented_points_host_f64(sn_plan_t* plan, const double* disp_host, int64_t B, int64_t H,
                                int64_t W, const sn_rig_t* rig, const int32_t* offsets_xy,
                                int32_t n_off, float* out6_host, uint8_t* mask_host) {
  return host_pipeline<double>(plan, disp_host, B, H, W, rig, offsets_xy, n_off, 0.0, out6_host,
                               mask_host, nullptr);
}

int sn_pipeline_host(sn_plan_t* plan, const float* disp_host, int64_t B, int64_t H, int64_t W,
                     const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off, double t,
                     float* out6_host, uint8_t* mask_host, int32_t* labels_host) {
  if (B * H * W > 0 && !labels_host) return set_error(SN_EINVAL, "NULL label buffer");
  return host_pipeline<float>(plan, disp_host, B, H, W, rig, offsets_xy, n_off, t, out6_host,
                              mask_host, labels_host);
}

int sn_pipeline_host_f64(sn_plan_t* plan, const double* disp_host, int64_t B, int64_t H,
                         int64_t W, const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off,
                         double t, float* out6_host, uint8_t* mask_host, int32_t* labels_host) {
  if (B * H * W > 0 && !labels_host) return set_error(SN_EINVAL, "NULL label buffer");
  return host_pipeline<double>(plan, disp_host, B, H, W, rig, offsets_xy, n_off, t, out6_host,
                               mask_host, labels_host);
}

}  // extern "C"
