// Device-side accuracy evaluation for sm_100a.
//
// Reference: evaluation.py:34-73.  angular_error_map: on jointly valid
// pixels (optionally restricted by a mask), both normals renormalised, the
// unsigned angle degrees(arccos(clip(|n_est . n_gt|, 0, 1))); summarize:
// mean, min, max, lower median (element (n-1)/2 of the sorted values),
// population std -- per frame.  fp64 throughout.
//
//   eval_angle_kernel    angle map + per-chunk (count, sum, min, max)
//   eval_reduce_kernel   per frame: deterministic sums over chunks -> mean
//   eval_dev_kernel      per-chunk sums of squared deviations
//   eval_hist/pick       lower median by an 8-pass radix select on
//                        order-preserving keys of the values
// Sums use fixed chunk order, so the statistics are deterministic.

#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "sn_internal.h"

namespace sn {

constexpr int kEvalChunk = 8192;  // pixels per chunk (one CTA)
constexpr int kEvalThreads = 256;

struct EvalWs {
  double* err;         // [B][HW] angle map (NaN invalid), if the caller gave none
  double* part;        // [B][n_chunks][4] count, sum, min, max -> then [.][1] = dev sum
  double* mean;        // [B]
  uint32_t* hist;      // [B][256]
  uint64_t* prefix;    // [B] radix-select prefix
  int64_t* rank;       // [B] rank remaining within the prefix
};

__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kEvalThreads / 32; ++w) s += red[w];
  return s;  // valid in thread 0
}

template <typename TE>
__global__ void __launch_bounds__(kEvalThreads)
    eval_angle_kernel(const TE* __restrict__ est, int est_stride, const double* __restrict__ gt,
                      const uint8_t* __restrict__ gt_mask, const uint8_t* __restrict__ extra,
                      int64_t HW, int n_chunks, double* __restrict__ err,
                      double* __restrict__ part) {
  __shared__ double red[kEvalThreads / 32];
  const int f = blockIdx.y, ch = blockIdx.x;
  const int64_t base = (int64_t)f * HW;
  double cnt = 0.0, sum = 0.0, mn = DBL_MAX, mx = -DBL_MAX;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  for (int64_t i = (int64_t)ch * kEvalChunk + threadIdx.x;
       i < min((int64_t)(ch + 1) * kEvalChunk, HW); i += kEvalThreads) {
    const TE* e = est + (base + i) * est_stride;
    const double* g = gt + (base + i) * 3;
    const double ex = e[0], ey = e[1], ez = e[2];
    bool ok = (ex == ex) && (ey == ey) && (ez == ez) && gt_mask[base + i] != 0 &&
              (extra == nullptr || extra[base + i] != 0);
    double ang = qnan;
    if (ok) {
      const double en = sqrt(ex * ex + ey * ey + ez * ez);
      const double gn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
      const double dot = fabs((ex / en) * (g[0] / gn) + (ey / en) * (g[1] / gn) +
                              (ez / en) * (g[2] / gn));
      // numpy's clip keeps a NaN (zero-length vector) and arccos(NaN) is NaN
      ang = dot == dot ? acos(fmin(fmax(dot, 0.0), 1.0)) * (180.0 / 3.14159265358979323846)
                       : qnan;
      ok = fabs(ang) <= DBL_MAX;
      if (!ok) ang = qnan;
    }
    err[base + i] = ang;
    if (ok) {
      cnt += 1.0;
      sum += ang;
      mn = fmin(mn, ang);
      mx = fmax(mx, ang);
    }
  }
  const double c = block_sum(cnt, red);
  const double s = block_sum(sum, red);
  // min / max by warp shuffles then smem
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    mn = fmin(mn, __shfl_down_sync(0xffffffffu, mn, d));
    mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, d));
  }
  __shared__ double rmn[kEvalThreads / 32], rmx[kEvalThreads / 32];
  if ((threadIdx.x & 31) == 0) {
    rmn[threadIdx.x >> 5] = mn;
    rmx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kEvalThreads / 32; ++w) {
      mn = fmin(mn, rmn[w]);
      mx = fmax(mx, rmx[w]);
    }
    double* o = part + ((int64_t)f * n_chunks + ch) * 4;
    o[0] = c;
    o[1] = s;
    o[2] = mn;
    o[3] = mx;
  }
}

// statistics of a given map (NaN = invalid): per-chunk count/sum/min/max
__global__ void __launch_bounds__(kEvalThreads)
    eval_values_kernel(const double* __restrict__ err, int64_t HW, int n_chunks,
                       double* __restrict__ part) {
  __shared__ double red[kEvalThreads / 32];
  __shared__ double rmn[kEvalThreads / 32], rmx[kEvalThreads / 32];
  const int f = blockIdx.y, ch = blockIdx.x;
  const int64_t base = (int64_t)f * HW;
  double cnt = 0.0, sum = 0.0, mn = DBL_MAX, mx = -DBL_MAX;
  for (int64_t i = (int64_t)ch * kEvalChunk + threadIdx.x;
       i < min((int64_t)(ch + 1) * kEvalChunk, HW); i += kEvalThreads) {
    const double v = err[base + i];
    if (fabs(v) <= DBL_MAX) {
      cnt += 1.0;
      sum += v;
      mn = fmin(mn, v);
      mx = fmax(mx, v);
    }
  }
  const double c = block_sum(cnt, red);
  const double s = block_sum(sum, red);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    mn = fmin(mn, __shfl_down_sync(0xffffffffu, mn, d));
    mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, d));
  }
  if ((threadIdx.x & 31) == 0) {
    rmn[threadIdx.x >> 5] = mn;
    rmx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kEvalThreads / 32; ++w) {
      mn = fmin(mn, rmn[w]);
      mx = fmax(mx, rmx[w]);
    }
    double* o = part + ((int64_t)f * n_chunks + ch) * 4;
    o[0] = c;
    o[1] = s;
    o[2] = mn;
    o[3] = mx;
  }
}

// per frame (one CTA): totals over chunks in chunk order; stats[f] =
// (avg, min, max, median, std, count) -- avg/min/max/count here
__global__ void eval_reduce_kernel(const double* __restrict__ part, int n_chunks,
                                   double* __restrict__ stats, double* __restrict__ mean,
                                   int64_t* __restrict__ rank, uint64_t* __restrict__ prefix) {
  const int f = blockIdx.x;
  if (threadIdx.x != 0) return;
  double c = 0.0, s = 0.0, mn = DBL_MAX, mx = -DBL_MAX;
  for (int ch = 0; ch < n_chunks; ++ch) {
    const double* o = part + ((int64_t)f * n_chunks + ch) * 4;
    c += o[0];
    s += o[1];
    mn = fmin(mn, o[2]);
    mx = fmax(mx, o[3]);
  }
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  double* st = stats + (int64_t)f * 6;
  st[0] = c > 0 ? s / c : qnan;
  st[1] = c > 0 ? mn : qnan;
  st[2] = c > 0 ? mx : qnan;
  st[5] = c;
  mean[f] = c > 0 ? s / c : 0.0;
  rank[f] = c > 0 ? (int64_t)((c - 1) / 2) : -1;  // lower middle element
  prefix[f] = 0;
}

__global__ void __launch_bounds__(kEvalThreads)
    eval_dev_kernel(const double* __restrict__ err, int64_t HW, int n_chunks,
                    const double* __restrict__ mean, double* __restrict__ part) {
  __shared__ double red[kEvalThreads / 32];
  const int f = blockIdx.y, ch = blockIdx.x;
  const int64_t base = (int64_t)f * HW;
  const double m = mean[f];
  double s = 0.0;
  for (int64_t i = (int64_t)ch * kEvalChunk + threadIdx.x;
       i < min((int64_t)(ch + 1) * kEvalChunk, HW); i += kEvalThreads) {
    const double v = err[base + i];
    if (fabs(v) <= DBL_MAX) s += (v - m) * (v - m);
  }
  const double t = block_sum(s, red);
  if (threadIdx.x == 0) part[((int64_t)f * n_chunks + ch) * 4 + 1] = t;
}

__global__ void eval_std_kernel(const double* __restrict__ part, int n_chunks,
                                double* __restrict__ stats) {
  const int f = blockIdx.x;
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int ch = 0; ch < n_chunks; ++ch) s += part[((int64_t)f * n_chunks + ch) * 4 + 1];
  double* st = stats + (int64_t)f * 6;
  st[4] = st[5] > 0 ? sqrt(s / st[5]) : __longlong_as_double(0x7ff8000000000000ll);
}

// order-preserving uint64 key of a double (negatives reversed), and back
__device__ __forceinline__ uint64_t order_key(double v) {
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// radix select, digit `pass` (0 = most significant byte) of the value keys
__global__ void __launch_bounds__(kEvalThreads)
    eval_hist_kernel(const double* __restrict__ err, int64_t HW, int pass,
                     const uint64_t* __restrict__ prefix, const int64_t* __restrict__ rank,
                     uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  const int f = blockIdx.y, ch = blockIdx.x;
  if (rank[f] < 0) return;
  for (int i = threadIdx.x; i < 256; i += kEvalThreads) h[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)f * HW;
  const int shift = 56 - 8 * pass;
  const uint64_t pre = prefix[f];
  const uint64_t hi_mask = pass == 0 ? 0ull : (~0ull << (64 - 8 * pass));
  for (int64_t i = (int64_t)ch * kEvalChunk + threadIdx.x;
       i < min((int64_t)(ch + 1) * kEvalChunk, HW); i += kEvalThreads) {
    const double v = err[base + i];
    if (!(fabs(v) <= DBL_MAX)) continue;
    const uint64_t b = order_key(v);
    if ((b & hi_mask) == pre) atomicAdd(&h[(b >> shift) & 0xff], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += kEvalThreads)
    if (h[i]) atomicAdd(&hist[f * 256 + i], h[i]);
}

__global__ void eval_pick_kernel(int pass, uint64_t* __restrict__ prefix,
                                 int64_t* __restrict__ rank, uint32_t* __restrict__ hist,
                                 double* __restrict__ stats) {
  const int f = blockIdx.x;
  if (threadIdx.x != 0) return;
  uint32_t* hf = hist + f * 256;
  if (rank[f] >= 0) {
    int64_t r = rank[f];
    int dgt = 0;
    for (; dgt < 256; ++dgt) {
      if (r < (int64_t)hf[dgt]) break;
      r -= hf[dgt];
    }
    prefix[f] |= (uint64_t)dgt << (56 - 8 * pass);
    rank[f] = r;
    if (pass == 7) stats[(int64_t)f * 6 + 3] = key_value(prefix[f]);
  } else if (pass == 7) {
    stats[(int64_t)f * 6 + 3] = __longlong_as_double(0x7ff8000000000000ll);
  }
  for (int i = 0; i < 256; ++i) hf[i] = 0;
}

size_t eval_workspace_bytes(int64_t B, int64_t H, int64_t W) {
  const int64_t HW = H * W;
  const int64_t nch = (HW + kEvalChunk - 1) / kEvalChunk;
  auto a = [](size_t v) { return (v + 255) / 256 * 256; };
  return a((size_t)(B * HW) * 8) + a((size_t)(B * nch * 4) * 8) + a((size_t)B * 8) +
         a((size_t)B * 256 * 4) + a((size_t)B * 8) + a((size_t)B * 8);
}

int run_eval(const LaunchCtx& ctx, const float* est, const double* est_d, int est_stride,
             const double* gt,
             const uint8_t* gt_mask, const uint8_t* extra, int64_t B, int64_t H, int64_t W,
             double* err_out, double* stats, void* workspace, size_t ws_bytes) {
  const int64_t HW = H * W;
  if (B == 0) return SN_OK;
  if (!workspace || ws_bytes < eval_workspace_bytes(B, H, W))
    return set_error(SN_EINVAL, "evaluation workspace too small");
  if (B > 65535) return set_error(SN_EINVAL, "at most 65535 frames per call");
  const int64_t nch64 = (HW + kEvalChunk - 1) / kEvalChunk;
  if (nch64 > 0x7fffffffLL || nch64 == 0) return set_error(SN_EINVAL, "bad frame size");
  const int nch = (int)nch64;
  auto a = [](size_t v) { return (v + 255) / 256 * 256; };
  uint8_t* q = static_cast<uint8_t*>(workspace);
  EvalWs ws;
  ws.err = reinterpret_cast<double*>(q);
  q += a((size_t)(B * HW) * 8);
  ws.part = reinterpret_cast<double*>(q);
  q += a((size_t)(B * nch * 4) * 8);
  ws.mean = reinterpret_cast<double*>(q);
  q += a((size_t)B * 8);
  ws.hist = reinterpret_cast<uint32_t*>(q);
  q += a((size_t)B * 256 * 4);
  ws.prefix = reinterpret_cast<uint64_t*>(q);
  q += a((size_t)B * 8);
  ws.rank = reinterpret_cast<int64_t*>(q);
  double* err = err_out ? err_out : ws.err;
  dim3 grid((unsigned)nch, (unsigned)B);
  if (cudaMemsetAsync(ws.hist, 0, (size_t)B * 256 * 4, ctx.stream) != cudaSuccess)
    return set_cuda_error("cudaMemsetAsync(eval histogram)");
  if (!est && !est_d)  // statistics of the map the caller passed in err_out
    eval_values_kernel<<<grid, kEvalThreads, 0, ctx.stream>>>(err, HW, nch, ws.part);
  else if (est_d)
    eval_angle_kernel<double><<<grid, kEvalThreads, 0, ctx.stream>>>(est_d, est_stride, gt, gt_mask,
                                                                     extra, HW, nch, err, ws.part);
  else
    eval_angle_kernel<float><<<grid, kEvalThreads, 0, ctx.stream>>>(est, est_stride, gt, gt_mask,
                                                                    extra, HW, nch, err, ws.part);
  int rc = check_launch("eval_angle_kernel");
  if (rc) return rc;
  eval_reduce_kernel<<<(unsigned)B, 32, 0, ctx.stream>>>(ws.part, nch, stats, ws.mean, ws.rank,
                                                         ws.prefix);
  if ((rc = check_launch("eval_reduce_kernel"))) return rc;
  eval_dev_kernel<<<grid, kEvalThreads, 0, ctx.stream>>>(err, HW, nch, ws.mean, ws.part);
  if ((rc = check_launch("eval_dev_kernel"))) return rc;
  eval_std_kernel<<<(unsigned)B, 32, 0, ctx.stream>>>(ws.part, nch, stats);
  if ((rc = check_launch("eval_std_kernel"))) return rc;
  for (int pass = 0; pass < 8; ++pass) {
    eval_hist_kernel<<<grid, kEvalThreads, 0, ctx.stream>>>(err, HW, pass, ws.prefix, ws.rank,
                                                            ws.hist);
    if ((rc = check_launch("eval_hist_kernel"))) return rc;
    eval_pick_kernel<<<(unsigned)B, 32, 0, ctx.stream>>>(pass, ws.prefix, ws.rank, ws.hist, stats);
    if ((rc = check_launch("eval_pick_kernel"))) return rc;
  }
  return SN_OK;
}

}  // namespace sn
