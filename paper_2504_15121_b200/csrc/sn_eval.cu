// Device-side accuracy evaluation for sm_100a.
//
// Reference: evaluation.py:34-73.  angular_error_map: on jointly valid
// pixels (optionally restricted by a mask), both normals renormalised, the
// unsigned angle degrees(arccos(clip(|n_est . n_gt|, 0, 1))); summarize:
// mean, min, max, lower median (element (n-1)/2 of the sorted values),
// population std -- per frame.  fp64 throughout.
//
// Three streaming passes over a frame (chunks of 8192 values, one CTA each):
//   eval_pass1_kernel   angle map (or the caller's map) + per-chunk count,
//                       sum, min, max and sum of squared deviations from the
//                       chunk mean (a second, L2-resident read), + a 4096-bin
//                       histogram of the top 12 bits of order-preserving
//                       value keys (sign + exponent)
//   eval_reduce_kernel  per frame: chunk totals in chunk order (mean, and
//                       M2 = sum M2_i + n_i (m_i - m)^2), the histogram bin
//                       holding the lower median
//   eval_hist2_kernel   next 12 key bits of the values in that bin
//   eval_pick2_kernel   -> a 24-bit key prefix and the candidate count
//   eval_collect_kernel the (few) values with that prefix -> candidate list
//   eval_select_kernel  one CTA per frame: radix select of the remaining 40
//                       bits over the candidates
// A frame whose median prefix holds more than kCandCap values (heavily
// repeated values) finishes with 8-bit radix passes over the whole map
// instead (eval_hist_kernel / eval_pick_kernel, key bytes 3..7).
// Every sum runs in a fixed order, so the statistics are deterministic; the
// histograms are exact counts.  HBM: ~57 B/px for the angle pass from fp32
// records (24 B est + 24 B gt + 1 B mask + 8 B map), + 2 x 8 B/px map reads.

#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "sn_internal.h"

namespace sn {

constexpr int kEvalChunk = 8192;  // values per chunk (one CTA)
constexpr int kEvalThreads = 256;
constexpr int kVpt = kEvalChunk / kEvalThreads;  // 32 values per thread
constexpr int kBins = 4096;                      // 12-bit histogram digits
constexpr int kPartStride = 5;                   // count, sum, min, max, M2
constexpr int64_t kCandCap = 1 << 16;            // candidate list per frame

struct EvalWs {
  double* err;       // [B][HW] angle map (NaN invalid), if the caller gave none
  double* part;      // [B][n_chunks][5]
  uint32_t* hist1;   // [B][4096] top-12-bit digit counts
  uint32_t* hist2;   // [B][4096] next 12 bits, inside the median's first digit
  uint32_t* hist;    // [B][256] fallback 8-bit radix passes
  uint64_t* prefix;  // [B] key prefix of the median
  int64_t* rank;     // [B] rank remaining inside the prefix (-1: no valid value)
  int32_t* mode;     // [B] 0 candidates, 1 fallback passes, 2 nothing to do
  uint32_t* cnt;     // [B] candidates collected
  uint64_t* cand;    // [B][cap] candidate keys
  int64_t cap;
};

// order-preserving uint64 key of a double (negatives reversed), and back
__device__ __forceinline__ uint64_t order_key(double v) {
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

__device__ __forceinline__ bool finite_v(double v) { return fabs(v) <= DBL_MAX; }

// a / b correctly rounded from y = RN(1/b): q = RN(a y) is within an ulp of
// a / b, r = a - q b is exact (FMA) and q + r y rounds to RN(a / b)
// (Markstein).  Outside 2^-500 <= |b| <= 2^500 (or for non-finite or zero b)
// the plain division is used, so no intermediate can overflow or underflow.
__device__ __forceinline__ double div_rn_by(double a, double b, double y) {
  const double ab = fabs(b);
  if (!(ab >= 3.054936363499605e-151 && ab <= 3.273390607896142e150)) return a / b;
  const double q = a * y;
  const double r = fma(-q, b, a);
  return fma(r, y, q);
}

// block-wide sum, valid in every thread (the same order in every thread)
__device__ __forceinline__ double block_sum_all(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < kEvalThreads / 32; ++w) s += red[w];
  return s;
}

// shared-memory histogram increment with the lanes that share a bin
// combined (values of one frame crowd a few exponent bins: per-lane atomics
// would serialise on them)
__device__ __forceinline__ void hist_add(uint32_t* h, bool ok, uint32_t bin) {
  const uint32_t active = __ballot_sync(0xffffffffu, ok);
  if (ok) {
    const uint32_t peers = __match_any_sync(active, bin);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[bin], (uint32_t)__popc(peers));
  }
}

// the values k0 .. k0+7 of this thread in chunk ch (NaN past the frame),
// loaded back to back: the loads are independent of the warp-synchronous
// histogram / ballot work that follows, so all eight are in flight at once
constexpr int kBatch = 8;
__device__ __forceinline__ void load_batch(const double* __restrict__ fe, int64_t HW, int ch,
                                           int k0, double (&v)[kBatch]) {
#pragma unroll
  for (int u = 0; u < kBatch; ++u) {
    const int64_t i = (int64_t)ch * kEvalChunk + (k0 + u) * kEvalThreads + threadIdx.x;
    v[u] = i < HW ? __ldcs(fe + i) : __longlong_as_double(0x7ff8000000000000ll);
  }
}

__device__ __forceinline__ void flush_hist(const uint32_t* h, uint32_t* dst) {
  for (int i = threadIdx.x; i < kBins; i += kEvalThreads)
    if (h[i]) atomicAdd(&dst[i], h[i]);
}

// SRC 0: statistics of the caller's map (err is the input); 1: angles from
// estimated normals (fp32 records / normals or fp64 normals) vs fp64 truth
template <int SRC, typename TE>
__global__ void __launch_bounds__(kEvalThreads, 4)
    eval_pass1_kernel(const TE* __restrict__ est, int est_stride, const double* __restrict__ gt,
                      const uint8_t* __restrict__ gt_mask, const uint8_t* __restrict__ extra,
                      int64_t HW, int n_chunks, double* __restrict__ err,
                      double* __restrict__ part, uint32_t* __restrict__ hist1) {
  __shared__ uint32_t h[kBins];
  __shared__ double red[kEvalThreads / 32];
  __shared__ double rmn[kEvalThreads / 32], rmx[kEvalThreads / 32];
  const int f = blockIdx.y, tid = threadIdx.x;
  const int64_t base = (int64_t)f * HW;
  for (int i = tid; i < kBins; i += kEvalThreads) h[i] = 0u;
  __syncthreads();
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  // a CTA takes chunks blockIdx.x, + gridDim.x, ... (one histogram flush)
  for (int ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
  double cnt = 0.0, sum = 0.0, mn = DBL_MAX, mx = -DBL_MAX;
  auto accumulate = [&](double v) {
    const bool ok = finite_v(v);
    if (ok) {
      cnt += 1.0;
      sum += v;
      mn = fmin(mn, v);
      mx = fmax(mx, v);
    }
    hist_add(h, ok, (uint32_t)(order_key(v) >> 52));
  };
  if (SRC == 0) {  // the caller's map: batched streaming loads
    for (int k0 = 0; k0 < kVpt; k0 += kBatch) {
      double vb[kBatch];
      load_batch(err + base, HW, ch, k0, vb);
#pragma unroll
      for (int u = 0; u < kBatch; ++u) accumulate(vb[u]);
    }
  } else {
#pragma unroll 4
  for (int k = 0; k < kVpt; ++k) {
    const int64_t i = (int64_t)ch * kEvalChunk + k * kEvalThreads + tid;
    double v = qnan;
    if (i < HW) {
      {
        const TE* e = est + (base + i) * est_stride;
        const double* g = gt + (base + i) * 3;
        const double ex = e[0], ey = e[1], ez = e[2];
        const bool ok = (ex == ex) && (ey == ey) && (ez == ez) && gt_mask[base + i] != 0 &&
                        (extra == nullptr || extra[base + i] != 0);
        if (ok) {
          const double en = sqrt(ex * ex + ey * ey + ez * ez);
          const double gn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
          // the reference's per-component divisions, correctly rounded: one
          // reciprocal per vector + Markstein's correction (div_rn_by)
          const double ye = __drcp_rn(en), yg = __drcp_rn(gn);
          const double dot = fabs(div_rn_by(ex, en, ye) * div_rn_by(g[0], gn, yg) +
                                  div_rn_by(ey, en, ye) * div_rn_by(g[1], gn, yg) +
                                  div_rn_by(ez, en, ye) * div_rn_by(g[2], gn, yg));
          // numpy's clip keeps a NaN (zero-length vector) and arccos(NaN) is NaN
          if (dot == dot) v = acos(fmin(fmax(dot, 0.0), 1.0)) * (180.0 / 3.14159265358979323846);
          if (!finite_v(v)) v = qnan;
        }
        err[base + i] = v;
      }
    }
    accumulate(v);
  }
  }
  const double c = block_sum_all(cnt, red);
  const double s = block_sum_all(sum, red);
  const double m = c > 0.0 ? s / c : 0.0;
  // squared deviations from the chunk mean: the chunk's values again (this
  // CTA just wrote / read them: L2 hits)
  double dev = 0.0;
  for (int k0 = 0; k0 < kVpt; k0 += kBatch) {
    double vb[kBatch];
    load_batch(err + base, HW, ch, k0, vb);
#pragma unroll
    for (int u = 0; u < kBatch; ++u)
      if (finite_v(vb[u])) dev += (vb[u] - m) * (vb[u] - m);
  }
  const double m2 = block_sum_all(dev, red);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, d));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
  }
  if ((tid & 31) == 0) {
    rmn[tid >> 5] = mn;
    rmx[tid >> 5] = mx;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kEvalThreads / 32; ++w) {
      mn = fmin(mn, rmn[w]);
      mx = fmax(mx, rmx[w]);
    }
    double* o = part + ((int64_t)f * n_chunks + ch) * kPartStride;
    o[0] = c;
    o[1] = s;
    o[2] = mn;
    o[3] = mx;
    o[4] = m2;
  }
  }
  __syncthreads();
  flush_hist(h, hist1 + (int64_t)f * kBins);
}

// the bin of a 4096-bin histogram holding rank r (one CTA): (bin, rank
// inside the bin), valid in every thread
__device__ __forceinline__ void find_bin(const uint32_t* hf, int64_t r, int& bin, int64_t& rin) {
  __shared__ int64_t wsum[kEvalThreads / 32];
  __shared__ int s_bin;
  __shared__ int64_t s_rin;
  constexpr int per = kBins / kEvalThreads;  // 16 bins per thread
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t mine = 0;
#pragma unroll
  for (int j = 0; j < per; ++j) mine += hf[tid * per + j];
  int64_t inc = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t u = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += u;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  int64_t before = inc - mine;
  for (int w = 0; w < warp; ++w) before += wsum[w];
  if (r >= before && r < before + mine) {
    int64_t q = r - before;
    int j = 0;
    for (; j < per - 1; ++j) {
      const int64_t c = hf[tid * per + j];
      if (q < c) break;
      q -= c;
    }
    s_bin = tid * per + j;
    s_rin = q;
  }
  __syncthreads();
  bin = s_bin;
  rin = s_rin;
}

// per frame: totals over the chunks (thread t takes chunks t, t + 256, ...,
// then a fixed-order tree: deterministic) -> stats (avg, min, max, _, std,
// count); the first median digit
__global__ void __launch_bounds__(kEvalThreads)
    eval_reduce_kernel(const double* __restrict__ part, int n_chunks,
                       const uint32_t* __restrict__ hist1, double* __restrict__ stats,
                       uint64_t* __restrict__ prefix, int64_t* __restrict__ rank,
                       int32_t* __restrict__ mode) {
  __shared__ double red[kEvalThreads / 32];
  __shared__ double rmn[kEvalThreads / 32], rmx[kEvalThreads / 32];
  const int f = blockIdx.x, tid = threadIdx.x;
  const double* pf = part + (int64_t)f * n_chunks * kPartStride;
  double c = 0.0, s = 0.0, mn = DBL_MAX, mx = -DBL_MAX;
  for (int ch = tid; ch < n_chunks; ch += kEvalThreads) {
    const double* o = pf + ch * kPartStride;
    c += o[0];
    s += o[1];
    mn = fmin(mn, o[2]);
    mx = fmax(mx, o[3]);
  }
  c = block_sum_all(c, red);
  s = block_sum_all(s, red);
  const double m = c > 0 ? s / c : 0.0;
  double m2 = 0.0;  // Chan et al.: within-chunk + between-chunk squared deviations
  for (int ch = tid; ch < n_chunks; ch += kEvalThreads) {
    const double* o = pf + ch * kPartStride;
    if (o[0] > 0.0) {
      const double dm = o[1] / o[0] - m;
      m2 += o[4] + o[0] * dm * dm;
    }
  }
  m2 = block_sum_all(m2, red);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, d));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
  }
  if ((tid & 31) == 0) {
    rmn[tid >> 5] = mn;
    rmx[tid >> 5] = mx;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kEvalThreads / 32; ++w) {
      mn = fmin(mn, rmn[w]);
      mx = fmax(mx, rmx[w]);
    }
    const double qnan = __longlong_as_double(0x7ff8000000000000ll);
    double* st = stats + (int64_t)f * 6;
    st[0] = c > 0 ? s / c : qnan;
    st[1] = c > 0 ? mn : qnan;
    st[2] = c > 0 ? mx : qnan;
    st[3] = qnan;
    st[4] = c > 0 ? sqrt(m2 / c) : qnan;
    st[5] = c;
  }
  if (c <= 0.0) {
    if (tid == 0) {
      rank[f] = -1;
      mode[f] = 2;
    }
    return;
  }
  int bin;
  int64_t rin;
  find_bin(hist1 + (int64_t)f * kBins, (int64_t)((c - 1) / 2), bin, rin);  // lower middle
  if (tid == 0) {
    prefix[f] = (uint64_t)bin << 52;
    rank[f] = rin;
    mode[f] = 0;
  }
}

__global__ void __launch_bounds__(kEvalThreads)
    eval_hist2_kernel(const double* __restrict__ err, int64_t HW, int n_chunks,
                      const uint64_t* __restrict__ prefix, const int32_t* __restrict__ mode,
                      uint32_t* __restrict__ hist2) {
  __shared__ uint32_t h[kBins];
  const int f = blockIdx.y, tid = threadIdx.x;
  if (mode[f] == 2) return;
  for (int i = tid; i < kBins; i += kEvalThreads) h[i] = 0u;
  __syncthreads();
  const uint64_t d1 = prefix[f] >> 52;
  const int64_t base = (int64_t)f * HW;
  int any = 0;
  for (int ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
    for (int k0 = 0; k0 < kVpt; k0 += kBatch) {
      double v[kBatch];
      load_batch(err + base, HW, ch, k0, v);
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const uint64_t key = order_key(v[u]);
        const bool take = finite_v(v[u]) && (key >> 52) == d1;
        any |= take;
        hist_add(h, take, (uint32_t)(key >> 40) & 0xfffu);
      }
    }
  }
  if (__syncthreads_or(any)) flush_hist(h, hist2 + (int64_t)f * kBins);
}

__global__ void __launch_bounds__(kEvalThreads)
    eval_pick2_kernel(const uint32_t* __restrict__ hist2, int64_t cap,
                      uint64_t* __restrict__ prefix, int64_t* __restrict__ rank,
                      int32_t* __restrict__ mode, uint32_t* __restrict__ cnt) {
  const int f = blockIdx.x;
  if (mode[f] == 2) return;
  int bin;
  int64_t rin;
  const uint32_t* hf = hist2 + (int64_t)f * kBins;
  find_bin(hf, rank[f], bin, rin);
  if (threadIdx.x == 0) {
    prefix[f] |= (uint64_t)bin << 40;
    rank[f] = rin;
    mode[f] = (int64_t)hf[bin] <= cap ? 0 : 1;
    cnt[f] = 0u;
  }
}

__global__ void __launch_bounds__(kEvalThreads)
    eval_collect_kernel(const double* __restrict__ err, int64_t HW, int n_chunks,
                        const uint64_t* __restrict__ prefix, const int32_t* __restrict__ mode,
                        uint32_t* __restrict__ cnt, uint64_t* __restrict__ cand, int64_t cap) {
  const int f = blockIdx.y, tid = threadIdx.x, lane = tid & 31;
  if (mode[f] != 0) return;
  const uint64_t p24 = prefix[f] >> 40;
  const int64_t base = (int64_t)f * HW;
  uint64_t* cf = cand + (int64_t)f * cap;
  for (int ch = blockIdx.x; ch < n_chunks; ch += gridDim.x)
    for (int k0 = 0; k0 < kVpt; k0 += kBatch) {
      double v[kBatch];
      load_batch(err + base, HW, ch, k0, v);
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
    const uint64_t key = order_key(v[u]);
    const bool take = finite_v(v[u]) && (key >> 40) == p24;
    const uint32_t b = __ballot_sync(0xffffffffu, take);
    if (b) {  // one atomic per warp
      const int leader = __ffs(b) - 1;
      uint32_t at = 0;
      if (lane == leader) at = atomicAdd(&cnt[f], (uint32_t)__popc(b));
      at = __shfl_sync(0xffffffffu, at, leader);
      if (take) cf[at + __popc(b & ((1u << lane) - 1u))] = key;
    }
      }
    }
}

// one CTA per frame: radix select of key bits 39..0 over the candidates
__global__ void __launch_bounds__(kEvalThreads)
    eval_select_kernel(const uint64_t* __restrict__ cand, int64_t cap,
                       const uint32_t* __restrict__ cnt, const int32_t* __restrict__ mode,
                       const uint64_t* __restrict__ prefix, const int64_t* __restrict__ rank,
                       double* __restrict__ stats) {
  __shared__ uint32_t h[256];
  __shared__ uint64_t s_pre;
  __shared__ int64_t s_rank;
  const int f = blockIdx.x, tid = threadIdx.x;
  if (mode[f] != 0) return;
  const uint64_t* cf = cand + (int64_t)f * cap;
  const int n = (int)cnt[f];
  if (tid == 0) {
    s_pre = prefix[f];
    s_rank = rank[f];
  }
  for (int shift = 32; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += kEvalThreads) h[i] = 0u;
    __syncthreads();
    const uint64_t pre = s_pre;
    const uint64_t hi_mask = ~0ull << (shift + 8);
    for (int i = tid; i < n; i += kEvalThreads) {
      const uint64_t key = cf[i];
      if ((key & hi_mask) == pre) atomicAdd(&h[(key >> shift) & 0xff], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      int64_t r = s_rank;
      int dgt = 0;
      for (; dgt < 255; ++dgt) {
        if (r < (int64_t)h[dgt]) break;
        r -= h[dgt];
      }
      s_pre = pre | ((uint64_t)dgt << shift);
      s_rank = r;
    }
    __syncthreads();
  }
  if (tid == 0) stats[(int64_t)f * 6 + 3] = key_value(s_pre);
}

// fallback: 8-bit radix passes over the whole map for key byte `pass` (3..7)
__global__ void __launch_bounds__(kEvalThreads)
    eval_hist_kernel(const double* __restrict__ err, int64_t HW, int pass,
                     const uint64_t* __restrict__ prefix, const int32_t* __restrict__ mode,
                     uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  const int f = blockIdx.y, ch = blockIdx.x;
  if (mode[f] != 1) return;
  for (int i = threadIdx.x; i < 256; i += kEvalThreads) h[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)f * HW;
  const int shift = 56 - 8 * pass;
  const uint64_t pre = prefix[f];
  const uint64_t hi_mask = ~0ull << (64 - 8 * pass);
  for (int64_t i = (int64_t)ch * kEvalChunk + threadIdx.x;
       i < min((int64_t)(ch + 1) * kEvalChunk, HW); i += kEvalThreads) {
    const double v = err[base + i];
    if (!finite_v(v)) continue;
    const uint64_t b = order_key(v);
    if ((b & hi_mask) == pre) atomicAdd(&h[(b >> shift) & 0xff], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += kEvalThreads)
    if (h[i]) atomicAdd(&hist[f * 256 + i], h[i]);
}

__global__ void eval_pick_kernel(int pass, uint64_t* __restrict__ prefix,
                                 int64_t* __restrict__ rank, const int32_t* __restrict__ mode,
                                 uint32_t* __restrict__ hist, double* __restrict__ stats) {
  const int f = blockIdx.x;
  if (threadIdx.x != 0 || mode[f] != 1) return;
  uint32_t* hf = hist + f * 256;
  int64_t r = rank[f];
  int dgt = 0;
  for (; dgt < 255; ++dgt) {
    if (r < (int64_t)hf[dgt]) break;
    r -= hf[dgt];
  }
  prefix[f] |= (uint64_t)dgt << (56 - 8 * pass);
  rank[f] = r;
  if (pass == 7) stats[(int64_t)f * 6 + 3] = key_value(prefix[f]);
  for (int i = 0; i < 256; ++i) hf[i] = 0;
}

static int64_t cand_cap(int64_t HW) { return HW < kCandCap ? HW : kCandCap; }

size_t eval_workspace_bytes(int64_t B, int64_t H, int64_t W) {
  const int64_t HW = H * W;
  const int64_t nch = (HW + kEvalChunk - 1) / kEvalChunk;
  auto a = [](size_t v) { return (v + 255) / 256 * 256; };
  return a((size_t)(B * HW) * 8) + a((size_t)(B * nch * kPartStride) * 8) +
         2 * a((size_t)B * kBins * 4) + a((size_t)B * 256 * 4) + 2 * a((size_t)B * 8) +
         2 * a((size_t)B * 4) + a((size_t)(B * cand_cap(HW)) * 8);
}

int run_eval(const LaunchCtx& ctx, const float* est, const double* est_d, int est_stride,
             const double* gt, const uint8_t* gt_mask, const uint8_t* extra, int64_t B, int64_t H,
             int64_t W, double* err_out, double* stats, void* workspace, size_t ws_bytes) {
  const int64_t HW = H * W;
  if (B == 0) return SN_OK;
  if (!workspace || ws_bytes < eval_workspace_bytes(B, H, W))
    return set_error(SN_EINVAL, "evaluation workspace too small");
  if (B > 65535) {  // grid.y: consecutive calls of <= 65535 frames reusing the workspace
    for (int64_t f0 = 0; f0 < B; f0 += 65535) {
      const int64_t b = B - f0 < 65535 ? B - f0 : 65535;
      const int64_t o = f0 * HW;
      const int rc = run_eval(ctx, est ? est + o * est_stride : nullptr,
                              est_d ? est_d + o * est_stride : nullptr, est_stride,
                              gt ? gt + o * 3 : nullptr, gt_mask ? gt_mask + o : nullptr,
                              extra ? extra + o : nullptr, b, H, W, err_out ? err_out + o : nullptr,
                              stats + f0 * 6, workspace, ws_bytes);
      if (rc) return rc;
    }
    return SN_OK;
  }
  const int64_t nch64 = (HW + kEvalChunk - 1) / kEvalChunk;
  if (nch64 > 0x7fffffffLL || nch64 == 0) return set_error(SN_EINVAL, "bad frame size");
  const int nch = (int)nch64;
  auto a = [](size_t v) { return (v + 255) / 256 * 256; };
  uint8_t* q = static_cast<uint8_t*>(workspace);
  EvalWs ws;
  ws.cap = cand_cap(HW);
  ws.err = reinterpret_cast<double*>(q);
  q += a((size_t)(B * HW) * 8);
  ws.part = reinterpret_cast<double*>(q);
  q += a((size_t)(B * nch * kPartStride) * 8);
  uint8_t* hists = q;
  ws.hist1 = reinterpret_cast<uint32_t*>(q);
  q += a((size_t)B * kBins * 4);
  ws.hist2 = reinterpret_cast<uint32_t*>(q);
  q += a((size_t)B * kBins * 4);
  ws.hist = reinterpret_cast<uint32_t*>(q);
  q += a((size_t)B * 256 * 4);
  const size_t hist_bytes = (size_t)(q - hists);  // the three histograms: one memset
  ws.prefix = reinterpret_cast<uint64_t*>(q);
  q += a((size_t)B * 8);
  ws.rank = reinterpret_cast<int64_t*>(q);
  q += a((size_t)B * 8);
  ws.mode = reinterpret_cast<int32_t*>(q);
  q += a((size_t)B * 4);
  ws.cnt = reinterpret_cast<uint32_t*>(q);
  q += a((size_t)B * 4);
  ws.cand = reinterpret_cast<uint64_t*>(q);
  double* err = err_out ? err_out : ws.err;
  if (cudaMemsetAsync(hists, 0, hist_bytes, ctx.stream) != cudaSuccess)
    return set_cuda_error("cudaMemsetAsync(eval histograms)");
  // one CTA per chunk (measured: folding several chunks into a CTA to save
  // histogram flushes was slower -- fewer resident CTAs to hide latency)
  dim3 grid((unsigned)nch, (unsigned)B);
  dim3 grid_all = grid;
  if (!est && !est_d)  // statistics of the map the caller passed in err_out
    eval_pass1_kernel<0, double><<<grid, kEvalThreads, 0, ctx.stream>>>(
        nullptr, 3, nullptr, nullptr, nullptr, HW, nch, err, ws.part, ws.hist1);
  else if (est_d)
    eval_pass1_kernel<1, double><<<grid, kEvalThreads, 0, ctx.stream>>>(
        est_d, est_stride, gt, gt_mask, extra, HW, nch, err, ws.part, ws.hist1);
  else
    eval_pass1_kernel<1, float><<<grid, kEvalThreads, 0, ctx.stream>>>(
        est, est_stride, gt, gt_mask, extra, HW, nch, err, ws.part, ws.hist1);
  int rc = check_launch("eval_pass1_kernel");
  if (rc) return rc;
  eval_reduce_kernel<<<(unsigned)B, kEvalThreads, 0, ctx.stream>>>(
      ws.part, nch, ws.hist1, stats, ws.prefix, ws.rank, ws.mode);
  if ((rc = check_launch("eval_reduce_kernel"))) return rc;
  eval_hist2_kernel<<<grid, kEvalThreads, 0, ctx.stream>>>(err, HW, nch, ws.prefix, ws.mode,
                                                           ws.hist2);
  if ((rc = check_launch("eval_hist2_kernel"))) return rc;
  eval_pick2_kernel<<<(unsigned)B, kEvalThreads, 0, ctx.stream>>>(ws.hist2, ws.cap, ws.prefix,
                                                                  ws.rank, ws.mode, ws.cnt);
  if ((rc = check_launch("eval_pick2_kernel"))) return rc;
  eval_collect_kernel<<<grid, kEvalThreads, 0, ctx.stream>>>(err, HW, nch, ws.prefix, ws.mode,
                                                             ws.cnt, ws.cand, ws.cap);
  if ((rc = check_launch("eval_collect_kernel"))) return rc;
  eval_select_kernel<<<(unsigned)B, kEvalThreads, 0, ctx.stream>>>(
      ws.cand, ws.cap, ws.cnt, ws.mode, ws.prefix, ws.rank, stats);
  if ((rc = check_launch("eval_select_kernel"))) return rc;
  for (int pass = 3; pass < 8; ++pass) {  // frames whose median prefix is crowded
    eval_hist_kernel<<<grid_all, kEvalThreads, 0, ctx.stream>>>(err, HW, pass, ws.prefix, ws.mode,
                                                            ws.hist);
    if ((rc = check_launch("eval_hist_kernel"))) return rc;
    eval_pick_kernel<<<(unsigned)B, 32, 0, ctx.stream>>>(pass, ws.prefix, ws.rank, ws.mode,
                                                         ws.hist, stats);
    if ((rc = check_launch("eval_pick_kernel"))) return rc;
  }
  return SN_OK;
}

}  // namespace sn
