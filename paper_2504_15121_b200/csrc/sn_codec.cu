// Device input codecs for sm_100a.
//
// The reference decodes its disparity files on the host (formats.py):
//   * 16-bit PNG  (formats.py:133-150): d = (raw - 1.0) / scale in fp64,
//     raw == invalid_value -> NaN (masked);
//   * PFM         (formats.py:84-102): 4-byte floats, little-endian when the
//     header scale is negative, else big-endian, rows stored bottom-up;
//     1 ('Pf') or 3 ('PF') channels.
// Here the compressed container (zlib / header parsing) stays on the host and
// the per-sample work runs on the device over the raw payload after one H2D
// copy of 2 (PNG16) or 4 (PFM) bytes per sample:
//   dequant_png16_kernel  uint16 -> fp32 and/or fp64 disparity (bit-exact fp64,
//                         fp32 = that value rounded once)
//   decode_pfm_kernel     byte swap + vertical flip, 16-byte words when rows
//                         are 16-byte multiples
// Both are pure streaming kernels: HBM-bound at 2 + 4|8 (PNG16) and 4 + 4
// (PFM) bytes per sample.  The fused oriented-point pass also reads PNG16
// payloads directly (sn_oriented_points_png16, sn_fixed.cu), skipping the
// dequantised copy.

#include <cuda_runtime.h>
#include <stdint.h>

#include "sn_internal.h"

namespace sn {

// 8 samples (16 B) per thread when the buffer is 16-B aligned and n % 8 == 0
template <bool VEC>
__global__ void __launch_bounds__(256)
    dequant_png16_kernel(const uint16_t* __restrict__ raw, int64_t n, int invalid, double scale,
                         double rcp, float* __restrict__ out32, double* __restrict__ out64) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (VEC) {
    const int64_t n8 = n / 8;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
      const uint4 w = __ldcs(reinterpret_cast<const uint4*>(raw) + i);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      double v[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[2 * k] = png16_value(ws[k] & 0xffffu, invalid, scale, rcp);
        v[2 * k + 1] = png16_value(ws[k] >> 16, invalid, scale, rcp);
      }
      if (out32) {
        float4* o = reinterpret_cast<float4*>(out32 + i * 8);
        __stcs(o, make_float4((float)v[0], (float)v[1], (float)v[2], (float)v[3]));
        __stcs(o + 1, make_float4((float)v[4], (float)v[5], (float)v[6], (float)v[7]));
      }
      if (out64) {
        double2* o = reinterpret_cast<double2*>(out64 + i * 8);
#pragma unroll
        for (int k = 0; k < 4; ++k) __stcs(o + k, make_double2(v[2 * k], v[2 * k + 1]));
      }
    }
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      const double v = png16_value(raw[i], invalid, scale, rcp);
      if (out32) out32[i] = (float)v;
      if (out64) out64[i] = v;
    }
  }
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// payload: B images of H rows x L words (L = W * channels), bottom row first.
// Output row y of image b = payload row H-1-y, byte-swapped when big-endian.
template <bool VEC>
__global__ void __launch_bounds__(256)
    decode_pfm_kernel(const uint32_t* __restrict__ payload, int64_t B, int64_t H, int64_t L,
                      bool big_endian, uint32_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (VEC) {
    const int64_t L4 = L / 4, n4 = B * H * L4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
      const int64_t row = i / L4, c = i - row * L4;  // row = b * H + y
      const int64_t b = row / H, y = row - b * H;
      uint4 w = __ldcs(reinterpret_cast<const uint4*>(payload) + ((b * H + (H - 1 - y)) * L4 + c));
      if (big_endian) w = make_uint4(bswap32(w.x), bswap32(w.y), bswap32(w.z), bswap32(w.w));
      __stcs(reinterpret_cast<uint4*>(out) + i, w);
    }
  } else {
    const int64_t n = B * H * L;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      const int64_t row = i / L, c = i - row * L;
      const int64_t b = row / H, y = row - b * H;
      uint32_t w = payload[(b * H + (H - 1 - y)) * L + c];
      out[i] = big_endian ? bswap32(w) : w;
    }
  }
}

static unsigned stream_grid(const LaunchCtx& ctx, int64_t items) {
  int64_t g = (items + 255) / 256;
  const int64_t cap = (int64_t)ctx.num_sms * 8;  // 8 x 256 threads per SM
  if (g > cap) g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

int run_dequant_png16(const LaunchCtx& ctx, const uint16_t* raw, int64_t n, int invalid,
                      double scale, float* out32, double* out64) {
  if (n == 0) return SN_OK;
  const double rcp = png16_rcp(scale);
  const bool vec = n % 8 == 0 && reinterpret_cast<uintptr_t>(raw) % 16 == 0 &&
                   (!out32 || reinterpret_cast<uintptr_t>(out32) % 16 == 0) &&
                   (!out64 || reinterpret_cast<uintptr_t>(out64) % 16 == 0);
  if (vec)
    dequant_png16_kernel<true><<<stream_grid(ctx, n / 8), 256, 0, ctx.stream>>>(
        raw, n, invalid, scale, rcp, out32, out64);
  else
    dequant_png16_kernel<false><<<stream_grid(ctx, n), 256, 0, ctx.stream>>>(
        raw, n, invalid, scale, rcp, out32, out64);
  return check_launch("dequant_png16_kernel");
}

int run_decode_pfm(const LaunchCtx& ctx, const void* payload, int64_t B, int64_t H, int64_t L,
                   bool big_endian, float* out) {
  if (B * H * L == 0) return SN_OK;
  const auto* in = static_cast<const uint32_t*>(payload);
  auto* o = reinterpret_cast<uint32_t*>(out);
  const bool vec = L % 4 == 0 && reinterpret_cast<uintptr_t>(payload) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(out) % 16 == 0;
  if (vec)
    decode_pfm_kernel<true><<<stream_grid(ctx, B * H * L / 4), 256, 0, ctx.stream>>>(
        in, B, H, L, big_endian, o);
  else
    decode_pfm_kernel<false><<<stream_grid(ctx, B * H * L), 256, 0, ctx.stream>>>(
        in, B, H, L, big_endian, o);
  return check_launch("decode_pfm_kernel");
}

}  // namespace sn
