// Oriented point cloud compaction for sm_100a.
//
// Reference: cli.py:118-123 keeps pixels with a valid normal and a finite
// point (keep = normals.mask & isfinite(pts)) and writes them in raster order
// as binary-PLY vertices (x, y, z, nx, ny, nz) float32 (formats.py:170-185).
// A valid normal implies d finite and > 0, hence a finite reference point,
// so keep = the normal mask the fused pass emits.  The dense [B][H][W][6]
// record is already the vertex layout; compaction is a stable stream
// compaction of 24-byte records over the whole batch in raster order:
//   1. cloud_count_kernel    per 2048-pixel block: popcount of the mask
//   2. cloud_scan_kernel     exclusive scan of the block counts (one CTA)
//   3. cloud_scatter_kernel  warp ballots give each kept pixel its slot;
//                            records are copied as 3 x 8-byte words
// Frame f's vertices start at offsets[f] (= the scan at its first block);
// offsets[B] is the total.

#include <cuda_runtime.h>
#include <stdint.h>

#include "sn_internal.h"

namespace sn {

constexpr int kCloudBlock = 2048;  // pixels per count block (blocks tile each frame separately)
constexpr int kCloudThreads = 256;

// blocks never straddle frames: frame f owns blocks [f*bpf, (f+1)*bpf)
__global__ void __launch_bounds__(kCloudThreads)
    cloud_count_kernel(const uint8_t* __restrict__ mask, int64_t HW, int bpf, int64_t n_blocks,
                       int64_t* __restrict__ counts) {
  __shared__ int warp_cnt[kCloudThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t blk = blockIdx.x; blk < n_blocks; blk += gridDim.x) {
    const int64_t f = blk / bpf;
    const int64_t p0 = (blk - f * bpf) * kCloudBlock;
    const uint8_t* m = mask + f * HW;
    int c = 0;
    if (p0 + kCloudBlock <= HW && (reinterpret_cast<uintptr_t>(m + p0) & 7u) == 0) {
      // 8 mask bytes per thread: nonzero bytes by a SIMD compare, then popc
      static_assert(kCloudBlock == kCloudThreads * 8, "one uint2 per thread");
      const uint2 w = reinterpret_cast<const uint2*>(m + p0)[tid];
      c = (__popc(__vcmpne4(w.x, 0u)) + __popc(__vcmpne4(w.y, 0u))) >> 3;
    } else {
      for (int i = tid; i < kCloudBlock; i += kCloudThreads) {
        const int64_t px = p0 + i;
        c += (px < HW && m[px] != 0) ? 1 : 0;
      }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
    if (lane == 0) warp_cnt[warp] = c;
    __syncthreads();
    if (tid == 0) {
      int s = 0;
      for (int w = 0; w < kCloudThreads / 32; ++w) s += warp_cnt[w];
      counts[blk] = s;
    }
    __syncthreads();
  }
}

// in-place exclusive scan of counts[0 .. n) with one CTA; counts[n] = total
__global__ void __launch_bounds__(1024) cloud_scan_kernel(int64_t* __restrict__ counts, int64_t n) {
  __shared__ int64_t warp_sum[32];
  __shared__ int64_t carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += 1024) {
    const int64_t i = base + tid;
    const int64_t v = i < n ? counts[i] : 0;
    int64_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += u;
    }
    if (lane == 31) warp_sum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      int64_t ws = warp_sum[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, ws, d);
        if (lane >= d) ws += u;
      }
      warp_sum[lane] = ws;  // inclusive over warps
    }
    __syncthreads();
    const int64_t before = carry + (warp > 0 ? warp_sum[warp - 1] : 0);
    if (i < n) counts[i] = before + inc - v;
    __syncthreads();
    if (tid == 1023) carry = before + inc;
    __syncthreads();
  }
  if (tid == 0) counts[n] = carry;
}

// each warp owns a contiguous 256-pixel segment of the 2048-pixel block: it
// counts its segment (8 ballots), one block-wide exclusive scan of the 8
// warp counts gives its start, then it scatters its segment alone (ballot +
// popc per 32 pixels) -- one CTA barrier per block instead of two per 256
// pixels
constexpr int kSegPx = kCloudBlock / (kCloudThreads / 32);  // 256

__global__ void __launch_bounds__(kCloudThreads)
    cloud_scatter_kernel(const float* __restrict__ out6, const uint8_t* __restrict__ mask,
                         int64_t HW, int bpf, int64_t n_blocks, const int64_t* __restrict__ starts,
                         float* __restrict__ cloud, int64_t capacity) {
  __shared__ int warp_cnt[kCloudThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t blk = blockIdx.x; blk < n_blocks; blk += gridDim.x) {
    const int64_t f = blk / bpf;
    const int64_t s0 = (blk - f * bpf) * kCloudBlock + warp * kSegPx;  // segment start in the frame
    const uint8_t* m = mask + f * HW;
    uint32_t bal[kSegPx / 32];
    int c = 0;
#pragma unroll
    for (int r = 0; r < kSegPx / 32; ++r) {
      const int64_t px = s0 + r * 32 + lane;
      bal[r] = __ballot_sync(0xffffffffu, px < HW && m[px] != 0);
      c += __popc(bal[r]);
    }
    if (lane == 0) warp_cnt[warp] = c;
    __syncthreads();
    int64_t next = starts[blk];
    for (int w = 0; w < warp; ++w) next += warp_cnt[w];
    __syncthreads();  // warp_cnt is rewritten by the next block
#pragma unroll
    for (int r = 0; r < kSegPx / 32; ++r) {
      const uint32_t b = bal[r];
      if (b == 0xffffffffu && next + 32 <= capacity) {
        // 32 kept pixels in a row: one contiguous 768-byte copy, lanes on
        // consecutive 8-byte words (every access fully coalesced; records
        // are 8-byte aligned at both ends)
        const float2* src = reinterpret_cast<const float2*>(out6 + (f * HW + s0 + r * 32) * 6);
        float2* dst = reinterpret_cast<float2*>(cloud + next * 6);
        const float2 a0 = src[lane], a1 = src[lane + 32], a2 = src[lane + 64];
        dst[lane] = a0;
        dst[lane + 32] = a1;
        dst[lane + 64] = a2;
      } else if ((b >> lane) & 1u) {
        const int64_t px = s0 + r * 32 + lane;
        const int64_t slot = next + __popc(b & ((1u << lane) - 1u));
        if (slot < capacity) {
          const float2* src = reinterpret_cast<const float2*>(out6 + (f * HW + px) * 6);
          float2* dst = reinterpret_cast<float2*>(cloud + slot * 6);
          const float2 a0 = src[0], a1 = src[1], a2 = src[2];
          dst[0] = a0;
          dst[1] = a1;
          dst[2] = a2;
        }
      }
      next += __popc(b);
    }
  }
}

size_t cloud_workspace_bytes(int64_t B, int64_t H, int64_t W) {
  const int64_t bpf = (H * W + kCloudBlock - 1) / kCloudBlock;
  return (size_t)(B * bpf + 1) * sizeof(int64_t);
}

int run_cloud_count(const LaunchCtx& ctx, const uint8_t* mask, int64_t B, int64_t H, int64_t W,
                    int64_t* frame_offsets, void* workspace, size_t ws_bytes) {
  const int64_t HW = H * W;
  if (B * HW == 0) {
    return cudaMemsetAsync(frame_offsets, 0, (size_t)(B + 1) * sizeof(int64_t), ctx.stream) ==
                   cudaSuccess
               ? SN_OK
               : set_cuda_error("cudaMemsetAsync(frame offsets)");
  }
  if (!workspace || ws_bytes < cloud_workspace_bytes(B, H, W))
    return set_error(SN_EINVAL, "compaction workspace too small");
  const int64_t bpf64 = (HW + kCloudBlock - 1) / kCloudBlock;
  if (bpf64 > 0x7fffffffLL) return set_error(SN_EINVAL, "frame too large");
  const int bpf = (int)bpf64;
  const int64_t n_blocks = B * bpf64;
  int64_t* counts = static_cast<int64_t*>(workspace);
  int64_t grid = n_blocks;
  if (grid > (int64_t)ctx.num_sms * 16) grid = (int64_t)ctx.num_sms * 16;
  cloud_count_kernel<<<(unsigned)grid, kCloudThreads, 0, ctx.stream>>>(mask, HW, bpf, n_blocks,
                                                                      counts);
  int rc = check_launch("cloud_count_kernel");
  if (rc) return rc;
  cloud_scan_kernel<<<1, 1024, 0, ctx.stream>>>(counts, n_blocks);
  if ((rc = check_launch("cloud_scan_kernel"))) return rc;
  // frame offsets: the scan at each frame's first block, and the total
  if (cudaMemcpy2DAsync(frame_offsets, sizeof(int64_t), counts, (size_t)bpf * sizeof(int64_t),
                        sizeof(int64_t), (size_t)B, cudaMemcpyDeviceToDevice,
                        ctx.stream) != cudaSuccess ||
      cudaMemcpyAsync(frame_offsets + B, counts + n_blocks, sizeof(int64_t),
                      cudaMemcpyDeviceToDevice, ctx.stream) != cudaSuccess)
    return set_cuda_error("frame offsets copy");
  return SN_OK;
}

int run_cloud_scatter(const LaunchCtx& ctx, const float* out6, const uint8_t* mask, int64_t B,
                      int64_t H, int64_t W, float* cloud, int64_t capacity, void* workspace,
                      size_t ws_bytes) {
  const int64_t HW = H * W;
  if (B * HW == 0 || capacity == 0) return SN_OK;
  if (!workspace || ws_bytes < cloud_workspace_bytes(B, H, W))
    return set_error(SN_EINVAL, "compaction workspace too small");
  const int64_t bpf64 = (HW + kCloudBlock - 1) / kCloudBlock;
  if (bpf64 > 0x7fffffffLL) return set_error(SN_EINVAL, "frame too large");
  const int bpf = (int)bpf64;
  const int64_t n_blocks = B * bpf64;
  int64_t grid = n_blocks;
  if (grid > (int64_t)ctx.num_sms * 16) grid = (int64_t)ctx.num_sms * 16;
  cloud_scatter_kernel<<<(unsigned)grid, kCloudThreads, 0, ctx.stream>>>(
      out6, mask, HW, bpf, n_blocks, static_cast<const int64_t*>(workspace), cloud, capacity);
  return check_launch("cloud_scatter_kernel");
}

int run_compact_cloud(const LaunchCtx& ctx, const float* out6, const uint8_t* mask, int64_t B,
                      int64_t H, int64_t W, float* cloud, int64_t capacity,
                      int64_t* frame_offsets, void* workspace, size_t ws_bytes) {
  const int rc = run_cloud_count(ctx, mask, B, H, W, frame_offsets, workspace, ws_bytes);
  if (rc) return rc;
  return run_cloud_scatter(ctx, out6, mask, B, H, W, cloud, capacity, workspace, ws_bytes);
}

}  // namespace sn
