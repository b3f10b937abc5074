// Host-side internals shared by the C-ABI translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "sn_b200.h"
#include "sn_common.cuh"

namespace sn {

struct LaunchCtx {
  cudaStream_t stream;
  int device;
  int num_sms;
};

// error plumbing (thread-local message, see sn_api.cu)
int set_error(int code, const char* fmt, ...);
int set_cuda_error(const char* what);
int check_launch(const char* what);
// cudaFuncAttributeMaxDynamicSharedMemorySize is per device: set once per
// (kernel, device) pair, under a lock (the caller has made `device` current)
int ensure_dyn_smem(const void* func, int bytes, int device, const char* name);
// resident blocks per SM of a kernel launch shape, queried once per device
int occupancy_per_sm(const void* func, int threads, size_t smem, int device);
// stream-ordered scratch from the library's private per-device pool
int scratch_alloc(const LaunchCtx& ctx, size_t bytes, void** ptr);
void scratch_free(const LaunchCtx& ctx, void* ptr);

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
int encode_tiled(CUtensorMap* map, CUtensorMapDataType dt, int rank, void* gaddr,
                 const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                 const cuuint32_t* elem_strides, CUtensorMapSwizzle swizzle,
                 CUtensorMapFloatOOBfill oob);

constexpr int kMaxOffsets = 1024;
struct OffsetTable {
  int n;
  int2 v[kMaxOffsets];
};

template <typename T>
int run_fixed(const LaunchCtx& ctx, const T* disp, const FixedParams& p, const sn_moments_t& m,
              const OffsetTable& tab, float* out6, uint8_t* mask, double* a1, double* a2,
              bool affine, int force_generic);

template <typename T>
int run_fixed_strided(const LaunchCtx& ctx, const T* disp, int64_t ld, const FixedParams& p,
                      const sn_moments_t& m, const OffsetTable& tab, float* out6, uint8_t* mask);

struct CclParams {
  int64_t B, H, W;
  double fxb;       // fx * b in Python's double order (geometry.py:43)
  double t;         // ST threshold
  float fxb_f;      // fp32(fxb) for the filtered predicate
  float t_f;        // fp32(t)
  int exact_only;   // fxb outside the filter's range: every pixel takes the fp64 path
};

CclParams make_ccl_params(int64_t B, int64_t H, int64_t W, double fxb, double t);
// labeller workspace of B frames; from kCclSplitFrames frames on it also holds
// two half-batch workspaces (labels from disparities run the halves on two
// streams, sn_api.cu ccl_labels_ws_impl)
constexpr int64_t kCclSplitFrames = 128;
size_t ccl_workspace_bytes(int64_t B, int64_t H, int64_t W);
size_t ccl_workspace_bytes_one(int64_t B, int64_t H, int64_t W);  // one batch, no split

// T = float or double disparities (explicit instantiations in sn_ccl.cu)
template <typename T>
int run_passable(const LaunchCtx& ctx, const T* disp, const CclParams& p, uint8_t* passable,
                 double* edges);
template <typename T>
int run_ccl(const LaunchCtx& ctx, const T* disp, const uint8_t* passable, const CclParams& p,
            int64_t index_base, int32_t* labels, void* workspace, size_t ws_bytes,
            const uint32_t* bits_in = nullptr);
template <typename T>
int run_passable_bits(const LaunchCtx& ctx, const T* disp, const FixedParams& p,
                      uint32_t* bits);
// host-side fill of the predicate fields of FixedParams
void fill_predicate(FixedParams& p, double fxb, double t, uint32_t* bits);
int run_seam_merge(const LaunchCtx& ctx, const int32_t* seams, int n_strips, int64_t W,
                   int32_t* table, int64_t table_n);
int run_relabel_table(const LaunchCtx& ctx, int32_t* labels, int64_t n, const int32_t* table,
                      int64_t table_n);
int run_relabel(const LaunchCtx& ctx, int32_t* labels, int64_t n, int64_t base,
                const int32_t* keys, const int32_t* vals, const int32_t* n_map, int32_t cap,
                int32_t* scratch);

// adaptive star-fill (sn_adaptive.cu)
constexpr int kStarMaxRays = 64, kStarMaxSteps = 2048, kStarKeyWords = 16;
constexpr int kStarMaxKeys = kStarKeyWords * 32;  // 512 distinct offsets
struct StarTable {
  int n_rays, n_keys;
  int wide;                         // moment sums may exceed int32: 64-bit accumulation
  int reach;                        // max |x|, |y| over the offsets
  int ray_start[kStarMaxRays + 1];  // steps of ray j: [ray_start[j], ray_start[j+1])
  int16_t step_key[kStarMaxSteps];  // key of each step
  int32_t step_xy[kStarMaxSteps];   // offset of each step: x in the low, y in the high 16 bits
  int32_t step_lin[kStarMaxSteps];  // y * W + x of each step
  int32_t key_xy[kStarMaxKeys];     // keys in first-occurrence order (packed like step_xy)
  int32_t key_lin[kStarMaxKeys];
};
struct AdaptiveParams {
  FixedParams fp;     // rig, shape, point constants (bits / bits_ww for ST)
  double threshold;   // t (ST) or k (CD)
  double baseline;
  double fxfx;        // fx * fx (Python double, geometry.py:197)
  double nfxfy;       // -fx * fy (geometry.py:199)
  int shared_range;
};
size_t adaptive_workspace_bytes(int64_t B, int64_t H, int64_t W);
template <typename T>
int run_adaptive(const LaunchCtx& ctx, const T* disp, const AdaptiveParams& ap,
                 const StarTable& tab, int stop, float* out6, uint8_t* mask, void* workspace,
                 size_t ws_bytes);

size_t eval_workspace_bytes(int64_t B, int64_t H, int64_t W);
int run_eval(const LaunchCtx& ctx, const float* est, const double* est_d, int est_stride,
             const double* gt,
             const uint8_t* gt_mask, const uint8_t* extra, int64_t B, int64_t H, int64_t W,
             double* err_out, double* stats, void* workspace, size_t ws_bytes);

// RN(1/scale) for png16_value's fast division, 0 (divide) outside
// 2^-100 <= |scale| <= 2^100
inline double png16_rcp(double scale) {
  const double a = scale < 0 ? -scale : scale;
  return (a >= 7.888609052210118e-31 && a <= 1.2676506002282294e30) ? 1.0 / scale : 0.0;
}
int run_fixed_png16(const LaunchCtx& ctx, const uint16_t* raw, const FixedParams& p,
                    const sn_moments_t& m, float* out6, uint8_t* mask);
int run_dequant_png16(const LaunchCtx& ctx, const uint16_t* raw, int64_t n, int invalid,
                      double scale, float* out32, double* out64);
int run_decode_pfm(const LaunchCtx& ctx, const void* payload, int64_t B, int64_t H, int64_t L,
                   bool big_endian, float* out);

// element-wise geometry (sn_geometry.cu)
template <typename T>
int run_depth_map(const LaunchCtx& ctx, const T* disp, int64_t n, double fxb, double* z);
int run_triangulate(const LaunchCtx& ctx, const double* u, const double* v, const double* d,
                    int64_t n, const FixedParams& p, double* x, double* y, double* z);
template <typename T>
int run_triangulate_grid(const LaunchCtx& ctx, const T* disp, const FixedParams& p, double* xyz);
int run_laplacian(const LaunchCtx& ctx, const double* z, const uint8_t* mask, int64_t B,
                  int64_t H, int64_t W, double* e, uint8_t* ok);

size_t cloud_workspace_bytes(int64_t B, int64_t H, int64_t W);
int run_cloud_count(const LaunchCtx& ctx, const uint8_t* mask, int64_t B, int64_t H, int64_t W,
                    int64_t* frame_offsets, void* workspace, size_t ws_bytes);
int run_cloud_scatter(const LaunchCtx& ctx, const float* out6, const uint8_t* mask, int64_t B,
                      int64_t H, int64_t W, float* cloud, int64_t capacity, void* workspace,
                      size_t ws_bytes);
int run_compact_cloud(const LaunchCtx& ctx, const float* out6, const uint8_t* mask, int64_t B,
                      int64_t H, int64_t W, float* cloud, int64_t capacity,
                      int64_t* frame_offsets, void* workspace, size_t ws_bytes);

}  // namespace sn
