// Element-wise geometry of the reference's public API on the device
// (geometry.py:39-64,85-89,169-172 and adaptive.py:80-97), bit-exact in fp64:
// every operation is one correctly rounded __d*_rn in the reference's
// (numpy's) left-to-right order, with no contraction, so the results equal
// numpy's float64 results bit for bit.
//
//   depth_map_kernel        disparity_to_depth  z = (fx*b)/d, NaN unless d is
//                           finite and > 0 (inf kept: geometry.py:39-45)
//   triangulate_kernel      triangulate (geometry.py:57-64) on flat arrays
//   triangulate_grid_kernel triangulate_grid (geometry.py:85-89): u = column,
//                           v = row, (x, y, z) per pixel -- the points-only
//                           pass (4 or 8 B in, 24 B out per pixel)
//   laplacian_kernel        depth_laplacian (adaptive.py:80-97) of a depth
//                           field given as values + mask
//
// All four are HBM-streaming grid-stride loops (fp64 division bound at most:
// one DDIV per pixel), 16-byte-aligned coalesced accesses per warp.

#include <cuda_runtime.h>
#include <stdint.h>

#include "sn_internal.h"

namespace sn {

__device__ __forceinline__ double qnan_d() { return __longlong_as_double(0x7ff8000000000000ll); }

// geometry.py:39-45: rig.fx * rig.baseline / d, then NaN where d is not
// finite or not > 0 (z itself may be inf for a tiny positive d)
template <typename T>
__device__ __forceinline__ double disp_to_depth(T d, double fxb) {
  const double dd = (double)d;
  return (dd > 0.0 && dd <= 1.7976931348623157e308) ? __ddiv_rn(fxb, dd) : qnan_d();
}

template <typename T>
__global__ void __launch_bounds__(256)
    depth_map_kernel(const T* __restrict__ disp, int64_t n, double fxb, double* __restrict__ z) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    z[i] = disp_to_depth(__ldg(disp + i), fxb);
}

// geometry.py:57-64: z = disparity_to_depth(d); x = (u - u0) * z / fx;
// y = (v - v0) * z / fy (numpy evaluates ((u - u0) * z) / fx)
__device__ __forceinline__ void tri(double u, double v, double z, double u0, double v0, double fx,
                                    double fy, double& x, double& y) {
  x = __ddiv_rn(__dmul_rn(__dsub_rn(u, u0), z), fx);
  y = __ddiv_rn(__dmul_rn(__dsub_rn(v, v0), z), fy);
}

__global__ void __launch_bounds__(256)
    triangulate_kernel(const double* __restrict__ u, const double* __restrict__ v,
                       const double* __restrict__ d, int64_t n, double fxb, double u0, double v0,
                       double fx, double fy, double* __restrict__ x, double* __restrict__ y,
                       double* __restrict__ z) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double zz = disp_to_depth(__ldg(d + i), fxb);
    double xx, yy;
    tri(__ldg(u + i), __ldg(v + i), zz, u0, v0, fx, fy, xx, yy);
    x[i] = xx;
    y[i] = yy;
    z[i] = zz;
  }
}

// one thread per pixel; the (x, y, z) triple of a pixel is 24 contiguous
// bytes, so a warp writes 768 contiguous bytes per step
template <typename T>
__global__ void __launch_bounds__(256)
    triangulate_grid_kernel(const T* __restrict__ disp, int64_t H, int64_t W, int64_t n,
                            double fxb, double u0, double v0, double fx, double fy,
                            double* __restrict__ xyz) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = i % W;
    const int64_t row = (i / W) % H;
    const double zz = disp_to_depth(__ldg(disp + i), fxb);
    double xx, yy;
    tri((double)col, (double)row, zz, u0, v0, fx, fy, xx, yy);
    double* o = xyz + 3 * i;
    o[0] = xx;
    o[1] = yy;
    o[2] = zz;
  }
}

// adaptive.py:80-97: e = |4c - z[v,u-1] - z[v,u+1] - z[v-1,u] - z[v+1,u]|
// (left to right) at interior pixels whose five mask entries are all set,
// NaN and ok = 0 elsewhere.  The values are read whatever the mask says, as
// numpy does (a NaN value under a set mask gives a NaN edge value with
// ok = 1).
__global__ void __launch_bounds__(256)
    laplacian_kernel(const double* __restrict__ z, const uint8_t* __restrict__ m, int64_t H,
                     int64_t W, int64_t n, double* __restrict__ e, uint8_t* __restrict__ ok) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = i % W;
    const int64_t row = (i / W) % H;
    bool good = false;
    double ev = qnan_d();
    if (col >= 1 && col + 1 < W && row >= 1 && row + 1 < H) {
      good = m[i] && m[i - 1] && m[i + 1] && m[i - W] && m[i + W];
      if (good) {
        const double c4 = __dmul_rn(4.0, __ldg(z + i));
        ev = fabs(__dsub_rn(
            __dsub_rn(__dsub_rn(__dsub_rn(c4, __ldg(z + i - 1)), __ldg(z + i + 1)), __ldg(z + i - W)),
            __ldg(z + i + W)));
      }
    }
    if (e) e[i] = ev;
    if (ok) ok[i] = good ? 1 : 0;
  }
}

static unsigned stream_grid(const LaunchCtx& ctx, int64_t n) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = (int64_t)ctx.num_sms * 16;
  if (g > cap) g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

template <typename T>
int run_depth_map(const LaunchCtx& ctx, const T* disp, int64_t n, double fxb, double* z) {
  if (n == 0) return SN_OK;
  depth_map_kernel<T><<<stream_grid(ctx, n), 256, 0, ctx.stream>>>(disp, n, fxb, z);
  return check_launch("depth_map_kernel");
}
template int run_depth_map<float>(const LaunchCtx&, const float*, int64_t, double, double*);
template int run_depth_map<double>(const LaunchCtx&, const double*, int64_t, double, double*);

int run_triangulate(const LaunchCtx& ctx, const double* u, const double* v, const double* d,
                    int64_t n, const FixedParams& p, double* x, double* y, double* z) {
  if (n == 0) return SN_OK;
  triangulate_kernel<<<stream_grid(ctx, n), 256, 0, ctx.stream>>>(u, v, d, n, p.fxb, p.u0, p.v0,
                                                                 p.fx, p.fy, x, y, z);
  return check_launch("triangulate_kernel");
}

template <typename T>
int run_triangulate_grid(const LaunchCtx& ctx, const T* disp, const FixedParams& p,
                         double* xyz) {
  const int64_t n = p.B * p.H * p.W;
  if (n == 0) return SN_OK;
  triangulate_grid_kernel<T><<<stream_grid(ctx, n), 256, 0, ctx.stream>>>(
      disp, p.H, p.W, n, p.fxb, p.u0, p.v0, p.fx, p.fy, xyz);
  return check_launch("triangulate_grid_kernel");
}
template int run_triangulate_grid<float>(const LaunchCtx&, const float*, const FixedParams&,
                                         double*);
template int run_triangulate_grid<double>(const LaunchCtx&, const double*, const FixedParams&,
                                          double*);

int run_laplacian(const LaunchCtx& ctx, const double* z, const uint8_t* mask, int64_t B,
                  int64_t H, int64_t W, double* e, uint8_t* ok) {
  const int64_t n = B * H * W;
  if (n == 0) return SN_OK;
  laplacian_kernel<<<stream_grid(ctx, n), 256, 0, ctx.stream>>>(z, mask, H, W, n, e, ok);
  return check_launch("laplacian_kernel");
}

}  // namespace sn
