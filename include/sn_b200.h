/*
 * sn_b200.h -- C ABI of the B200-native stereonorm hot path.
 *
 * Plain pointers and sizes only (no torch / CUDA types in signatures); a
 * stream is passed as `void*` (a cudaStream_t / CUstream handle, NULL =
 * legacy default stream).  Device entry points are asynchronous on that
 * stream and never synchronise the host; *_host entry points take host
 * buffers and return when the result is in host memory.
 *
 * Every entry point returns one of the SN_* codes below; on failure
 * sn_last_error() (thread-local) describes it.  Python maps the codes to
 * ValueError / DegenerateSupportError / RuntimeError exactly as the
 * reference raises them.
 *
 * Reference interfaces replaced (paths relative to pkg/src/stereonorm):
 *   sn_oriented_points[_f64]  estimate_normals_fixed   kernels.py:237-261
 *                             + triangulate_grid        geometry.py:85-89
 *                             dense record of the CLI's PLY path cli.py:118-123
 *   sn_affine[_f64]           convolve_affine           kernels.py:182-203
 *   sn_passable               depth_field + depth_laplacian + ST test
 *                             geometry.py:169-172, adaptive.py:80-97,130-132
 *   sn_ccl_labels             (new) 8-connected labels of
 *                             the ST-passable set, canonical min raster index
 *   sn_kernel_moments         build_kernels             kernels.py:78-103
 *
 * Every entry point that reads disparities has an fp32 form and an _f64 form.
 * The _f64 forms take the reference's own float64 values (ScalarField,
 * fields.py:37-40) unrounded: masks, passable sets, labels and star-fill
 * supports are then bit-exact with the reference on its inputs (no fp32 cast
 * anywhere on the decision paths).
 *
 * Layouts: disparity [B][H][W] row-major (fp32 or fp64, NaN/+-inf = invalid),
 * out6 [B][H][W][6] fp32 = (x, y, z, nx, ny, nz) -- the PLY vertex record
 * (formats.py:167-183) -- with NaN normals where the normal is invalid and
 * NaN points where the disparity is not finite and > 0; mask [B][H][W]
 * uint8 (1 = valid normal), optional (NULL).  Offsets are (vx, vy) int32
 * pairs, exactly KernelSpec.offsets (kernels.py:31-55).
 */
#ifndef SN_B200_H
#define SN_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SN_API __attribute__((visibility("default")))
#else
#define SN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SN_OK 0
#define SN_EINVAL 1      /* invalid argument            -> ValueError             */
#define SN_EDEGENERATE 2 /* collinear offset pattern    -> DegenerateSupportError */
#define SN_ECUDA 3       /* CUDA / driver failure       -> RuntimeError           */

#define SN_ABI_VERSION 2

typedef struct sn_rig {
  double fx, fy, u0, v0, baseline; /* geometry.py:22-36 (StereoRig) */
} sn_rig_t;

/* Integer moments of an offset pattern (kernels.py:87-103). */
typedef struct sn_moments {
  int64_t alpha, beta, gamma, det, sx, sy;
  int32_t hx, hy;       /* half extents of the support box               */
  int32_t square_r;     /* R if the pattern is the centred (2R+1)^2 square, else -1 */
} sn_moments_t;

typedef struct sn_plan sn_plan_t;

SN_API int sn_abi_version(void);
SN_API const char* sn_last_error(void);

/* A plan binds a device and owns the host-path workspace (copy/compute
 * streams, double-buffered device chunks, and pinned host staging used when a
 * caller's host buffers are pageable).  Device entry points only use the plan
 * for the device id and cached properties (their scratch comes from the
 * caller's workspace or from stream-ordered allocations on the caller's
 * stream) and are safe to call concurrently on distinct streams; *_host
 * calls on one plan are serialised by the plan's lock.  sn_ccl_labels[_ws]
 * [_f64] with B >= 128 frames also use the plan's second stream: the two half
 * batches run on the caller's stream and that one (forked from and joined
 * back into the caller's stream with events; concurrent calls on one plan
 * queue their second halves behind each other there). */
SN_API int sn_plan_create(int device, sn_plan_t** plan);
SN_API int sn_plan_destroy(sn_plan_t* plan);

/* kernels.py:78-103: validates the pattern (N>0, distinct) and returns its
 * integer moments; SN_EDEGENERATE when det <= 0.5. */
SN_API int sn_kernel_moments(const int32_t* offsets_xy, int32_t n_off, sn_moments_t* out);

/* Fused fixed-kernel pass: LSQ affine fit + closed-form normal + triangulated
 * point, dense AoS-6 output.  Device pointers. */
SN_API int sn_oriented_points(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                       const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off,
                       float* out6, uint8_t* mask, void* stream);
SN_API int sn_oriented_points_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H,
                           int64_t W, const sn_rig_t* rig, const int32_t* offsets_xy,
                           int32_t n_off, float* out6, uint8_t* mask, void* stream);

/* Same pass on row-pitched input (SURVEY.md §8(b) sn_fixed_points' `ld`):
 * row v of frame b starts at disp + (b * H + v) * ld, ld >= W elements (a
 * crop of a wider buffer, or rows padded for alignment).  Pitches whose rows
 * are 16-byte aligned feed the TMA tensor map directly; others are packed
 * into stream-ordered scratch first.  Output is dense [B][H][W][6]. */
SN_API int sn_oriented_points_strided(sn_plan_t* plan, const float* disp, int64_t B, int64_t H,
                               int64_t W, int64_t ld, const sn_rig_t* rig,
                               const int32_t* offsets_xy, int32_t n_off, float* out6,
                               uint8_t* mask, void* stream);
SN_API int sn_oriented_points_strided_f64(sn_plan_t* plan, const double* disp, int64_t B,
                                   int64_t H, int64_t W, int64_t ld, const sn_rig_t* rig,
                                   const int32_t* offsets_xy, int32_t n_off, float* out6,
                                   uint8_t* mask, void* stream);

/* Same pass over a block of rows of a taller image (strip partitioning,
 * SURVEY.md §8(e)): block row i is image row row0 + i, which only changes the
 * pixel coordinate v of the normal and point; the block's first and last
 * rows are treated as image borders, so a strip passes its owned rows plus
 * a halo of R rows on each interior side and keeps the owned rows. */
SN_API int sn_oriented_points_rows(sn_plan_t* plan, const float* disp, int64_t B, int64_t H,
                            int64_t W, int64_t row0, const sn_rig_t* rig,
                            const int32_t* offsets_xy, int32_t n_off, float* out6,
                            uint8_t* mask, void* stream);
SN_API int sn_oriented_points_rows_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H,
                                int64_t W, int64_t row0, const sn_rig_t* rig,
                                const int32_t* offsets_xy, int32_t n_off, float* out6,
                                uint8_t* mask, void* stream);

/* Same pass + the ST-passable bit mask (adaptive.py:80-97,130-132;
 * threshold t > 0; the fused pass and sn_passable_bits back to back on the
 * stream): bits is [B][H][ceil(W/32)]
 * uint32, bit (u % 32) of word u / 32 set iff pixel u of the row is passable.
 * row0 as for sn_oriented_points_rows. */
SN_API int sn_oriented_points_bits(sn_plan_t* plan, const float* disp, int64_t B, int64_t H,
                            int64_t W, int64_t row0, const sn_rig_t* rig,
                            const int32_t* offsets_xy, int32_t n_off, double t, float* out6,
                            uint8_t* mask, uint32_t* bits, void* stream);
SN_API int sn_oriented_points_bits_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H,
                                int64_t W, int64_t row0, const sn_rig_t* rig,
                                const int32_t* offsets_xy, int32_t n_off, double t, float* out6,
                                uint8_t* mask, uint32_t* bits, void* stream);

/* The ST-passable bit mask alone (layout of sn_oriented_points_bits), as one
 * streaming kernel over the disparity. */
SN_API int sn_passable_bits(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                     const sn_rig_t* rig, double t, uint32_t* bits, void* stream);
SN_API int sn_passable_bits_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H,
                         int64_t W, const sn_rig_t* rig, double t, uint32_t* bits,
                         void* stream);

/* The whole north-star pipeline in one call: fused fit + normal + point +
 * passable bits, then component labels from the bits (label semantics as
 * sn_ccl_labels with row_base 0).  Device pointers.  The _ws variants take a
 * caller workspace of sn_ccl_workspace_bytes(B, H, W) bytes; the others take
 * stream-ordered scratch from the library's private pool on `stream`, so
 * concurrent calls on different streams never share it. */
SN_API int sn_pipeline(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off, double t,
                float* out6, uint8_t* mask, int32_t* labels, void* stream);
SN_API int sn_pipeline_ws(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                   const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off, double t,
                   float* out6, uint8_t* mask, int32_t* labels, void* workspace,
                   size_t ws_bytes, void* stream);
SN_API int sn_pipeline_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H, int64_t W,
                    const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off, double t,
                    float* out6, uint8_t* mask, int32_t* labels, void* stream);
SN_API int sn_pipeline_ws_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H,
                       int64_t W, const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off,
                       double t, float* out6, uint8_t* mask, int32_t* labels, void* workspace,
                       size_t ws_bytes, void* stream);

/* Same pass, host buffers: chunks of whole frames with H2D / compute / D2H
 * overlapped on three streams; returns when out6 (and mask, if non-NULL)
 * hold the result.  Page-locked buffers (cudaHostAlloc / cudaHostRegister /
 * torch pin_memory) are copied directly; pageable ones are staged through
 * the plan's pinned slots by multi-threaded host copies.  On an error every
 * queued copy and kernel is drained before the call returns. */
SN_API int sn_oriented_points_host(sn_plan_t* plan, const float* disp_host, int64_t B, int64_t H,
                            int64_t W, const sn_rig_t* rig, const int32_t* offsets_xy,
                            int32_t n_off, float* out6_host, uint8_t* mask_host);
SN_API int sn_oriented_points_host_f64(sn_plan_t* plan, const double* disp_host, int64_t B,
                                int64_t H, int64_t W, const sn_rig_t* rig,
                                const int32_t* offsets_xy, int32_t n_off, float* out6_host,
                                uint8_t* mask_host);

/* The whole pipeline on host buffers (staging as sn_oriented_points_host):
 * points, optional mask, and component labels, chunked with H2D / compute /
 * D2H overlapped; returns when every output is in host memory. */
SN_API int sn_pipeline_host(sn_plan_t* plan, const float* disp_host, int64_t B, int64_t H,
                     int64_t W, const sn_rig_t* rig, const int32_t* offsets_xy, int32_t n_off,
                     double t, float* out6_host, uint8_t* mask_host, int32_t* labels_host);
SN_API int sn_pipeline_host_f64(sn_plan_t* plan, const double* disp_host, int64_t B, int64_t H,
                         int64_t W, const sn_rig_t* rig, const int32_t* offsets_xy,
                         int32_t n_off, double t, float* out6_host, uint8_t* mask_host,
                         int32_t* labels_host);

/* convolve_affine (gradient convention a1 - 1 = dd/du, a2 = dd/dv); a1/a2 are
 * NaN where mask is 0.  Device pointers, fp64 outputs. */
SN_API int sn_affine(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
              const int32_t* offsets_xy, int32_t n_off, double* a1, double* a2,
              uint8_t* mask, void* stream);
SN_API int sn_affine_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H, int64_t W,
                  const int32_t* offsets_xy, int32_t n_off, double* a1, double* a2,
                  uint8_t* mask, void* stream);

/* ST-passable set: edge value valid and <= t (bit-exact fp64 predicate).
 * edges (optional, NULL to skip) receives the depth-Laplacian values, NaN
 * where invalid. */
SN_API int sn_passable(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                const sn_rig_t* rig, double t, uint8_t* passable, double* edges,
                void* stream);
SN_API int sn_passable_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H, int64_t W,
                    const sn_rig_t* rig, double t, uint8_t* passable, double* edges,
                    void* stream);

/* 8-connected component labels of the passable set; label = smallest raster
 * index v*W + u + index_base in the component (per frame), -1 elsewhere.
 * row_base lets a strip of a larger frame use global raster indices
 * (index_base = row_base * W).  Device pointers. */
SN_API int sn_ccl_labels(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                  const sn_rig_t* rig, double t, int64_t row_base, int32_t* labels,
                  void* stream);
SN_API int sn_ccl_labels_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H, int64_t W,
                      const sn_rig_t* rig, double t, int64_t row_base, int32_t* labels,
                      void* stream);

/* Label an already-computed passable grid (uint8) -- used by strip mode and
 * by tests of the labeller alone. */
SN_API int sn_ccl_from_passable(sn_plan_t* plan, const uint8_t* passable, int64_t B, int64_t H,
                         int64_t W, int64_t row_base, int32_t* labels, void* stream);

/* The labeller needs a device workspace (passable bit mask + tile seam rows
 * + slot labels, sn_ccl_workspace_bytes; from 128 frames on it has room for
 * the two half-batch workspaces sn_ccl_labels_ws uses).  The entry points above take
 * stream-ordered scratch from the library's private pool on `stream`; the
 * *_ws variants take the caller's, so concurrent streams each pass their
 * own. */
SN_API int sn_ccl_workspace_bytes(int64_t B, int64_t H, int64_t W, size_t* bytes);
SN_API int sn_ccl_labels_ws(sn_plan_t* plan, const float* disp, int64_t B, int64_t H, int64_t W,
                     const sn_rig_t* rig, double t, int64_t row_base, int32_t* labels,
                     void* workspace, size_t ws_bytes, void* stream);
SN_API int sn_ccl_labels_ws_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H,
                         int64_t W, const sn_rig_t* rig, double t, int64_t row_base,
                         int32_t* labels, void* workspace, size_t ws_bytes, void* stream);
/* Label from a passable bit mask (layout of sn_oriented_points_bits); the
 * workspace's own bit-mask region is unused. */
SN_API int sn_ccl_from_bits_ws(sn_plan_t* plan, const uint32_t* bits, int64_t B, int64_t H,
                        int64_t W, int64_t row_base, int32_t* labels, void* workspace,
                        size_t ws_bytes, void* stream);
SN_API int sn_ccl_from_passable_ws(sn_plan_t* plan, const uint8_t* passable, int64_t B,
                            int64_t H, int64_t W, int64_t row_base, int32_t* labels,
                            void* workspace, size_t ws_bytes, void* stream);

/* Element-wise geometry of the reference's public API, bit-exact fp64
 * (device pointers, flat arrays of n elements):
 *   sn_depth_map[_f64]     disparity_to_depth (geometry.py:39-45): z = (fx*b)/d,
 *                          NaN unless d is finite and > 0 (inf kept).
 *   sn_triangulate_f64     triangulate (geometry.py:57-64): x = ((u-u0)*z)/fx,
 *                          y = ((v-v0)*z)/fy, z as above.
 *   sn_triangulate_grid[_f64]  triangulate_grid (geometry.py:85-89): [B][H][W][3]
 *                          fp64 points with u = column, v = row -- a points-only
 *                          pass, no fit.
 *   sn_depth_laplacian_f64 depth_laplacian (adaptive.py:80-97) of a depth field
 *                          (values + uint8 mask): edges NaN and ok 0 outside the
 *                          interior pixels whose five mask entries are set;
 *                          either output may be NULL. */
SN_API int sn_depth_map(sn_plan_t* plan, const float* disp, int64_t n, const sn_rig_t* rig,
                 double* z, void* stream);
SN_API int sn_depth_map_f64(sn_plan_t* plan, const double* disp, int64_t n, const sn_rig_t* rig,
                     double* z, void* stream);
SN_API int sn_triangulate_f64(sn_plan_t* plan, const double* u, const double* v, const double* d,
                       int64_t n, const sn_rig_t* rig, double* x, double* y, double* z,
                       void* stream);
SN_API int sn_triangulate_grid(sn_plan_t* plan, const float* disp, int64_t B, int64_t H,
                        int64_t W, const sn_rig_t* rig, double* xyz, void* stream);
SN_API int sn_triangulate_grid_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H,
                            int64_t W, const sn_rig_t* rig, double* xyz, void* stream);
SN_API int sn_depth_laplacian_f64(sn_plan_t* plan, const double* depth, const uint8_t* mask,
                           int64_t B, int64_t H, int64_t W, double* edges, uint8_t* ok,
                           void* stream);

/* Strip-seam merge.  HOST memory: `seams` holds, for each
 * of the n_strips strips in row order, its first and last owned label rows
 * ([n_strips][2][W] int32, global raster indices, -1 = not passable), as
 * gathered from all ranks.  8-adjacent passable pixels across each seam are
 * united with min-root links; writes the (label -> root) pairs of every label
 * that changes, sorted by label, to map_keys/map_vals (capacity
 * 2*n_strips*W) and their count to *n_map.  Deterministic and identical on
 * every rank. */
SN_API int sn_seam_merge_host(const int32_t* seams, int32_t n_strips, int64_t W, int32_t* map_keys,
                       int32_t* map_vals, int32_t* n_map);

/* The same merge on the device, with no host round trip (the multi-GPU strip
 * path: the all-gathered rows stay in device memory).  seams: device
 * [n_strips][2][W] int32; table: device int32[table_n] with table_n > every
 * label value (the frame's pixel count); on return table[v] is the root of
 * every label v on a seam, -1 elsewhere.  sn_relabel_table then maps a
 * strip's labels in place: v -> table[v] where that is >= 0.  Deterministic
 * (min-root links) and identical on every rank. */
SN_API int sn_seam_merge(sn_plan_t* plan, const int32_t* seams, int32_t n_strips, int64_t W,
                  int32_t* table, int64_t table_n, void* stream);
SN_API int sn_relabel_table(sn_plan_t* plan, int32_t* labels, int64_t n, const int32_t* table,
                     int64_t table_n, void* stream);

/* Apply a (label -> root) map to a strip's label grid in place (device).
 * Labels of the strip are global raster indices in [index_base,
 * index_base + n); scratch is an int32 device buffer of n elements. */
SN_API int sn_relabel(sn_plan_t* plan, int32_t* labels, int64_t n, int64_t index_base,
               const int32_t* map_keys, const int32_t* map_vals, const int32_t* n_map,
               int32_t map_capacity, int32_t* scratch, void* stream);

/* Adaptive star-fill normals (estimate_normals_adaptive, adaptive.py:177-268;
 * StarConfig adaptive.py:32-57): the dense record of the fixed pass with
 * normals fitted over edge-aware star supports.  The rays are the
 * reference's ray_offsets(config) (adaptive.py:60-77), passed as n_rays
 * lengths + the concatenated (vx, vy) int32 pairs; stop 0 = "st" (edge value
 * valid and <= threshold), 1 = "cd" (covered depth range <= threshold * z_c,
 * per ray or shared_range).  Masks bit-exact with the reference.  Workspace:
 * sn_adaptive_workspace_bytes (fp64 depth map + bit mask). */
SN_API int sn_adaptive_workspace_bytes(int64_t B, int64_t H, int64_t W, size_t* bytes);
SN_API int sn_adaptive_points(sn_plan_t* plan, const float* disp, int64_t B, int64_t H,
                       int64_t W, const sn_rig_t* rig, int32_t n_rays, const int32_t* ray_len,
                       const int32_t* ray_xy, int32_t stop, int32_t shared_range,
                       double threshold, float* out6, uint8_t* mask, void* workspace,
                       size_t ws_bytes, void* stream);
SN_API int sn_adaptive_points_f64(sn_plan_t* plan, const double* disp, int64_t B, int64_t H,
                           int64_t W, const sn_rig_t* rig, int32_t n_rays,
                           const int32_t* ray_len, const int32_t* ray_xy, int32_t stop,
                           int32_t shared_range, double threshold, float* out6, uint8_t* mask,
                           void* workspace, size_t ws_bytes, void* stream);

/* Accuracy evaluation on the device (evaluation.py:34-73): per frame, the
 * unsigned angle map degrees(arccos(|n_est . n_gt|)) over jointly valid
 * pixels (est normals: 3 floats at the start of each est_stride-float record,
 * NaN = invalid -- est_stride 6 reads the dense oriented-point record; gt:
 * [B][H][W][3] double + uint8 mask; extra_mask optional) and its statistics
 * stats[B][6] = (avg, min, max, lower median, population std, count), NaN
 * where a frame has no valid pixel.  err_out (optional) receives the map
 * (NaN invalid).  Device pointers; workspace: sn_eval_workspace_bytes. */
SN_API int sn_eval_workspace_bytes(int64_t B, int64_t H, int64_t W, size_t* bytes);
SN_API int sn_angular_error(sn_plan_t* plan, const float* est, int32_t est_stride,
                     const double* gt, const uint8_t* gt_mask, const uint8_t* extra_mask,
                     int64_t B, int64_t H, int64_t W, double* err_out, double* stats,
                     void* workspace, size_t ws_bytes, void* stream);
/* summarize (evaluation.py:58-73) of a given map: values [B][H][W] double,
 * non-finite = invalid; same stats layout. */
SN_API int sn_error_stats(sn_plan_t* plan, const double* values, int64_t B, int64_t H,
                   int64_t W, double* stats, void* workspace, size_t ws_bytes, void* stream);
SN_API int sn_angular_error_f64(sn_plan_t* plan, const double* est, int32_t est_stride,
                         const double* gt, const uint8_t* gt_mask, const uint8_t* extra_mask,
                         int64_t B, int64_t H, int64_t W, double* err_out, double* stats,
                         void* workspace, size_t ws_bytes, void* stream);

/* Oriented point cloud compaction (cli.py:118-123, the vertices
 * formats.py:170-185 writes): the records of pixels whose normal is valid
 * (mask != 0, as emitted by the fused pass), in raster order over the whole
 * batch, packed into cloud [N][6] float32 -- the binary-PLY vertex body.
 * frame_offsets (device, B + 1 int64): frame f's vertices are
 * [offsets[f], offsets[f+1]); offsets[B] = N even when N > capacity (only
 * the first capacity vertices are written).  Workspace:
 * sn_cloud_workspace_bytes. */
SN_API int sn_cloud_workspace_bytes(int64_t B, int64_t H, int64_t W, size_t* bytes);
SN_API int sn_compact_cloud(sn_plan_t* plan, const float* out6, const uint8_t* mask, int64_t B,
                     int64_t H, int64_t W, float* cloud, int64_t capacity,
                     int64_t* frame_offsets, void* workspace, size_t ws_bytes, void* stream);

/* Device input codecs (formats.py).  The container (PNG zlib stream, PFM
 * header) is parsed on the host; these take the raw sample payload already
 * in device memory.
 *
 * sn_dequant_png16: read_disparity_png16 (formats.py:133-150) per sample:
 * d = (raw - 1.0) / scale in fp64, raw == invalid -> NaN (invalid = -1: no
 * invalid value).  out_f64 gets the reference's value bit-exactly, out_f32
 * that value rounded once; either may be NULL. */
SN_API int sn_dequant_png16(sn_plan_t* plan, const uint16_t* raw, int64_t B, int64_t H, int64_t W,
                     double scale, int32_t invalid, float* out_f32, double* out_f64,
                     void* stream);

/* sn_decode_pfm: the payload step of read_pfm / read_pfm_normals
 * (formats.py:84-113): B payloads of H x W x channels 4-byte floats, bottom
 * row first, big-endian when the header scale is positive -> out [B][H][W]
 * (x channels) native fp32, top row first.  Non-finite samples stay as they
 * are (they mark invalid pixels, fields.py ScalarField.from_array). */
SN_API int sn_decode_pfm(sn_plan_t* plan, const void* payload, int64_t B, int64_t H, int64_t W,
                  int32_t channels, int32_t big_endian, float* out, void* stream);

/* sn_oriented_points with a 16-bit PNG disparity payload read directly by
 * the fused pass (read_disparity_png16 + estimate_normals_fixed +
 * triangulate_grid): 2 B/px in instead of 4 (widths that are not a multiple of 8
 * go through a row-pitched copy).  Needs a centred square kernel (3..17) and
 * 2^-100 <= |scale| <= 2^100; SN_EINVAL otherwise (dequantise with
 * sn_dequant_png16 and use sn_oriented_points_f64). */
SN_API int sn_oriented_points_png16(sn_plan_t* plan, const uint16_t* raw, int64_t B, int64_t H,
                             int64_t W, double scale, int32_t invalid, const sn_rig_t* rig,
                             const int32_t* offsets_xy, int32_t n_off, float* out6,
                             uint8_t* mask, void* stream);

/* The two halves of sn_compact_cloud, for callers that size the output from
 * the count: sn_cloud_count writes frame_offsets (device, B + 1; the total in
 * offsets[B]) and leaves the block scan in the workspace; sn_cloud_scatter
 * then writes the vertices, given the same mask and workspace. */
SN_API int sn_cloud_count(sn_plan_t* plan, const uint8_t* mask, int64_t B, int64_t H, int64_t W,
                   int64_t* frame_offsets, void* workspace, size_t ws_bytes, void* stream);
SN_API int sn_cloud_scatter(sn_plan_t* plan, const float* out6, const uint8_t* mask, int64_t B,
                     int64_t H, int64_t W, float* cloud, int64_t capacity, void* workspace,
                     size_t ws_bytes, void* stream);

/* Test hook: the fixed pass forced onto the generic (non-TMA) kernel, used to
 * cross-check the TMA fast path on identical inputs. */
SN_API int sn_oriented_points_generic(sn_plan_t* plan, const float* disp, int64_t B, int64_t H,
                               int64_t W, const sn_rig_t* rig, const int32_t* offsets_xy,
                               int32_t n_off, float* out6, uint8_t* mask, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SN_B200_H */
