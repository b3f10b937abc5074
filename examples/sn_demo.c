/* A plain-C client of the drop-in boundary (include/sn_b200.h): the whole
 * hot path on host buffers through one call, as a non-Python caller of the
 * reference's estimate_normals_fixed + triangulate_grid (kernels.py:237-261,
 * geometry.py:85-89) would make it.
 *
 *   gcc -O2 -Iinclude examples/sn_demo.c -Lpaper_2504_15121_b200 -lsn_b200 \
 *       -Wl,-rpath,'$ORIGIN/../paper_2504_15121_b200' -lm -o examples/sn_demo
 *   examples/sn_demo            # exit code 0 on success
 *
 * Input: a tilted plane in disparity space, d(u, v) = a + b u + c v, whose
 * normal is known in closed form: with the reference's formula
 * (geometry.py:175-216; a1 - 1 = b, a2 = c) the normal is proportional to
 * (-b fx, -c fy, -(a + b u0 + c v0)) -- camera-facing, n_z < 0. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "sn_b200.h"

static int fail(const char* what, int rc) {
  fprintf(stderr, "%s failed (rc=%d): %s\n", what, rc, sn_last_error());
  return 1;
}

int main(void) {
  const int64_t B = 2, H = 128, W = 256;
  const double a = 40.0, b = 0.03, c = -0.02;
  const sn_rig_t rig = {300.0, 300.0, 127.5, 63.5, 0.25};
  float* disp = (float*)malloc(sizeof(float) * B * H * W);
  float* rec = (float*)malloc(sizeof(float) * B * H * W * 6);
  uint8_t* mask = (uint8_t*)malloc(B * H * W);
  int32_t* labels = (int32_t*)malloc(sizeof(int32_t) * B * H * W);
  int32_t off[2 * 81];
  int n = 0;
  for (int dy = -4; dy <= 4; ++dy)
    for (int dx = -4; dx <= 4; ++dx) {
      off[2 * n] = dx;
      off[2 * n + 1] = dy;
      ++n;
    }
  for (int64_t f = 0; f < B; ++f)
    for (int64_t v = 0; v < H; ++v)
      for (int64_t u = 0; u < W; ++u) disp[(f * H + v) * W + u] = (float)(a + b * u + c * v);

  sn_plan_t* plan = NULL;
  int rc = sn_plan_create(0, &plan);
  if (rc) return fail("sn_plan_create", rc);
  rc = sn_pipeline_host(plan, disp, B, H, W, &rig, off, n, 1.0, rec, mask, labels);
  if (rc) return fail("sn_pipeline_host", rc);

  /* expected unit normal (camera-facing) */
  double e[3] = {-b * rig.fx, -c * rig.fy, -(a + b * rig.u0 + c * rig.v0)};
  const double en = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
  for (int i = 0; i < 3; ++i) e[i] /= en;
  double worst = 0.0;
  int64_t valid = 0, bad_mask = 0;
  for (int64_t f = 0; f < B; ++f)
    for (int64_t v = 0; v < H; ++v)
      for (int64_t u = 0; u < W; ++u) {
        const int64_t i = (f * H + v) * W + u;
        const int interior = u >= 4 && u < W - 4 && v >= 4 && v < H - 4;
        if ((mask[i] != 0) != interior) ++bad_mask;
        if (!mask[i]) continue;
        ++valid;
        const float* r = rec + 6 * i;
        /* atan2(|n x e|, n . e): acos of a dot product near 1 would turn the
         * fp32 storage rounding into ~0.03 deg */
        const double cx = r[4] * e[2] - r[5] * e[1], cy = r[5] * e[0] - r[3] * e[2],
                     cz = r[3] * e[1] - r[4] * e[0];
        const double dot = r[3] * e[0] + r[4] * e[1] + r[5] * e[2];
        const double ang = atan2(sqrt(cx * cx + cy * cy + cz * cz), dot) * 180.0 / M_PI;
        if (ang > worst) worst = ang;
      }
  /* the plane is one passable component: label = the first interior pixel */
  int64_t bad_label = 0;
  for (int64_t f = 0; f < B; ++f)
    for (int64_t v = 1; v < H - 1; ++v)
      for (int64_t u = 1; u < W - 1; ++u)
        if (labels[(f * H + v) * W + u] != (int32_t)(1 * W + 1)) ++bad_label;
  printf("sn_demo: abi %d, %lld valid normals, worst angle %.2e deg, mask errors %lld, "
         "label errors %lld\n",
         sn_abi_version(), (long long)valid, worst, (long long)bad_mask, (long long)bad_label);
  sn_plan_destroy(plan);
  free(disp);
  free(rec);
  free(mask);
  free(labels);
  return (bad_mask == 0 && bad_label == 0 && worst < 1e-4) ? 0 : 1;
}
