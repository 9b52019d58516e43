/* CPU oracle for heatmap/PAF upsampling and peak NMS — TEST INFRASTRUCTURE ONLY.
 *
 * OpenPose resizes the network output back to input resolution and runs a
 * 3x3 non-maximum suppression on the body-part heatmaps (not
 * in the reference). The arithmetic below is the exact IEEE op sequence the
 * CUDA kernels perform (they use __fmul_rn/__fadd_rn/__fdiv_rn, this file is
 * compiled with -ffp-contract=off), so parity is bit-exact on identical input.
 */
#include "avec_oracle.h"

static float src_coord(int o, int scale, int n, int* i0, int* i1) {
  float f = ((float)o + 0.5f) / (float)scale - 0.5f;
  if (f < 0.0f) f = 0.0f;
  int a = (int)f;
  if (a > n - 1) a = n - 1;
  *i0 = a;
  *i1 = (a + 1 < n) ? a + 1 : n - 1;
  return f - (float)a;
}

void oracle_upsample_plane(const float* in, int h, int w, int scale, float* out) {
  const int ho = h * scale, wo = w * scale;
  for (int oy = 0; oy < ho; ++oy) {
    int y0, y1;
    float ly = src_coord(oy, scale, h, &y0, &y1);
    for (int ox = 0; ox < wo; ++ox) {
      int x0, x1;
      float lx = src_coord(ox, scale, w, &x0, &x1);
      float a = in[y0 * w + x0], b = in[y0 * w + x1];
      float c = in[y1 * w + x0], d = in[y1 * w + x1];
      float top = (1.0f - lx) * a + lx * b;
      float bot = (1.0f - lx) * c + lx * d;
      out[(long)oy * wo + ox] = (1.0f - ly) * top + ly * bot;
    }
  }
}

int oracle_nms_plane(const float* in, int h, int w, float threshold, int max_peaks,
                     int* peak_xy, float* peak_refined_xy, float* peak_score) {
  int count = 0;
  for (int y = 0; y < h && count < max_peaks; ++y) {
    for (int x = 0; x < w && count < max_peaks; ++x) {
      float v = in[(long)y * w + x];
      if (!(v > threshold)) continue;
      int peak = 1;
      for (int dy = -1; dy <= 1 && peak; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (!dy && !dx) continue;
          int yy = y + dy, xx = x + dx;
          if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
          if (!(v > in[(long)yy * w + xx])) { peak = 0; break; }
        }
      if (!peak) continue;
      /* 3x3 score-weighted centroid, row-major accumulation order */
      float sw = 0.0f, sx = 0.0f, sy = 0.0f;
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          int yy = y + dy, xx = x + dx;
          if (yy < 0 || yy >= h || xx < 0 || xx >= w) continue;
          float s = in[(long)yy * w + xx];
          sw = sw + s;
          sx = sx + (float)xx * s;
          sy = sy + (float)yy * s;
        }
      peak_xy[2 * count] = x;
      peak_xy[2 * count + 1] = y;
      peak_refined_xy[2 * count] = sx / sw;
      peak_refined_xy[2 * count + 1] = sy / sw;
      peak_score[count] = v;
      ++count;
    }
  }
  return count;
}
