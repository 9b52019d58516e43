/* CPU oracle for the OpenPose pose-net layers — TEST INFRASTRUCTURE ONLY.
 *
 * The reference has no CNN (MockPose stands in for OpenPose), so
 * this is the build's own restatement of the Caffe layer semantics OpenPose's
 * pose_deploy_linevec.prototxt uses: Convolution (stride 1, pad k/2, bias),
 * ReLU, Pooling MAX 2x2/2 (Caffe ceil mode; exact for even sizes), Concat.
 * Parity for these tensors is therefore "unpinned" against the reference and
 * pinned only against this oracle.
 *
 * Precision contract mirrored from the CUDA path: activations and weights are
 * bf16 values, products accumulated here in double (the CUDA path accumulates
 * fp32 in TMEM), bias added, ReLU, optional bf16 RNE rounding of the output.
 */
#include <pthread.h>
#include <stdlib.h>
#include <unistd.h>
#include <string.h>

#include "avec_oracle.h"

int oracle_threads(void) {
  const char* e = getenv("AVEC_ORACLE_THREADS");
  long n = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
  if (n < 1) n = 1;
  if (n > 64) n = 64;
  return (int)n;
}

float oracle_bf16_round(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) { /* inf / nan: truncate, keep nan quiet */
    if (u & 0x007fffffu) u |= 0x00400000u;
    u &= 0xffff0000u;
  } else {
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    u &= 0xffff0000u;
  }
  float r;
  memcpy(&r, &u, 4);
  return r;
}

typedef struct {
  const float* in; const double* wt; const float* bias; float* out;
  int n, h, w, cin, cout, k, act, rnd;
  const float* slope; /* PReLU slopes when act == 2 */
  int next_row;       /* guarded by atomic fetch-add */
} conv_job;

static void* conv_worker(void* arg) {
  conv_job* j = (conv_job*)arg;
  const int pad = j->k / 2, k = j->k, cin = j->cin, cout = j->cout, h = j->h, w = j->w;
  double* acc = (double*)malloc(sizeof(double) * (size_t)cout);
  for (;;) {
    int row = __atomic_fetch_add(&j->next_row, 1, __ATOMIC_RELAXED);
    if (row >= j->n * h) break;
    int b = row / h, y = row % h;
    for (int x = 0; x < w; ++x) {
      for (int co = 0; co < cout; ++co) acc[co] = 0.0;
      for (int r = 0; r < k; ++r) {
        int iy = y + r - pad;
        if (iy < 0 || iy >= h) continue;
        for (int s = 0; s < k; ++s) {
          int ix = x + s - pad;
          if (ix < 0 || ix >= w) continue;
          const float* px = j->in + (((size_t)b * h + iy) * w + ix) * cin;
          const double* wrs = j->wt + ((size_t)r * k + s) * cin * cout;
          for (int ci = 0; ci < cin; ++ci) {
            const double v = (double)px[ci];
            const double* wr = wrs + (size_t)ci * cout;
            for (int co = 0; co < cout; ++co) acc[co] += v * wr[co];
          }
        }
      }
      float* o = j->out + (((size_t)b * h + y) * w + x) * cout;
      for (int co = 0; co < cout; ++co) {
        float v = (float)(acc[co] + (double)j->bias[co]);
        if (j->act == 1 && v < 0.f) v = 0.f;             /* Caffe ReLU */
        if (j->act == 2 && v < 0.f) v = v * j->slope[co];  /* Caffe PReLU, channel-wise */
        o[co] = j->rnd ? oracle_bf16_round(v) : v;
      }
    }
  }
  free(acc);
  return NULL;
}

void oracle_conv2d_nhwc(const float* in, int n, int h, int w, int cin,
                        const float* weight, const float* bias, int cout, int k,
                        int act, const float* slope, int out_round_bf16, float* out) {
  /* repack W[co][ci][r][s] -> Wt[r][s][ci][co] so the inner loop runs over co */
  double* wt = (double*)malloc(sizeof(double) * (size_t)k * k * cin * cout);
  for (int co = 0; co < cout; ++co)
    for (int ci = 0; ci < cin; ++ci)
      for (int r = 0; r < k; ++r)
        for (int s = 0; s < k; ++s)
          wt[(((size_t)r * k + s) * cin + ci) * cout + co] =
              (double)weight[(((size_t)co * cin + ci) * k + r) * k + s];
  conv_job j = {in, wt, bias, out, n, h, w, cin, cout, k, act, out_round_bf16, slope, 0};
  int nt = oracle_threads();
  pthread_t th[64];
  for (int t = 0; t < nt; ++t) pthread_create(&th[t], NULL, conv_worker, &j);
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  free(wt);
}

/* Selected output rows of one conv layer (full-size parity checks): each of
 * the n_rows outputs row r comes from its own k-row input window
 * win[r][0..k-1][w][cin] (rows outside the image already zero — the layer's
 * zero padding), columns padded by k/2 zeros here. Same arithmetic as
 * oracle_conv2d_nhwc, so a row computed here equals that row of the whole
 * tensor. Work is split over (row, 16-column chunk). */
typedef struct {
  const float* win; const double* wt; const float* bias; float* out;
  int n_rows, k, w, cin, cout, act, rnd;
  const float* slope;
  int next; /* guarded by atomic fetch-add */
} rows_job;

static void* rows_worker(void* arg) {
  rows_job* j = (rows_job*)arg;
  const int k = j->k, pad = k / 2, w = j->w, cin = j->cin, cout = j->cout;
  const int chunks = (w + 15) / 16;
  double* acc = (double*)malloc(sizeof(double) * (size_t)cout);
  for (;;) {
    int item = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
    if (item >= j->n_rows * chunks) break;
    const int row = item / chunks, x0 = (item % chunks) * 16;
    const int x1 = x0 + 16 < w ? x0 + 16 : w;
    const float* win = j->win + (size_t)row * k * w * cin;
    for (int x = x0; x < x1; ++x) {
      for (int co = 0; co < cout; ++co) acc[co] = 0.0;
      for (int r = 0; r < k; ++r)
        for (int s = 0; s < k; ++s) {
          const int ix = x + s - pad;
          if (ix < 0 || ix >= w) continue;
          const float* px = win + ((size_t)r * w + ix) * cin;
          const double* wrs = j->wt + ((size_t)r * k + s) * cin * cout;
          for (int ci = 0; ci < cin; ++ci) {
            const double v = (double)px[ci];
            const double* wr = wrs + (size_t)ci * cout;
            for (int co = 0; co < cout; ++co) acc[co] += v * wr[co];
          }
        }
      float* o = j->out + ((size_t)row * w + x) * cout;
      for (int co = 0; co < cout; ++co) {
        float v = (float)(acc[co] + (double)j->bias[co]);
        if (j->act == 1 && v < 0.f) v = 0.f;
        if (j->act == 2 && v < 0.f) v = v * j->slope[co];
        o[co] = j->rnd ? oracle_bf16_round(v) : v;
      }
    }
  }
  free(acc);
  return NULL;
}

void oracle_conv2d_rows(const float* win, int n_rows, int k, int w, int cin, const float* weight,
                        const float* bias, int cout, int act, const float* slope, int out_round_bf16,
                        float* out) {
  double* wt = (double*)malloc(sizeof(double) * (size_t)k * k * cin * cout);
  for (int co = 0; co < cout; ++co)
    for (int ci = 0; ci < cin; ++ci)
      for (int r = 0; r < k; ++r)
        for (int s = 0; s < k; ++s)
          wt[(((size_t)r * k + s) * cin + ci) * cout + co] =
              (double)weight[(((size_t)co * cin + ci) * k + r) * k + s];
  rows_job j = {win, wt, bias, out, n_rows, k, w, cin, cout, act, out_round_bf16, slope, 0};
  int nt = oracle_threads();
  pthread_t th[64];
  for (int t = 0; t < nt; ++t) pthread_create(&th[t], NULL, rows_worker, &j);
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
  free(wt);
}

/* Caffe Pooling MAX kernel 2 stride 2, NHWC; h and w even */
void oracle_maxpool2_nhwc(const float* in, int n, int h, int w, int c, float* out) {
  const int ho = h / 2, wo = w / 2;
  for (int b = 0; b < n; ++b)
    for (int y = 0; y < ho; ++y)
      for (int x = 0; x < wo; ++x)
        for (int ch = 0; ch < c; ++ch) {
          const float* p = in + (((size_t)b * h + 2 * y) * w + 2 * x) * c + ch;
          float m = p[0];
          float v1 = p[c], v2 = p[(size_t)w * c], v3 = p[(size_t)w * c + c];
          if (v1 > m) m = v1;
          if (v2 > m) m = v2;
          if (v3 > m) m = v3;
          out[(((size_t)b * ho + y) * wo + x) * c + ch] = m;
        }
}
