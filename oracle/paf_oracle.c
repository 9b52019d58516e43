/* CPU oracle for OpenPose person assembly from part affinity fields — TEST
 * INFRASTRUCTURE ONLY (SURVEY.md §8 f, rank 4: not in the reference, which
 * has no CNN; the semantics follow the public OpenPose bottom-up parsing:
 * PAF line integral per candidate limb, greedy bipartite matching per limb,
 * then merging limbs into people).
 *
 * Candidate score of limb l between peak a of part A and peak b of part B
 * (peak coordinates are the integer NMS peaks, x/y as floats):
 *   d = B - A, norm = sqrt(dx*dx + dy*dy); u = d / norm
 *   for k = 0..9: t = k / 9; p = A + d * t; (ix, iy) = round-half-even(p),
 *     clamped into the plane; s_k = paf_x[iy][ix] * ux + paf_y[iy][ix] * uy
 *   score = (sum_k s_k, left to right) / 10 + min(0.5 * H / norm - 1, 0)
 *   valid = norm > 0 && #(s_k > paf_thr) >= 9 && score > 0
 * Every operation is a single IEEE op in this order (-ffp-contract=off); the
 * CUDA kernel uses the matching _rn intrinsics, so scores are bit-exact.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "avec_oracle.h"

void oracle_paf_candidates(const float* paf, int H, int W, const int* counts, const float* peaks, int max_peaks,
                           const int* limb_parts, const int* limb_paf, int n_limbs, float paf_thr, float* cand) {
  for (int l = 0; l < n_limbs; ++l) {
    const int pa = limb_parts[2 * l], pb = limb_parts[2 * l + 1];
    const float* px_plane = paf + (long)limb_paf[2 * l] * H * W;
    const float* py_plane = paf + (long)limb_paf[2 * l + 1] * H * W;
    const int na = counts[pa] < max_peaks ? counts[pa] : max_peaks;
    const int nb = counts[pb] < max_peaks ? counts[pb] : max_peaks;
    for (int a = 0; a < max_peaks; ++a)
      for (int b = 0; b < max_peaks; ++b) {
        float* c = cand + (((long)l * max_peaks + a) * max_peaks + b) * 2;
        c[0] = 0.0f;
        c[1] = 0.0f;
        if (a >= na || b >= nb) continue;
        const float ax = peaks[((long)pa * max_peaks + a) * 5], ay = peaks[((long)pa * max_peaks + a) * 5 + 1];
        const float bx = peaks[((long)pb * max_peaks + b) * 5], by = peaks[((long)pb * max_peaks + b) * 5 + 1];
        const float dx = bx - ax, dy = by - ay;
        const float norm = sqrtf(dx * dx + dy * dy);
        if (!(norm > 0.0f)) continue;
        const float ux = dx / norm, uy = dy / norm;
        float sum = 0.0f;
        int hits = 0;
        for (int k = 0; k < 10; ++k) {
          const float t = (float)k / 9.0f;
          const float x = ax + dx * t, y = ay + dy * t;
          int ix = (int)nearbyintf(x), iy = (int)nearbyintf(y);
          ix = ix < 0 ? 0 : ix >= W ? W - 1 : ix;
          iy = iy < 0 ? 0 : iy >= H ? H - 1 : iy;
          const float s = px_plane[(long)iy * W + ix] * ux + py_plane[(long)iy * W + ix] * uy;
          sum = sum + s;
          hits += s > paf_thr;
        }
        float prior = 0.5f * (float)H / norm - 1.0f;
        if (prior > 0.0f) prior = 0.0f;
        const float score = sum / 10.0f + prior;
        c[0] = score;
        c[1] = (hits >= 9 && score > 0.0f) ? 1.0f : 0.0f;
      }
  }
}

/* ---- assembly: greedy per limb, then merge into people ------------------ */

typedef struct {
  float score;
  int a, b;
} Conn;

static int conn_cmp(const void* x, const void* y) {
  const Conn* p = (const Conn*)x;
  const Conn* q = (const Conn*)y;
  if (p->score > q->score) return -1;
  if (p->score < q->score) return 1;
  /* ties: lower (a, b) first, so the order is total and deterministic */
  if (p->a != q->a) return p->a < q->a ? -1 : 1;
  return p->b < q->b ? -1 : p->b > q->b ? 1 : 0;
}

/* people: [max_people][n_parts] peak index per part (-1 = none);
 * people_score: [max_people][2] = (total score, parts found). Limbs l >=
 * new_row_limbs never start a person. A person is kept when it has >= 4 parts
 * and total/parts >= 0.4. Returns the person count. */
int oracle_assemble_people(const int* counts, const float* peaks, int n_parts, int max_peaks, const float* cand,
                           const int* limb_parts, int n_limbs, int new_row_limbs, int max_people, int* people,
                           float* people_score) {
  const int cap = 4 * max_people + 64;
  int* rows = (int*)malloc(sizeof(int) * (size_t)cap * n_parts);
  float* rscore = (float*)malloc(sizeof(float) * (size_t)cap * 2);
  Conn* conns = (Conn*)malloc(sizeof(Conn) * (size_t)max_peaks * max_peaks);
  int* used_a = (int*)malloc(sizeof(int) * max_peaks);
  int* used_b = (int*)malloc(sizeof(int) * max_peaks);
  int nrows = 0;
  for (int l = 0; l < n_limbs; ++l) {
    const int pa = limb_parts[2 * l], pb = limb_parts[2 * l + 1];
    const int na = counts[pa] < max_peaks ? counts[pa] : max_peaks;
    const int nb = counts[pb] < max_peaks ? counts[pb] : max_peaks;
    int nc = 0;
    for (int a = 0; a < na; ++a)
      for (int b = 0; b < nb; ++b) {
        const float* c = cand + (((long)l * max_peaks + a) * max_peaks + b) * 2;
        if (c[1] != 0.0f) {
          conns[nc].score = c[0];
          conns[nc].a = a;
          conns[nc].b = b;
          ++nc;
        }
      }
    qsort(conns, (size_t)nc, sizeof(Conn), conn_cmp);
    memset(used_a, 0, sizeof(int) * max_peaks);
    memset(used_b, 0, sizeof(int) * max_peaks);
    const int limit = na < nb ? na : nb;
    int taken = 0;
    for (int i = 0; i < nc && taken < limit; ++i) {
      const int a = conns[i].a, b = conns[i].b;
      if (used_a[a] || used_b[b]) continue;
      used_a[a] = used_b[b] = 1;
      ++taken;
      const float sa = peaks[((long)pa * max_peaks + a) * 5 + 4];
      const float sb = peaks[((long)pb * max_peaks + b) * 5 + 4];
      int found = 0, idx[2] = {-1, -1};
      for (int j = 0; j < nrows && found < 2; ++j)
        if (rows[j * n_parts + pa] == a || rows[j * n_parts + pb] == b) idx[found++] = j;
      if (found == 1) {
        const int j = idx[0];
        if (rows[j * n_parts + pb] != b) {
          rows[j * n_parts + pb] = b;
          rscore[2 * j + 1] += 1.0f;
          rscore[2 * j] += sb + conns[i].score;
        }
      } else if (found == 2) {
        const int j1 = idx[0], j2 = idx[1];
        int overlap = 0;
        for (int p = 0; p < n_parts; ++p) overlap |= rows[j1 * n_parts + p] >= 0 && rows[j2 * n_parts + p] >= 0;
        if (!overlap) { /* merge j2 into j1 */
          for (int p = 0; p < n_parts; ++p)
            if (rows[j2 * n_parts + p] >= 0) rows[j1 * n_parts + p] = rows[j2 * n_parts + p];
          rscore[2 * j1] += rscore[2 * j2] + conns[i].score;
          rscore[2 * j1 + 1] += rscore[2 * j2 + 1];
          for (int r = j2; r + 1 < nrows; ++r) {
            memcpy(rows + r * n_parts, rows + (r + 1) * n_parts, sizeof(int) * n_parts);
            rscore[2 * r] = rscore[2 * (r + 1)];
            rscore[2 * r + 1] = rscore[2 * (r + 1) + 1];
          }
          --nrows;
        } else if (rows[j1 * n_parts + pb] != b) {
          rows[j1 * n_parts + pb] = b;
          rscore[2 * j1 + 1] += 1.0f;
          rscore[2 * j1] += sb + conns[i].score;
        }
      } else if (l < new_row_limbs && nrows < cap) { /* the redundant ear-shoulder limbs only extend people */
        for (int p = 0; p < n_parts; ++p) rows[nrows * n_parts + p] = -1;
        rows[nrows * n_parts + pa] = a;
        rows[nrows * n_parts + pb] = b;
        rscore[2 * nrows] = sa + sb + conns[i].score;
        rscore[2 * nrows + 1] = 2.0f;
        ++nrows;
      }
    }
  }
  int out = 0;
  for (int j = 0; j < nrows && out < max_people; ++j) {
    if (rscore[2 * j + 1] < 4.0f || rscore[2 * j] / rscore[2 * j + 1] < 0.4f) continue;
    memcpy(people + (long)out * n_parts, rows + (long)j * n_parts, sizeof(int) * n_parts);
    people_score[2 * out] = rscore[2 * j];
    people_score[2 * out + 1] = rscore[2 * j + 1];
    ++out;
  }
  free(rows);
  free(rscore);
  free(conns);
  free(used_a);
  free(used_b);
  return out;
}
