/* CPU oracle for the AVEC server-side hot path — TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker. The product path never links it
 * and fails loudly when its CUDA library is missing.
 *
 * Parity is pinned: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by the reference library itself
 * (oracle/ref_drivers/ref_golden.cpp -> tests/golden/reference_golden.json).
 */
#ifndef AVEC_ORACLE_H
#define AVEC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- sizing law: proj/src/wire.cpp:18-27 ---- */
uint64_t oracle_output_elems(uint64_t input_elems, double divisor);
uint64_t oracle_transfer_size(uint32_t n, uint32_t c, uint32_t h, uint32_t w, double divisor);

/* ---- segment means: proj/src/backend.cpp:39-67 ----
 * returns 0 ok, 1 empty input, 2 degenerate output (k<1 or k>e) */
int oracle_segment_means(const float* data, uint64_t e, double divisor, double* out, uint64_t k);
int oracle_mockpose_forward(const float* data, uint64_t e, double divisor, float* out, uint64_t k);

/* ---- harness generators: proj/src/harness.cpp:29-42, 355-370 ---- */
void oracle_gen_frame(uint64_t seed, uint32_t index, uint32_t width, uint32_t height, float* out);
/* little-endian bytes of successive mt19937_64(seed) draws: structure then weights */
void oracle_synth_blobs(uint64_t seed, uint8_t* structure, size_t sn, uint8_t* weights, size_t wn);

/* ---- OpenPose net oracle (build-only; no reference counterpart) ---- */
/* worker threads used by the conv oracle (AVEC_ORACLE_THREADS, default nproc) */
int oracle_threads(void);
/* bf16 round-to-nearest-even of an fp32 value, returned as fp32 */
float oracle_bf16_round(float x);
/* One conv layer on NHWC fp32 activations (values already bf16-representable),
 * weights in wire order W[cout][cin][kh][kw] fp32, bias[cout]; act 0 none,
 * 1 ReLU, 2 PReLU with per-channel `slope` (may be NULL otherwise).
 * Output NHWC fp32 with `out_round_bf16` choosing bf16 RNE rounding.
 * Accumulates each output in double. */
void oracle_conv2d_nhwc(const float* in, int n, int h, int w, int cin,
                        const float* weight, const float* bias, int cout, int k,
                        int act, const float* slope, int out_round_bf16, float* out);
/* Selected output rows: out[r][w][cout] from the k-row input window
 * win[r][k][w][cin] of each row (rows outside the image zero-filled by the
 * caller); identical arithmetic to oracle_conv2d_nhwc. */
void oracle_conv2d_rows(const float* win, int n_rows, int k, int w, int cin, const float* weight,
                        const float* bias, int cout, int act, const float* slope, int out_round_bf16,
                        float* out);
void oracle_maxpool2_nhwc(const float* in, int n, int h, int w, int c, float* out);

/* ---- post-processing oracle ---- */
/* bilinear x`scale` resize of one fp32 plane (h,w) -> (h*scale, w*scale),
 * half-pixel centres, edge clamp; exact op sequence of the CUDA kernel */
void oracle_upsample_plane(const float* in, int h, int w, int scale, float* out);
/* 3x3 NMS on one plane: a peak is > threshold and strictly > its 8 neighbours
 * (out-of-plane neighbours ignored). Writes up to max_peaks (x, y, score) in
 * raster order plus 3x3 weighted-average refined coordinates. Returns count. */
/* PAF candidate scores [n_limbs][max_peaks][max_peaks][2] = (score, valid)
 * and person assembly (oracle/paf_oracle.c). */
void oracle_paf_candidates(const float* paf, int H, int W, const int* counts, const float* peaks, int max_peaks,
                           const int* limb_parts, const int* limb_paf, int n_limbs, float paf_thr, float* cand);
int oracle_assemble_people(const int* counts, const float* peaks, int n_parts, int max_peaks, const float* cand,
                           const int* limb_parts, int n_limbs, int new_row_limbs, int max_people, int* people,
                           float* people_score);
int oracle_nms_plane(const float* in, int h, int w, float threshold, int max_peaks,
                     int* peak_xy, float* peak_refined_xy, float* peak_score);

#ifdef __cplusplus
}
#endif
#endif
