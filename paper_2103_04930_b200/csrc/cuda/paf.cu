// Bottom-up person assembly from part affinity fields (SURVEY.md §8 f, rank 4;
// after the x8 upsample and peak NMS of post.cu).
//
// Device: every candidate limb (peak a of part A, peak b of part B) of every
// limb type gets its PAF line integral in one thread:
//   d = B - A, u = d / |d|, 10 samples p_k = A + d * k/9 rounded to the
//   nearest pixel, s_k = PAF(p_k) . u, score = mean(s_k) + min(0.5 H / |d| - 1, 0),
//   valid = #(s_k > thr) >= 9 && score > 0
// in explicit _rn intrinsics, the op order of oracle/paf_oracle.c (bit-exact).
// Host (assemble_people, people.cpp): greedy matching per limb, then merging
// limbs into people.
#include <cstdint>

#include "engine.hpp"

namespace avec {

namespace {

constexpr int kMaxLimbs = 32;

struct LimbTable {
  int parts[2 * kMaxLimbs];
  int paf[2 * kMaxLimbs];
};

// grid (candidate a, limb); threads over candidate b
__global__ void paf_candidates_kernel(const float* __restrict__ paf, int H, int W, const int* __restrict__ counts,
                                      const float* __restrict__ peaks, int max_peaks, LimbTable t, float thr,
                                      float* __restrict__ cand) {
  const int a = blockIdx.x, l = blockIdx.y;
  const int pa = t.parts[2 * l], pb = t.parts[2 * l + 1];
  const int na = min(counts[pa], max_peaks), nb = min(counts[pb], max_peaks);
  const size_t plane = static_cast<size_t>(H) * W;
  const float* pxp = paf + static_cast<size_t>(t.paf[2 * l]) * plane;
  const float* pyp = paf + static_cast<size_t>(t.paf[2 * l + 1]) * plane;
  for (int b = threadIdx.x; b < max_peaks; b += blockDim.x) {
    float* c = cand + ((static_cast<size_t>(l) * max_peaks + a) * max_peaks + b) * 2;
    float score = 0.0f, valid = 0.0f;
    if (a < na && b < nb) {
      const float* A = peaks + (static_cast<size_t>(pa) * max_peaks + a) * 5;
      const float* B = peaks + (static_cast<size_t>(pb) * max_peaks + b) * 5;
      const float dx = __fsub_rn(B[0], A[0]), dy = __fsub_rn(B[1], A[1]);
      const float norm = __fsqrt_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)));
      if (norm > 0.0f) {
        const float ux = __fdiv_rn(dx, norm), uy = __fdiv_rn(dy, norm);
        float sum = 0.0f;
        int hits = 0;
#pragma unroll
        for (int k = 0; k < 10; ++k) {
          const float tk = __fdiv_rn(static_cast<float>(k), 9.0f);
          const float x = __fadd_rn(A[0], __fmul_rn(dx, tk)), y = __fadd_rn(A[1], __fmul_rn(dy, tk));
          int ix = __float2int_rn(x), iy = __float2int_rn(y);
          ix = ix < 0 ? 0 : ix >= W ? W - 1 : ix;
          iy = iy < 0 ? 0 : iy >= H ? H - 1 : iy;
          const size_t o = static_cast<size_t>(iy) * W + ix;
          const float s = __fadd_rn(__fmul_rn(__ldg(pxp + o), ux), __fmul_rn(__ldg(pyp + o), uy));
          sum = __fadd_rn(sum, s);
          hits += s > thr;
        }
        float prior = __fsub_rn(__fdiv_rn(__fmul_rn(0.5f, static_cast<float>(H)), norm), 1.0f);
        if (prior > 0.0f) prior = 0.0f;
        score = __fadd_rn(__fdiv_rn(sum, 10.0f), prior);
        valid = (hits >= 9 && score > 0.0f) ? 1.0f : 0.0f;
      }
    }
    c[0] = score;
    c[1] = valid;
  }
}

}  // namespace

void launch_paf_candidates(const float* d_paf, int H, int W, const int* d_counts, const float* d_peaks, int max_peaks,
                           const int* limb_parts, const int* limb_paf, int n_limbs, float thr, float* d_cand,
                           cudaStream_t stream) {
  if (n_limbs < 1 || n_limbs > kMaxLimbs) fail(AVEC_ERR_INVALID_ARGUMENT, "1..32 limb types");
  if (max_peaks < 1 || max_peaks > 65535) fail(AVEC_ERR_INVALID_ARGUMENT, "max_peaks out of range");
  LimbTable t{};
  for (int i = 0; i < 2 * n_limbs; ++i) {
    t.parts[i] = limb_parts[i];
    t.paf[i] = limb_paf[i];
  }
  dim3 grid(max_peaks, n_limbs);
  const int threads = max_peaks >= 128 ? 128 : (max_peaks + 31) / 32 * 32;
  paf_candidates_kernel<<<grid, threads, 0, stream>>>(d_paf, H, W, d_counts, d_peaks, max_peaks, t, thr, d_cand);
  check_cuda(cudaGetLastError(), "paf candidates launch");
}

}  // namespace avec
