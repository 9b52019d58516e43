// MockPose forward on the B200: out[j] = f32(mean(x[lo_j:hi_j])) with the
// reference's exact arithmetic (proj/src/backend.cpp:39-67):
//   width = double(E) / double(K)                 (computed once on the host)
//   hi_j  = (j+1 == K) ? E : uint64(double(j+1) * width)
//   sum   = left-to-right double accumulation, mean = sum / double(hi-lo)
// Explicit _rn intrinsics keep the device op sequence identical to the CPU's,
// so the result is bit-exact (tests/test_gpu_mockpose.py).
//
// HBM-bound: 4E bytes read + 4K bytes written per frame. Each CTA stages its
// contiguous input span in shared memory with 16-byte loads, then every thread
// walks four (short) segments in order.
#include <cstdint>

#include "engine.hpp"

namespace avec {

namespace {

constexpr int kThreads = 256;
constexpr int kSegsPerThread = 4;  // segments per thread (interleaved by kThreads)
constexpr int kSegsPerCta = kThreads * kSegsPerThread;

__device__ __forceinline__ uint64_t seg_bound(uint64_t j, uint64_t K, uint64_t E, double width) {
  // boundary j is the start of segment j; boundary K is E
  if (j == 0) return 0;
  if (j >= K) return E;
  return __double2ull_rz(__dmul_rn(static_cast<double>(j), width));
}

__device__ __forceinline__ float seg_mean(const float* x, uint64_t lo, uint64_t hi) {
  double sum = 0.0;
  for (uint64_t i = lo; i < hi; ++i) sum = __dadd_rn(sum, static_cast<double>(x[i]));
  return __double2float_rn(__ddiv_rn(sum, static_cast<double>(hi - lo)));
}

// staged: each CTA copies the contiguous input span of its kSegsPerCta
// segments into shared memory (sized to the span: occupancy is bounded by
// threads, not by a worst-case static buffer), then thread t walks segments
// t, t + 256, ... so neighbouring lanes read neighbouring words.
__global__ void __launch_bounds__(kThreads) segmean_staged(const float* __restrict__ in,
                                                           float* __restrict__ out, uint64_t E,
                                                           uint64_t K, double width) {
  extern __shared__ __align__(16) float stage[];
  const uint64_t j0 = static_cast<uint64_t>(blockIdx.x) * kSegsPerCta;
  const uint64_t j1 = j0 + kSegsPerCta < K ? j0 + kSegsPerCta : K;
  const uint64_t span_lo = seg_bound(j0, K, E, width);
  const uint64_t span_hi = seg_bound(j1, K, E, width);
  // align the staged window down to 16 B so the bulk of it moves as float4
  const uint64_t base = span_lo & ~uint64_t(3);
  const uint64_t n = span_hi - base;
  const uint64_t n4 = n >> 2;
  const float4* src4 = reinterpret_cast<const float4*>(in + base);
  float4* dst4 = reinterpret_cast<float4*>(stage);
  for (uint64_t i = threadIdx.x; i < n4; i += kThreads) dst4[i] = __ldg(src4 + i);
  for (uint64_t i = (n4 << 2) + threadIdx.x; i < n; i += kThreads) stage[i] = __ldg(in + base + i);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSegsPerThread; ++r) {
    const uint64_t j = j0 + threadIdx.x + static_cast<uint64_t>(r) * kThreads;
    if (j < K) {
      const uint64_t lo = seg_bound(j, K, E, width), hi = seg_bound(j + 1, K, E, width);
      out[j] = seg_mean(stage - base, lo, hi);
    }
  }
}

// general: wide segments (large divisors) read straight from global/L1
__global__ void __launch_bounds__(kThreads) segmean_direct(const float* __restrict__ in,
                                                           float* __restrict__ out, uint64_t E,
                                                           uint64_t K, double width) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x;
  if (j >= K) return;
  const uint64_t lo = seg_bound(j, K, E, width), hi = seg_bound(j + 1, K, E, width);
  out[j] = seg_mean(in, lo, hi);
}

}  // namespace

void launch_segment_means(const float* d_in, float* d_out, uint64_t E, uint64_t K,
                          cudaStream_t stream) {
  const double width = static_cast<double>(E) / static_cast<double>(K);
  // a CTA spans at most ceil(kSegsPerCta * width) + 1 inputs (+3 for alignment)
  const double span = width * kSegsPerCta + 8;
  if (span * 4 <= 48 * 1024) {
    const uint64_t blocks = (K + kSegsPerCta - 1) / kSegsPerCta;
    const size_t smem = static_cast<size_t>(span) * 4 + 16;
    segmean_staged<<<static_cast<unsigned>(blocks), kThreads, smem, stream>>>(d_in, d_out, E, K, width);
  } else {
    const uint64_t blocks = (K + kThreads - 1) / kThreads;
    segmean_direct<<<static_cast<unsigned>(blocks), kThreads, 0, stream>>>(d_in, d_out, E, K, width);
  }
  check_cuda(cudaGetLastError(), "segment means launch");
}

}  // namespace avec
