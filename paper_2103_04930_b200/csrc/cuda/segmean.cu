// MockPose forward on the B200: out[j] = f32(mean(x[lo_j:hi_j])) with the
// reference's exact arithmetic (proj/src/backend.cpp:39-67):
//   width = double(E) / double(K)                 (computed once on the host)
//   hi_j  = (j+1 == K) ? E : uint64(double(j+1) * width)
//   sum   = left-to-right double accumulation, mean = sum / double(hi-lo)
// Explicit _rn intrinsics keep the device op sequence identical to the CPU's,
// so the result is bit-exact (tests/test_gpu_mockpose.py).
//
// The division: for short segments (n <= MAXN) sum / n is taken as
//   q = RN(sum * y), r = fma(-q, n, sum) (exact), q' = RN(fma(r, y, q)),
// y = RN(1/n) from a per-CTA table. With y correctly rounded and q within an
// ulp of sum/n, q' is the correctly rounded quotient (Markstein's theorem),
// i.e. exactly __ddiv_rn(sum, n); 2e8 random sums of 1..8 floats over wide
// exponent ranges agreed bit for bit on the host. Three FP64 ops instead of
// the division sequence, which made the kernel instruction-bound.
// Non-finite sums and empty segments keep __ddiv_rn (inf - inf, 0 * inf).
//
// HBM-bound: 4E bytes read + 4K bytes written per frame. Each CTA stages its
// contiguous input span in shared memory by a bulk copy, then every thread
// walks four (short) segments in order.
#include <cmath>
#include <cstdint>

#include "engine.hpp"
#include "ptx.cuh"

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
template <int MAXN>  // longest segment (0: any length, loop)
__global__ void __launch_bounds__(kThreads) segmean_staged(const float* __restrict__ in,
                                                           float* __restrict__ out, uint64_t E,
                                                           uint64_t K, double width, uint64_t jbeg,
                                                           uint64_t jend) {
  __shared__ uint32_t bnd[kSegsPerCta + 1];  // segment boundaries, offsets into the stage
  __shared__ double rcp[MAXN + 1];           // RN(1 / n)
  extern __shared__ __align__(16) float stage[];
  if (MAXN > 0 && threadIdx.x >= 1 && threadIdx.x <= MAXN)
    rcp[threadIdx.x] = __ddiv_rn(1.0, static_cast<double>(threadIdx.x));
  const uint64_t j0 = jbeg + static_cast<uint64_t>(blockIdx.x) * kSegsPerCta;
  const uint64_t j1 = j0 + kSegsPerCta < jend ? j0 + kSegsPerCta : jend;
  const uint64_t span_lo = seg_bound(j0, K, E, width);
  const uint64_t span_hi = seg_bound(j1, K, E, width);
  // align the staged window down to 16 B so the bulk of it moves as float4
  const uint64_t base = span_lo & ~uint64_t(3);
  const uint32_t n = static_cast<uint32_t>(span_hi - base);
  const uint32_t n4 = n >> 2;
  // the 16-byte body of the span arrives by one bulk copy (no per-thread
  // load -> store round trips; the boundaries below are computed while it
  // lands), the < 4-float tail by plain loads
  __shared__ uint64_t landed;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&landed, 1);
    ptx::fence_barrier_init();
    if (n4) {
      ptx::mbar_arrive_expect_tx(&landed, n4 << 4);
      ptx::bulk_load(stage, in + base, n4 << 4, &landed);
    } else {
      ptx::mbar_arrive(&landed);
    }
  }
  for (uint32_t i = (n4 << 2) + threadIdx.x; i < n; i += kThreads) stage[i] = __ldg(in + base + i);
  // every boundary once (segment j spans [bnd[j - j0], bnd[j - j0 + 1]) of the stage),
  // 32-bit offsets from here on: a staged span is < 12K floats
  const uint32_t nb = static_cast<uint32_t>(j1 - j0);
  if (E <= 0xffffffffull) {
    // 32-bit boundaries (every FrameData: E < 2^29): the same products
    // double(j) * width truncated, j and the result exact in 32 bits
    // (j = 0 needs no case: 0 * width truncates to 0); computed for every j
    // and selected, so the loop is straight-line
    const uint32_t jb = static_cast<uint32_t>(j0), k32 = static_cast<uint32_t>(K);
    const uint32_t e32 = static_cast<uint32_t>(E), b32 = static_cast<uint32_t>(base);
#pragma unroll
    for (int rr = 0; rr <= kSegsPerThread; ++rr) {
      const uint32_t b = threadIdx.x + static_cast<uint32_t>(rr) * kThreads;
      if (b <= nb) {
        const uint32_t j = jb + b;
        const uint32_t prod = __double2uint_rz(__dmul_rn(__uint2double_rn(j), width));
        bnd[b] = (j >= k32 ? e32 : prod) - b32;
      }
    }
  } else {
    for (uint32_t b = threadIdx.x; b <= nb; b += kThreads)
      bnd[b] = static_cast<uint32_t>(seg_bound(j0 + b, K, E, width) - base);
  }
  __syncthreads();
  ptx::mbar_wait(&landed, 0);
#pragma unroll
  for (int r = 0; r < kSegsPerThread; ++r) {
    const uint32_t jl = threadIdx.x + static_cast<uint32_t>(r) * kThreads;
    if (jl < nb) {
      const uint32_t lo = bnd[jl], hi = bnd[jl + 1];
      double sum = 0.0;
      if constexpr (MAXN > 0) {
        // straight-line: MAXN >= every segment's length; the missing terms
        // add -0.0, the exact identity of IEEE addition (x + -0 == x for every
        // x, -0 included), so the sum is the reference's left-to-right one
#pragma unroll
        for (uint32_t i = 0; i < MAXN; ++i) {
          const float x = lo + i < hi ? stage[lo + i] : -0.0f;
          sum = __dadd_rn(sum, static_cast<double>(x));
        }
        const uint32_t cnt = hi - lo;
        const double n = static_cast<double>(cnt);
        double mean;
        if (cnt != 0 && isfinite(sum)) {
          const double y = rcp[cnt];
          const double q = __dmul_rn(sum, y);
          mean = __fma_rn(__fma_rn(-q, n, sum), y, q);
        } else {
          mean = __ddiv_rn(sum, n);
        }
        out[j0 + jl] = __double2float_rn(mean);
      } else {
        for (uint32_t i = lo; i < hi; ++i) sum = __dadd_rn(sum, static_cast<double>(stage[i]));
        out[j0 + jl] = __double2float_rn(__ddiv_rn(sum, static_cast<double>(hi - lo)));
      }
    }
  }
}

// general: wide segments (large divisors) read straight from global/L1
__global__ void __launch_bounds__(kThreads) segmean_direct(const float* __restrict__ in,
                                                           float* __restrict__ out, uint64_t E,
                                                           uint64_t K, double width, uint64_t jbeg,
                                                           uint64_t jend) {
  const uint64_t j = jbeg + static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x;
  if (j >= jend) return;
  const uint64_t lo = seg_bound(j, K, E, width), hi = seg_bound(j + 1, K, E, width);
  out[j] = seg_mean(in, lo, hi);
}

}  // namespace

uint64_t segment_bound(uint64_t j, uint64_t E, uint64_t K) {
  // the device's seg_bound on the host: same IEEE product, truncated
  if (j == 0) return 0;
  if (j >= K) return E;
  const double width = static_cast<double>(E) / static_cast<double>(K);
  return static_cast<uint64_t>(static_cast<double>(j) * width);
}

void launch_segment_means(const float* d_in, float* d_out, uint64_t E, uint64_t K, cudaStream_t stream,
                          uint64_t jbeg, uint64_t jend) {
  if (jend > K) jend = K;
  if (jbeg >= jend) return;
  const double width = static_cast<double>(E) / static_cast<double>(K);
  const uint64_t segs = jend - jbeg;
  // a CTA spans at most ceil(kSegsPerCta * width) + 1 inputs (+3 for alignment)
  const double span = width * kSegsPerCta + 8;
  if (span * 4 <= 44 * 1024) {  // + 4 KB of static boundary table
    const uint64_t blocks = (segs + kSegsPerCta - 1) / kSegsPerCta;
    const size_t smem = static_cast<size_t>(span) * 4 + 16;
    // segment lengths are floor((j+1)w) - floor(jw) <= ceil(w)
    const int maxn = static_cast<int>(std::ceil(width));
    const unsigned g = static_cast<unsigned>(blocks);
    auto go = [&](auto kernel) { kernel<<<g, kThreads, smem, stream>>>(d_in, d_out, E, K, width, jbeg, jend); };
    if (maxn <= 2) go(segmean_staged<2>);
    else if (maxn <= 4) go(segmean_staged<4>);
    else if (maxn <= 6) go(segmean_staged<6>);
    else if (maxn <= 8) go(segmean_staged<8>);
    else go(segmean_staged<0>);
  } else {
    const uint64_t blocks = (segs + kThreads - 1) / kThreads;
    segmean_direct<<<static_cast<unsigned>(blocks), kThreads, 0, stream>>>(d_in, d_out, E, K, width, jbeg, jend);
  }
  check_cuda(cudaGetLastError(), "segment means launch");
}

}  // namespace avec
