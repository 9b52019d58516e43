// tcgen05 CTA-pair probe (test program, not product code).
//  1. correctness of cta_group::2 MMA with our descriptors: a 2-CTA cluster,
//     each CTA holding 128 rows of A (M = 256 in total) and N/2 rows of B;
//     D[256 x N] = A * B^T lands as 128 rows x N in each CTA's TMEM
//  2. MMA rate per SM pair for N = 64/128/256 (SS operands, M = 256), to
//     compare with the single-CTA rates of tc_probe.cu (the shared-memory
//     operand path caps SS MMAs at 128 B/clk per SM; the pair reads each B
//     half once for both SMs)
// Prints one JSON object.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2103_04930_b200/csrc/cuda/ptx.cuh"

using namespace avec::ptx;

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      std::printf("{\"ok\": false, \"error\": \"%s at %s:%d\"}\n", cudaGetErrorString(e), \
                  __FILE__, __LINE__);                                                     \
      std::exit(1);                                                                        \
    }                                                                                      \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q));
  return reinterpret_cast<EncodeTiledFn>(fn);
}

static CUtensorMap make_map(void* base, uint64_t rows, uint32_t box_rows) {
  static EncodeTiledFn enc = get_encode();
  CUtensorMap m;
  cuuint64_t dims[2] = {64, rows};
  cuuint64_t strides[1] = {64 * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::printf("{\"ok\": false, \"error\": \"encode %d\"}\n", int(r));
    std::exit(1);
  }
  return m;
}

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc2(uint32_t* slot) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}

// one 2-CTA cluster, 128 threads per CTA
__global__ void __cluster_dims__(2, 1, 1) probe2_mma(const __grid_constant__ CUtensorMap mapA,
                                                     const __grid_constant__ CUtensorMap mapB, float* D,
                                                     int N) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;          // 128 rows x 128 B
  uint8_t* sB = smem + 16384;  // N/2 rows x 128 B
  __shared__ uint64_t bar_full, bar_mma;
  __shared__ uint32_t tmem_base;
  const uint32_t rank = cta_rank();
  if (warp_id() == 0) tmem_alloc2<256>(&tmem_base);
  if (threadIdx.x == 0) {
    mbar_init(&bar_full, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar_full, 16384 + (N / 2) * 128);
    tma_load_2d(sA, &mapA, &bar_full, 0, rank * 128);
    tma_load_2d(sB, &mapB, &bar_full, 0, rank * (N / 2));
    mbar_wait(&bar_full, 0);
  }
  cluster_sync();  // both halves resident
  if (rank == 0 && threadIdx.x == 0) {
    tc_fence_after();
    const uint32_t idesc = idesc_bf16_f32(256, N);
    for (int k = 0; k < 4; ++k)
      mma2(tbase, desc_sw128(smem_u32(sA) + k * 32), desc_sw128(smem_u32(sB) + k * 32), idesc, k > 0);
    commit2(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  const uint32_t w = warp_id();
  for (int c = 0; c < N; c += 16) {
    uint32_t v[16];
    tmem_ld16(tbase + ((32 * w) << 16) + c, v);
    tmem_ld_wait();
    const int row = rank * 128 + 32 * w + lane_id();
    for (int j = 0; j < 16; ++j) D[row * N + c + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  cluster_sync();
  if (warp_id() == 0) tmem_dealloc2<256>(tbase);
}

// rate: clusters of 2, the leader streams MMAs on resident (zeroed) operands
__global__ void __cluster_dims__(2, 1, 1) probe2_rate(int N, int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar_mma;
  __shared__ uint32_t tmem_base;
  for (int i = threadIdx.x; i < (16384 + 16384) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp_id() == 0) tmem_alloc2<256>(&tmem_base);
  if (threadIdx.x == 0) {
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (cta_rank() == 0 && threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(256, N);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 16384);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) mma2(tmem_base, desc_sw128(a0 + k * 32), desc_sw128(b0 + k * 32), idesc, 1);
    }
    commit2(&bar_mma);
    mbar_wait(&bar_mma, 0);
    long long t1 = clock64();
    cycles[blockIdx.x / 2] = (unsigned long long)(t1 - t0);
  } else if (threadIdx.x == 0) {
    mbar_wait(&bar_mma, 0);
  }
  tc_fence_before();
  cluster_sync();
  if (warp_id() == 0) tmem_dealloc2<256>(tmem_base);
}

// rate with conv_pm's operand pattern: A = a 264-row window read at row
// offsets sub*128 + s (s = the filter tap, sub = the 128-row sub-tile), two
// accumulators, B one [N/2][64] block per tap; off_mode 0 = no row shift (s = 0)
__global__ void __cluster_dims__(2, 1, 1) probe2_rate_conv(int N, int iters, int off_mode, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar_mma;
  __shared__ uint32_t tmem_base;
  constexpr int kWin = 272 * 128, kB = 3 * 16384;
  for (int i = threadIdx.x; i < (kWin + kB) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp_id() == 0) tmem_alloc2<512>(&tmem_base);
  if (threadIdx.x == 0) {
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (cta_rank() == 0 && threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(256, N);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + kWin);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const uint64_t bd = desc_sw128(b0 + s * 16384);
#pragma unroll
        for (int sub = 0; sub < 2; ++sub) {
          const uint64_t ad = desc_sw128(a0 + (sub * 128 + (off_mode ? s : 0)) * 128);
#pragma unroll
          for (int k = 0; k < 4; ++k) mma2(tmem_base + sub * N, ad + 2 * k, bd + 2 * k, idesc, 1);
        }
      }
    }
    commit2(&bar_mma);
    mbar_wait(&bar_mma, 0);
    long long t1 = clock64();
    cycles[blockIdx.x / 2] = (unsigned long long)(t1 - t0);
  } else if (threadIdx.x == 0) {
    mbar_wait(&bar_mma, 0);
  }
  tc_fence_before();
  cluster_sync();
  if (warp_id() == 0) tmem_dealloc2<512>(tmem_base);
}

int main() {
  const int M = 256, K = 64, BR = 256;
  std::vector<__nv_bfloat16> hA(M * K), hB(BR * K);
  std::vector<float> fA(M * K), fB(BR * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) {
    float v = float(rand() % 9 - 4);
    hA[i] = __float2bfloat16(v);
    fA[i] = v;
  }
  for (int i = 0; i < BR * K; ++i) {
    float v = float(rand() % 7 - 3);
    hB[i] = __float2bfloat16(v);
    fB[i] = v;
  }
  __nv_bfloat16 *dA, *dB;
  float* dD;
  CK(cudaMalloc(&dA, hA.size() * 2));
  CK(cudaMalloc(&dB, hB.size() * 2));
  CK(cudaMalloc(&dD, M * 256 * 4));
  CK(cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice));
  const int smem = 1024 + 16384 + 16384;
  CK(cudaFuncSetAttribute(probe2_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe2_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));

  std::printf("{\"ok\": true, \"correctness\": [");
  std::vector<float> hD(M * 256);
  const int Ns[3] = {64, 128, 256};
  for (int ni = 0; ni < 3; ++ni) {
    const int N = Ns[ni];
    CUtensorMap mA = make_map(dA, M, 128), mB = make_map(dB, BR, N / 2);
    CK(cudaMemset(dD, 0, M * 256 * 4));
    probe2_mma<<<2, 128, smem>>>(mA, mB, dD, N);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    double maxerr = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        float ref = 0;
        for (int k = 0; k < K; ++k) ref += fA[i * K + k] * fB[j * K + k];
        const double e = std::fabs(ref - hD[i * N + j]);
        if (e > maxerr) maxerr = e;
        bad += e > 1e-3;
      }
    std::printf("%s{\"N\": %d, \"bad\": %d, \"max_err\": %g}", ni ? ", " : "", N, bad, maxerr);
  }
  std::printf("], \"rate\": [");
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int pairs = sms / 2;
  unsigned long long* dc;
  CK(cudaMalloc(&dc, pairs * sizeof(unsigned long long)));
  std::vector<unsigned long long> hc(pairs);
  const int Nr[7] = {32, 48, 64, 80, 96, 128, 256};
  for (int ni = 0; ni < 7; ++ni) {
    const int N = Nr[ni], iters = 2000;
    probe2_rate<<<2 * pairs, 128, smem>>>(N, iters, dc);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hc.data(), dc, pairs * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    double avg = 0;
    for (auto c : hc) avg += double(c);
    avg /= pairs;
    const double per_mma = avg / (iters * 4.0);
    // per SM: 128 x N x 16 MACs per MMA; ideal 8192 FLOP/clk/SM -> 128*N*16*2/8192 = N/2 clk
    std::printf("%s{\"N\": %d, \"cycles_per_mma\": %.2f, \"ideal\": %.1f}", ni ? ", " : "", N, per_mma,
                N / 2.0);
  }
  std::printf("], \"rate_conv\": [");
  const int smem_conv = 120 * 1024;  // > half the SM: one CTA (and one 512-column TMEM allocation) per SM
  CK(cudaFuncSetAttribute(probe2_rate_conv, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_conv));
  const int Nc[3] = {96, 128, 256};
  bool firstc = true;
  for (int ni = 0; ni < 3; ++ni)
    for (int om = 0; om < 2; ++om) {
      const int N = Nc[ni], iters = 500;
      probe2_rate_conv<<<2 * pairs, 128, smem_conv>>>(N, iters, om, dc);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(hc.data(), dc, pairs * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      double avg = 0;
      for (auto c : hc) avg += double(c);
      avg /= pairs;
      std::printf("%s{\"N\": %d, \"row_shift\": %d, \"cycles_per_mma\": %.2f, \"ideal\": %.1f}", firstc ? "" : ", ",
                  N, om, avg / (iters * 24.0), N / 2.0);
      firstc = false;
    }
  std::printf("]}\n");
  return 0;
}
