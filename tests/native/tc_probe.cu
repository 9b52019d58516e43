// tcgen05 / TMA probe (test program, not product code).
//  1. correctness of our SW128 K-major descriptors + instruction descriptor:
//     D[128 x N] = A[128 x 64] * B[N x 64]^T via TMA -> smem -> tcgen05.mma -> TMEM
//  2. operand row offsets that are not multiples of 8 (the sliding-window trick
//     the conv kernel uses for the kw taps), with and without the descriptor's
//     base-offset field
//  3. raw MMA issue rate per SM for N = 64/128/256 (SS operands, M = 128)
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

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      std::printf("{\"ok\": false, \"error\": \"%s at %s:%d\"}\n", cudaGetErrorString(e), \
                  __FILE__, __LINE__);                                                \
      std::exit(1);                                                                   \
    }                                                                                 \
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

// one CTA, 128 threads
__global__ void probe_mma(const __grid_constant__ CUtensorMap mapA,
                          const __grid_constant__ CUtensorMap mapB, float* D, int N,
                          int b_row_off, int use_base_off) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                  // 128 rows x 128 B = 16 KB
  uint8_t* sB = smem + 16384;          // 384 rows x 128 B = 48 KB
  __shared__ uint64_t bar_full, bar_mma;
  __shared__ uint32_t tmem_base;
  if (warp_id() == 0) tmem_alloc<256>(&tmem_base);
  if (threadIdx.x == 0) {
    mbar_init(&bar_full, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar_full, 16384 + 3 * 16384);
    tma_load_2d(sA, &mapA, &bar_full, 0, 0);
    for (int i = 0; i < 3; ++i) tma_load_2d(sB + i * 16384, &mapB, &bar_full, 0, i * 128);
    mbar_wait(&bar_full, 0);
    tc_fence_after();
    const uint32_t idesc = idesc_bf16_f32(128, N);
    for (int k = 0; k < 4; ++k) {
      uint32_t a_addr = smem_u32(sA) + k * 32;
      uint32_t b_addr = smem_u32(sB) + b_row_off * 128 + k * 32;
      uint64_t ad = desc_sw128(a_addr);
      uint64_t bd = desc_sw128(b_addr, use_base_off ? ((b_addr >> 7) & 7) : 0);
      mma_bf16_ss(tbase, ad, bd, idesc, k > 0);
    }
    mma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  const uint32_t w = warp_id();
  for (int c = 0; c < N; c += 16) {
    uint32_t v[16];
    tmem_ld16(tbase + ((32 * w) << 16) + c, v);
    tmem_ld_wait();
    const int row = 32 * w + lane_id();
    for (int j = 0; j < 16; ++j) D[row * N + c + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<256>(tbase);
}

// issue-rate probe: one CTA per SM, thread 0 streams MMAs on resident smem
__global__ void probe_rate(int N, int iters, unsigned long long* cycles, int b_row_off = 0) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_mma;
  __shared__ uint32_t tmem_base;
  // zero operands so the datapath sees finite values
  for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp_id() == 0) tmem_alloc<256>(&tmem_base);
  if (threadIdx.x == 0) {
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, N);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 16384) + b_row_off * 128;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_bf16_ss(tmem_base, desc_sw128(a0 + k * 32), desc_sw128(b0 + k * 32), idesc, 1);
    }
    mma_commit(&bar_mma);
    mbar_wait(&bar_mma, 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<256>(tmem_base);
}

// per "k-block": 7 taps x 2 subs x 4 k-slices, A from a 16 KB weight tile,
// B from a 520-row window at row offset s (+256 for sub 1), like conv_tc_kernel<2>
__global__ void probe_conv_pattern(int kblocks, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar_mma;
  __shared__ uint32_t tmem_base;
  for (int i = threadIdx.x; i < (16384 + 66560) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp_id() == 0) tmem_alloc<512>(&tmem_base);
  if (threadIdx.x == 0) {
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, 256);
    const uint32_t a0 = smem_u32(smem), w0 = smem_u32(smem + 16384);
    long long t0 = clock64();
    for (int kb = 0; kb < kblocks; ++kb) {
      for (int s = 0; s < 7; ++s) {
#pragma unroll
        for (int sub = 0; sub < 2; ++sub)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_bf16_ss(tmem_base + sub * 256, desc_sw128(a0 + kk * 32),
                        desc_sw128(w0 + (sub * 256 + s) * 128 + kk * 32), idesc, 1);
      }
    }
    mma_commit(&bar_mma);
    mbar_wait(&bar_mma, 0);
    long long t1 = clock64();
    cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tmem_base);
}

int main() {
  const int M = 128, K = 64, BR = 264;
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
  CUtensorMap mA = make_map(dA, M, 128), mB = make_map(dB, BR, 128);
  const int smem = 1024 + 16384 + 49152;
  CK(cudaFuncSetAttribute(probe_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(probe_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));

  std::printf("{\"ok\": true, \"correctness\": [");
  bool first = true;
  std::vector<float> hD(M * 256);
  const int Ns[3] = {64, 128, 256};
  for (int ni = 0; ni < 3; ++ni) {
    for (int off = 0; off < 9; ++off) {
      for (int bo = 0; bo < 2; ++bo) {
        if (off == 0 && bo == 1) continue;
        int N = Ns[ni];
        if (N != 256 && off > 1) continue;
        CK(cudaMemset(dD, 0, M * 256 * 4));
        probe_mma<<<1, 128, smem>>>(mA, mB, dD, N, off, bo);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost));
        int bad = 0;
        double maxerr = 0;
        for (int i = 0; i < M; ++i)
          for (int j = 0; j < N; ++j) {
            float ref = 0;
            for (int k = 0; k < K; ++k) ref += fA[i * K + k] * fB[(j + off) * K + k];
            double e = std::fabs(ref - hD[i * N + j]);
            if (e > 0) ++bad;
            if (e > maxerr) maxerr = e;
          }
        std::printf("%s{\"N\": %d, \"row_off\": %d, \"base_off_field\": %d, \"bad\": %d, \"maxerr\": %g}",
                    first ? "" : ", ", N, off, bo, bad, maxerr);
        first = false;
      }
    }
  }
  std::printf("], \"rate\": [");
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long* dc;
  CK(cudaMalloc(&dc, sms * 8));
  std::vector<unsigned long long> hc(sms);
  const int Nr[9] = {64, 96, 128, 160, 176, 192, 208, 224, 256};
  for (int ni = 0; ni < 9; ++ni) {
    int N = Nr[ni], iters = 4096;
    probe_rate<<<sms, 128, smem>>>(N, 16, dc);  // warm
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe_rate<<<sms, 128, smem>>>(N, iters, dc);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    CK(cudaMemcpy(hc.data(), dc, sms * 8, cudaMemcpyDeviceToHost));
    double cyc = 0;
    for (int i = 0; i < sms; ++i) cyc += double(hc[i]);
    cyc /= sms;
    double flops = 2.0 * 128 * N * 16 * 4.0 * iters * sms;
    std::printf("%s{\"N\": %d, \"cycles_per_mma\": %.2f, \"ideal_cycles\": %.1f, \"tflops\": %.1f}",
                ni ? ", " : "", N, cyc / (4.0 * iters), 128.0 * N / 256.0, flops / (ms * 1e-3) / 1e12);
  }
  // operand B read at a row offset that is not a multiple of the 8-row swizzle atom
  std::printf("], \"rate_offset\": [");
  const int offs[5] = {0, 1, 3, 7, 8};
  for (int oi = 0; oi < 5; ++oi) {
    probe_rate<<<sms, 128, smem>>>(256, 4096, dc, offs[oi]);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hc.data(), dc, sms * 8, cudaMemcpyDeviceToHost));
    double cyc = 0;
    for (int i = 0; i < sms; ++i) cyc += double(hc[i]);
    std::printf("%s{\"N\": 256, \"b_row_off\": %d, \"cycles_per_mma\": %.2f}", oi ? ", " : "", offs[oi],
                cyc / sms / (4.0 * 4096));
  }
  // the conv kernel's exact operand pattern (weights A, 520-row window B, two subs, 7 taps)
  std::printf("], \"rate_conv_pattern\": [");
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaFuncSetAttribute(probe_conv_pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + 16384 + 66560));
    probe_conv_pattern<<<sms, 128, 1024 + 16384 + 66560>>>(512, dc);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hc.data(), dc, sms * 8, cudaMemcpyDeviceToHost));
    double cyc = 0;
    for (int i = 0; i < sms; ++i) cyc += double(hc[i]);
    std::printf("%s{\"cycles_per_mma_N256\": %.2f}", rep ? ", " : "", cyc / sms / (512.0 * 7 * 2 * 4));
  }
  std::printf("], \"sms\": %d}\n", sms);
  return 0;
}
