// conv1_1 fused with the wire-format input conversion (sm_100a).
//
// The first layer has 3 input channels (K = 27), too thin to stream through
// the implicit-GEMM kernels, and a separate im2col pass costs a full
// 64-channel round trip through HBM (write + read 128 B per pixel). Here each
// CTA builds the im2col tile IN SHARED MEMORY and feeds it straight to the
// tensor cores:
//
//   fp32 NCHW frame (wire layout) --27 coalesced loads per pixel--> (x - 0.5)
//   -> bf16 -> A tile [128 px][64 ch] (taps ci*9 + r*3 + s, zeros beyond 27;
//   128B-swizzled K-major) --2 x tcgen05.mma M128 N64 K16--> TMEM
//   -> bias, activation, zero outside the image, bf16 -> per-warp staging box
//   -> TMA store of [32 px][64 ch] into the level-0 padded-flat NHWC buffer.
//
// HBM traffic per pixel: 12 B read (each input float is reused by 9 taps
// through L1) + 128 B written — the floor for this layer. The MMA, with its
// weights resident in smem for the CTA's lifetime, is negligible. Load latency
// is hidden by gathering each tile's taps one tile ahead (in registers) and by
// several co-resident CTAs per SM.
// Results are bit-identical to the im2col + 1x1 path it replaces (same bf16
// operands, same K order, same MMA shape).
//
// TF32 (a net whose spec says "input tf32"): the A row is the 27 taps as fp32
// rounded to tf32 (cvt.rna) plus 5 zeros, 32 floats = one 128-byte SW128 row,
// the weights [64 cout][32] tf32, and K = 32 runs as four kind::tf32 M128 N64
// K8 MMAs; same tile, staging and epilogue.
#include <cuda_bf16.h>

#include "conv_tc.cuh"
#include "engine.hpp"
#include "ptx.cuh"

namespace avec {

namespace {

using namespace ptx;

constexpr int kFThreads = 128;
constexpr int kFCtasPerSm = 4;
constexpr uint32_t kFTmemCols = 64;

struct FirstSmem {
  static constexpr int a = 0;                  // [128][64] bf16, SW128 (16 KB)
  static constexpr int w = a + 128 * 128;      // [64 cout][64 K] bf16, SW128 (8 KB)
  static constexpr int stg = w + 64 * 128;     // 4 warps x [32 px][64 ch] (16 KB)
  static constexpr int bias = stg + 4 * 32 * 128;
  static constexpr int slope = bias + 64 * 4;
  static constexpr int bars = slope + 64 * 4;  // w_full, mma_done
  static constexpr int total = bars + 64;
};

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <bool TF32>
__global__ void __launch_bounds__(kFThreads, kFCtasPerSm)
    conv_first_kernel(const __grid_constant__ ConvMaps maps, const __grid_constant__ ConvParams p,
                      const float* __restrict__ frames) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* sa = smem + FirstSmem::a;
  uint8_t* sw = smem + FirstSmem::w;
  float* sbias = reinterpret_cast<float*>(smem + FirstSmem::bias);
  float* sslope = reinterpret_cast<float*>(smem + FirstSmem::slope);
  uint64_t* w_full = reinterpret_cast<uint64_t*>(smem + FirstSmem::bars);
  uint64_t* mma_done = w_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_done + 1);

  const int tid = int(threadIdx.x);
  const uint32_t warp = warp_id(), lane = lane_id();
  const ConvGroupParams& g = p.g[0];
  if (tid == 0) {
    mbar_init(w_full, 1);
    mbar_init(mma_done, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<kFTmemCols>(tmem_slot);
  if (tid < 64) {
    sbias[tid] = tid < g.cout ? g.bias[tid] : 0.f;
    sslope[tid] = g.act == 1 ? 0.f : (g.act == 2 && tid < g.cout) ? g.slope[tid] : 1.f;
  }
  // K channels 32..63 of the A tile are always zero: write them once
  if (!TF32) {
    uint8_t* row = sa + tid * 128;
#pragma unroll
    for (int q = 4; q < 8; ++q) *reinterpret_cast<uint4*>(row + ((q ^ (tid & 7)) << 4)) = make_uint4(0, 0, 0, 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tid == 0) {
    mbar_arrive_expect_tx(w_full, 64 * 128);
    tma_load_2d(sw, &maps.wgt[0], w_full, 0, 0);
  }

  const int HW = p.H * p.W;
  const bool relu = g.act == 1;
  uint32_t phase = 0;
  bool first = true;
  uint8_t* stg = smem + FirstSmem::stg + warp * (32 * 128);
  // The 27 taps of this thread's pixel in tile t, normalised (x - 0.5), zero
  // outside the frame. Gathered one tile AHEAD: the loads for tile t+grid are
  // in flight while tile t's MMA and epilogue run.
  float x[27];
  auto gather = [&](int t) {
    const int n = t / p.tiles_per_image;
    const int o = (t - n * p.tiles_per_image) * 128 + tid;
    const int hh = o / p.Wp;
    const int ww = o - hh * p.Wp;
    const bool valid = hh < p.H && ww < p.W;
    const float* img = frames + static_cast<size_t>(n) * 3 * HW;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int yy = hh + r - 1;
      const bool rv = valid && yy >= 0 && yy < p.H;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int xx = ww + s - 1;
        const bool v = rv && xx >= 0 && xx < p.W;
        const float* q = img + yy * p.W + xx;
#pragma unroll
        for (int ci = 0; ci < 3; ++ci) x[ci * 9 + r * 3 + s] = v ? __ldg(q + ci * HW) - 0.5f : 0.f;
      }
    }
  };
  if (int(blockIdx.x) < p.total_tiles) gather(blockIdx.x);
  for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
    const int n = t / p.tiles_per_image;
    const int o = (t - n * p.tiles_per_image) * 128 + tid;  // padded-width output position
    const int hh = o / p.Wp;
    const int ww = o - hh * p.Wp;
    const bool valid = hh < p.H && ww < p.W;
    // ---- im2col row of this pixel: taps k = ci*9 + r*3 + s
    if constexpr (TF32) {
      float v[32];
#pragma unroll
      for (int i = 0; i < 27; ++i) v[i] = to_tf32(x[i]);
#pragma unroll
      for (int i = 27; i < 32; ++i) v[i] = 0.f;
      uint8_t* row = sa + tid * 128;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(row + ((q ^ (tid & 7)) << 4)) =
            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
      uint32_t packed[16];
#pragma unroll
      for (int i = 0; i < 13; ++i) packed[i] = pack2(x[2 * i], x[2 * i + 1]);
      packed[13] = __bfloat16_as_ushort(__float2bfloat16_rn(x[26]));
      packed[14] = packed[15] = 0;
      uint8_t* row = sa + tid * 128;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<uint4*>(row + ((q ^ (tid & 7)) << 4)) =
            make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();  // A tile complete; the previous tile's TMEM reads are done
    if (tid == 0) {
      tc_fence_after();
      if (first) mbar_wait(w_full, 0);
      const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sw);
      if constexpr (TF32) {
        const uint32_t idesc = idesc_tf32_f32(128, 64);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // K = 32 fp32 = the 128-byte row, 8 per MMA
          mma_tf32_ss(tmem, desc_sw128(a0 + kk * 32), desc_sw128(b0 + kk * 32), idesc, kk ? 1u : 0u);
      } else {
        const uint32_t idesc = idesc_bf16_f32(128, 64);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)  // K = 32 covers the 27 taps
          mma_bf16_ss(tmem, desc_sw128(a0 + kk * 32), desc_sw128(b0 + kk * 32), idesc, kk ? 1u : 0u);
      }
      mma_commit(mma_done);
    }
    first = false;
    if (t + int(gridDim.x) < p.total_tiles) gather(t + gridDim.x);  // next tile's taps
    mbar_wait(mma_done, phase);
    phase ^= 1;
    tc_fence_after();
    // ---- epilogue: lane = pixel, 64 channels
    uint32_t va[32], vb[32];
    tmem_ld32(tmem + ((warp * 32) << 16), va);
    tmem_ld32(tmem + ((warp * 32) << 16) + 32, vb);
    tmem_ld_wait();
    if (lane == 0) bulk_wait_read<0>();  // this warp's previous store has read the staging box
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = q * 8 + 2 * j;
        float a = __uint_as_float(q < 4 ? va[c] : vb[c - 32]) + sbias[c];
        float b = __uint_as_float(q < 4 ? va[c + 1] : vb[c - 31]) + sbias[c + 1];
        if (relu) {
          a = fmaxf(a, 0.f);
          b = fmaxf(b, 0.f);
        } else {
          a = fmaxf(a, 0.f) + sslope[c] * fminf(a, 0.f);
          b = fmaxf(b, 0.f) + sslope[c + 1] * fminf(b, 0.f);
        }
        w[j] = valid ? pack2(a, b) : 0u;
      }
      *reinterpret_cast<uint4*>(stg + lane * 128 + ((q ^ (lane & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      const int row = p.P * p.Wp + p.P + o;  // lane 0's output row (rows past the image are clipped)
      tma_store_3d(&maps.out[0], stg, g.out_c_off, row, n);
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait<0>();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<kFTmemCols>(tmem);
  }
}

}  // namespace

void conv_first_configure() {
  check_cuda(cudaFuncSetAttribute(conv_first_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  FirstSmem::total + 1024),
             "conv_first smem attribute");
  check_cuda(cudaFuncSetAttribute(conv_first_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  FirstSmem::total + 1024),
             "conv_first smem attribute");
}

void launch_conv_first(const ConvMaps& maps, const ConvParams& p, const float* frames, int sm_count,
                       cudaStream_t stream) {
  const int cap = sm_count * kFCtasPerSm;
  const int grid = p.total_tiles < cap ? p.total_tiles : cap;
  if (p.tf32)
    conv_first_kernel<true><<<grid, kFThreads, FirstSmem::total + 1024, stream>>>(maps, p, frames);
  else
    conv_first_kernel<false><<<grid, kFThreads, FirstSmem::total + 1024, stream>>>(maps, p, frames);
  check_cuda(cudaGetLastError(), "conv_first launch");
}

}  // namespace avec
