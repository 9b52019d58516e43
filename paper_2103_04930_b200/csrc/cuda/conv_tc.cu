// tcgen05 implicit-GEMM convolution — see conv_tc.cuh for the design.
#include <cuda_bf16.h>

#include "conv_tc.cuh"
#include "engine.hpp"
#include "ptx.cuh"

namespace avec {

namespace {

using namespace ptx;

constexpr int kTileM = 128;            // output channels per tile (MMA M)
constexpr int kSubN = 256;             // pixels per MMA (MMA N)
constexpr int kSubs = 2;               // MMAs per tile sharing one weight k-block
constexpr int kTileN = kSubN * kSubs;  // pixels per tile
constexpr int kWinRows = kTileN + 8;   // window rows (covers k-1 <= 7 extra rows)
constexpr int kWinBytes = kWinRows * 128;
constexpr int kWinStages = 2;
constexpr int kWgtBytes = kTileM * 128;  // 128 rows x 64 bf16
constexpr int kWgtStages = 5;
constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 512;

struct SmemLayout {
  static constexpr int win = 0;
  static constexpr int wgt = win + kWinStages * kWinBytes;
  static constexpr int bars = wgt + kWgtStages * kWgtBytes;
  static constexpr int total = bars + 256;
};
static_assert(SmemLayout::wgt % 1024 == 0, "SW128 operands need 1024 B alignment");

struct TileCoord {
  int g, n, pt, mt;
};

__device__ __forceinline__ TileCoord decode_tile(const ConvParams& p, int t) {
  TileCoord c;
  const int per_group = p.n_images * p.tiles_per_image * p.m_tiles;
  c.g = t / per_group;
  int rem = t - c.g * per_group;
  c.mt = rem % p.m_tiles;
  rem /= p.m_tiles;
  c.pt = rem % p.tiles_per_image;
  c.n = rem / p.tiles_per_image;
  return c;
}

__global__ void __launch_bounds__(kThreads, 1)
    conv_tc_kernel(const __grid_constant__ ConvMaps maps, const __grid_constant__ ConvParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* win = smem + SmemLayout::win;
  uint8_t* wgt = smem + SmemLayout::wgt;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SmemLayout::bars);
  uint64_t* win_full = bars;
  uint64_t* win_empty = bars + kWinStages;
  uint64_t* w_full = bars + 2 * kWinStages;
  uint64_t* w_empty = w_full + kWgtStages;
  uint64_t* acc_full = w_empty + kWgtStages;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

  const uint32_t warp = warp_id();
  if (warp == 0 && elect_one()) {
    for (int g = 0; g < p.n_groups; ++g) {
      tma_prefetch(&maps.act_big[g]);
      tma_prefetch(&maps.act_small[g]);
      tma_prefetch(&maps.wgt[g]);
    }
    for (int i = 0; i < kWinStages; ++i) {
      mbar_init(&win_full[i], 1);
      mbar_init(&win_empty[i], 1);
    }
    for (int i = 0; i < kWgtStages; ++i) {
      mbar_init(&w_full[i], 1);
      mbar_init(&w_empty[i], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int k = p.k;
  const int pad = k / 2;
  const int kblocks_per_tile = p.cin_chunks * k * k;
  (void)kblocks_per_tile;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      int ws = 0, wst = 0;
      uint32_t wph = 0, wtph = 0;
      const uint32_t win_tx = (k > 1 ? kWinRows : kTileN) * 128;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        const TileCoord tc = decode_tile(p, t);
        const int row0 = tc.n * p.Hp * p.Wp + (p.P - pad) * (p.Wp + 1) + tc.pt * kTileN;
        for (int c = 0; c < p.cin_chunks; ++c) {
          const int ch = p.in_c_off + c * 64;
          for (int r = 0; r < k; ++r) {
            mbar_wait(&win_empty[ws], wph ^ 1);
            mbar_arrive_expect_tx(&win_full[ws], win_tx);
            uint8_t* wbuf = win + ws * kWinBytes;
            const int wr = row0 + r * p.Wp;
            tma_load_2d(wbuf, &maps.act_big[tc.g], &win_full[ws], ch, wr);
            tma_load_2d(wbuf + 256 * 128, &maps.act_big[tc.g], &win_full[ws], ch, wr + 256);
            if (k > 1)
              tma_load_2d(wbuf + 512 * 128, &maps.act_small[tc.g], &win_full[ws], ch, wr + 512);
            if (++ws == kWinStages) { ws = 0; wph ^= 1; }
            for (int s = 0; s < k; ++s) {
              mbar_wait(&w_empty[wst], wtph ^ 1);
              mbar_arrive_expect_tx(&w_full[wst], kWgtBytes);
              tma_load_2d_hint(wgt + wst * kWgtBytes, &maps.wgt[tc.g], &w_full[wst],
                               ((r * k + s) * p.cin_chunks + c) * 64, tc.mt * kTileM, keep);
              if (++wst == kWgtStages) { wst = 0; wtph ^= 1; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16_f32(kTileM, kSubN);
      int ws = 0, wst = 0;
      uint32_t wph = 0, wtph = 0, aph = 0;
      const uint32_t win_base = smem_u32(win), wgt_base = smem_u32(wgt);
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        mbar_wait(acc_empty, aph ^ 1);
        tc_fence_after();
        bool first = true;
        for (int c = 0; c < p.cin_chunks; ++c) {
          for (int r = 0; r < k; ++r) {
            mbar_wait(&win_full[ws], wph);
            tc_fence_after();
            const uint32_t wb = win_base + ws * kWinBytes;
            for (int s = 0; s < k; ++s) {
              mbar_wait(&w_full[wst], wtph);
              tc_fence_after();
              const uint32_t ab = wgt_base + wst * kWgtBytes;
#pragma unroll
              for (int sub = 0; sub < kSubs; ++sub) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                  const uint64_t ad = desc_sw128(ab + kk * 32);
                  const uint64_t bd = desc_sw128(wb + (sub * kSubN + s) * 128 + kk * 32);
                  mma_bf16_ss(tmem + sub * kSubN, ad, bd, idesc, (first && kk == 0) ? 0u : 1u);
                }
              }
              first = false;
              mma_commit(&w_empty[wst]);
              if (++wst == kWgtStages) { wst = 0; wtph ^= 1; }
            }
            mma_commit(&win_empty[ws]);
            if (++ws == kWinStages) { ws = 0; wph ^= 1; }
          }
        }
        mma_commit(acc_full);
        aph ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const uint32_t quad = warp & 3;  // TMEM lane quadrant this warp may touch
    const int co_local = quad * 32 + lane_id();
    uint32_t aph = 0;
    for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
      const TileCoord tc = decode_tile(p, t);
      const ConvGroupParams& g = p.g[tc.g];
      const int co = tc.mt * kTileM + co_local;
      const bool live = co < g.cout;
      const float bias = live ? g.bias[co] : 0.f;
      mbar_wait(acc_full, aph);
      tc_fence_after();
      for (int sub = 0; sub < kSubs; ++sub) {
        const int o0 = tc.pt * kTileN + sub * kSubN;
        int h = o0 / p.Wp;
        int w = o0 - h * p.Wp;
        for (int col = 0; col < kSubN; col += 16) {
          uint32_t v[16];
          tmem_ld16(tmem + ((quad * 32) << 16) + sub * kSubN + col, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (live && h < p.H && w < p.W) {
              float x = __uint_as_float(v[j]) + bias;
              if (g.relu) x = fmaxf(x, 0.f);
              if (p.out_nchw_f32) {
                float* dst = static_cast<float*>(g.out) +
                             ((static_cast<size_t>(tc.n) * g.out_c_stride + g.out_c_off + co) * p.H + h) *
                                 p.W + w;
                *dst = x;
              } else {
                __nv_bfloat16* dst =
                    static_cast<__nv_bfloat16*>(g.out) +
                    (static_cast<size_t>(tc.n * p.out_Hp + h + p.out_P) * p.out_Wp + w + p.out_P) *
                        g.out_c_stride +
                    g.out_c_off + co;
                *dst = __float2bfloat16_rn(x);
              }
            }
            if (++w == p.Wp) { w = 0; ++h; }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(acc_empty);
      aph ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

}  // namespace

size_t conv_smem_bytes() { return SmemLayout::total + 1024; }

void conv_configure() {
  check_cuda(cudaFuncSetAttribute(conv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(conv_smem_bytes())),
             "conv smem attribute");
}

void launch_conv_tc(const ConvMaps& maps, const ConvParams& p, int sm_count, cudaStream_t stream) {
  const int grid = p.total_tiles < sm_count ? p.total_tiles : sm_count;
  conv_tc_kernel<<<grid, kThreads, conv_smem_bytes(), stream>>>(maps, p);
  check_cuda(cudaGetLastError(), "conv_tc launch");
}

}  // namespace avec
