// Pixel-major tcgen05 implicit-GEMM convolution (sm_100a): every conv of the
// pose nets except conv1_1 (conv_first.cu), the COCO 7x7 stage convs
// (conv_tc.cu) and the fused Mconv6+Mconv7 heads (conv_head.cu).
//
// Same padded-flat activation layout, window-reuse trick and warp roles as the
// swap-AB kernel (conv_tc.cu), with the GEMM oriented the other way:
//   M = 128 output pixels (activation window = operand A),
//   N = 64/96/128/256 output channels (weights = operand B), K = 64 per k-block.
// The accumulator row of a pixel sits in one TMEM lane, so each epilogue
// thread holds consecutive channels of ITS pixel per tcgen05.ld; it converts
// them (bias, ReLU/PReLU, zero outside the image, bf16) into its warp's
// swizzled [32 px][W ch] staging box and one lane issues a TMA store per box
// (W = 64/32/16/8, so 52/38/26/19-channel heads need no scalar stores).
//
// Tile = 128 * SUBS_M pixels x N channels; TMEM holds 2 accumulator stages
// (2 * SUBS_M * N <= 512 columns) so the epilogue of tile i overlaps the
// mainloop of tile i+1. Positions outside the image (padded-width columns,
// rows past H) are written as zeros, keeping the output's border valid
// padding; rows past the image's padded extent are clipped by the store map.
//
// Variants (template parameters):
//  * NCTA = 2: a CTA pair on one TPC (cta_group::2). The leader issues
//    M = 256 MMAs; each CTA loads its own window and half of every weight
//    k-block (N/2 rows), so the B operand is read once per SM.
//  * POOL: conv + 2x2/2 max-pool. A CTA's two sub-tiles are output rows y0 and
//    y0+1 at columns x0..x0+127 (four 136-row windows per chunk); the epilogue
//    takes the max of the four raw sums, then bias / ReLU / bf16, and stores
//    the pooled row through a 4D [N][Hp][Wp][C] map.
#include <cuda_bf16.h>

#include <type_traits>

#include "conv_tc.cuh"
#include "engine.hpp"
#include "ptx.cuh"
#include "trace.cuh"

namespace avec {

namespace {

using namespace ptx;

constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 512;

template <int N, int SUBS_M, int NCTA, bool POOL>
struct PmCfg {
  static_assert(!POOL || SUBS_M == 2, "pooled tiles are two rows");
  static constexpr int kTileN = 128 * SUBS_M;  // pixels per tile
  // pooled tiles read four 136-row windows (input rows y-1 .. y+2) per chunk
  static constexpr int kWinRows = POOL ? 136 : kTileN + 8;
  static constexpr int kWinBytes = kWinRows * 128;
  // N = 64 serves the short-K high-resolution conv1_2 (and the thin heads):
  // one more window in flight keeps its HBM reads streaming
#ifndef AVEC_PM_WIN_EXTRA
#define AVEC_PM_WIN_EXTRA 0
#endif
#ifndef AVEC_PM_ROWW128
#define AVEC_PM_ROWW128 0
#endif
  // AVEC_PM_ROWW128: N = 128 tiles trade their third window stage for row-wide
  // weight stages (5 instead of 3). N = 96 (BODY_25's dense blocks) keeps a
  // fourth window in flight (3 row-wide weight stages instead of 5): its
  // short-K chunks consume a window in ~600 cycles, less than a window load's
  // latency; C5 dense-block convs 95-107 -> 88-98 us (profiles/r02_layers_c5.txt)
  static constexpr int kWinStages = POOL ? 6 : N == 64 ? 4 : N == 256 ? 2 : N == 96 ? 4
                                  : (N == 128 && AVEC_PM_ROWW128) ? 2 : 3 + AVEC_PM_WIN_EXTRA;
  static constexpr int kWgtBytes = (N / NCTA) * 128;  // this CTA's N/NCTA rows x 64 bf16
  static constexpr int kAccCols = SUBS_M * N;
  static constexpr int kAccStages = 2;
  static_assert(kAccStages * kAccCols <= 512, "TMEM budget");
  // epilogue staging: per epilogue warp two [32 px][64 ch] bf16 boxes (SW128)
  static constexpr int kStgBox = 32 * 128;
  static constexpr int kStgBytes = 4 * 2 * kStgBox;
  static constexpr int win = 0;
  static constexpr int stg = win + kWinStages * kWinBytes;
  static constexpr int wgt = stg + kStgBytes;
  // N = 96: one weight stage holds the 3 taps of a filter row (one barrier
  // wait and one commit per row instead of per tap; BODY_25's 96-channel
  // dense-block convs -7..-13%, 5 row stages in flight). N = 128/256 have
  // only 3 row stages and measured no better (within C5's clock noise), so
  // they keep per-tap stages, as do pooled tiles. -DAVEC_PM_ROWW=0 turns it off.
#ifndef AVEC_PM_ROWW
#define AVEC_PM_ROWW 1
#endif
  static constexpr int kWgtFree = 232448 - 1024 - 4352 - wgt;
  static constexpr int kTaps =
      (AVEC_PM_ROWW && !POOL && (N == 96 || (N == 128 && AVEC_PM_ROWW128)) && kWgtFree / (3 * kWgtBytes) >= 3) ? 3 : 1;
  static constexpr int kWgtStageBytes = kTaps * kWgtBytes;
  static constexpr int kWgtStages = kWgtFree / kWgtStageBytes > 16 ? 16 : kWgtFree / kWgtStageBytes;
  static constexpr int bias = wgt + kWgtStages * kWgtStageBytes;  // N bias + N slope floats per acc stage
  static constexpr int bars = bias + 2 * kAccStages * N * 4;
  static constexpr int total = bars + 256;
  static_assert(kWinBytes % 1024 == 0 && wgt % 1024 == 0 && stg % 1024 == 0, "SW128 alignment");
  static_assert(total + 1024 <= 232448, "smem budget");
};

struct PmTile {
  int g, n, pt, nt;
};

__device__ __forceinline__ PmTile pm_decode(const ConvParams& p, int t) {
  PmTile c;
  const int per_group = p.n_images * p.tiles_per_image * p.m_tiles;
  c.g = t / per_group;
  int rem = t - c.g * per_group;
  c.nt = rem % p.m_tiles;
  rem /= p.m_tiles;
  c.pt = rem % p.tiles_per_image;
  c.n = rem / p.tiles_per_image;
  return c;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Row-pair tile of the fused-pool mode: this CTA's rows y0, y0+1 at columns
// x0 .. x0+127 (sub-tile s = row y0 + s)
__device__ __forceinline__ void pool_tile(const ConvParams& p, int pt, int ncta, uint32_t rank, int& y0, int& x0) {
  const int rp = pt / p.col_blocks;
  y0 = (rp * ncta + int(rank)) * 2;
  x0 = (pt - rp * p.col_blocks) * 128;
}

template <int N, int SUBS_M, int NCTA, bool POOL>
__global__ void __launch_bounds__(kThreads, 1)
    conv_pm_kernel(const __grid_constant__ ConvMaps maps, const __grid_constant__ ConvParams p) {
  using C = PmCfg<N, SUBS_M, NCTA, POOL>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* win = smem + C::win;
  uint8_t* wgt = smem + C::wgt;
  uint8_t* stg = smem + C::stg;
  float* sbias = reinterpret_cast<float*>(smem + C::bias);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::bars);
  uint64_t* win_full = bars;
  uint64_t* win_empty = win_full + C::kWinStages;
  uint64_t* w_full = win_empty + C::kWinStages;
  uint64_t* w_empty = w_full + C::kWgtStages;
  uint64_t* acc_full = w_empty + C::kWgtStages;
  uint64_t* acc_empty = acc_full + C::kAccStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + C::kAccStages);

  const uint32_t warp = warp_id();
  if (threadIdx.x == 0) AVEC_STAMP(0);
  // CTA pair (NCTA == 2): rank 0 (leader) issues the M = 256 MMAs and owns the
  // full / acc_empty barriers; both CTAs load their own window and half of
  // every weight k-block, and run the epilogue of their own 128-row halves
  const uint32_t rank = NCTA == 2 ? cluster_cta_rank() : 0;
  const bool leader = rank == 0;
  if (warp == 0 && elect_one()) {
    for (int g = 0; g < p.n_groups; ++g) {
      tma_prefetch(C::kTileN == 256 ? &maps.act_big[g] : &maps.act_mid[g]);
      tma_prefetch(&maps.act_small[g]);
      tma_prefetch(&maps.wgt[g]);
    }
    for (int i = 0; i < C::kWinStages; ++i) {
      mbar_init(&win_full[i], 1);
      mbar_init(&win_empty[i], 1);
    }
    for (int i = 0; i < C::kWgtStages; ++i) {
      mbar_init(&w_full[i], 1);
      mbar_init(&w_empty[i], 1);
    }
    for (int i = 0; i < C::kAccStages; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], NCTA == 2 ? 8 : 128);  // pair: one arrival per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (NCTA == 2) tmem_alloc_pair<kTmemCols>(tmem_slot);
    else tmem_alloc<kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (NCTA == 2) cluster_sync_all();  // peer barriers initialised before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // see conv_tc.cu
  if (threadIdx.x == 0) AVEC_STAMP(1);

  const int k = p.k;
  const int pad = k / 2;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      int ws = 0, wst = 0;
      uint32_t wph = 0, wtph = 0;
      const uint32_t win_tx = ((POOL ? 128 : C::kTileN) + (k > 1 ? 8 : 0)) * 128;
      auto load_window = [&](const PmTile& tc, int ch, int wr) {
        mbar_wait(&win_empty[ws], wph ^ 1);
        if (leader) mbar_arrive_expect_tx(&win_full[ws], NCTA * win_tx);  // both CTAs' bytes
        uint8_t* wbuf = win + ws * C::kWinBytes;
        constexpr int kBox = POOL ? 128 : C::kTileN;  // + 8-row halo box
        const CUtensorMap* wmap = kBox == 256 ? &maps.act_big[tc.g] : &maps.act_mid[tc.g];
        if constexpr (NCTA == 2) {
          const uint32_t fb = mapa_shared(&win_full[ws], 0);
          tma_load_2d_pair(wbuf, wmap, fb, ch, wr);
          if (k > 1) tma_load_2d_pair(wbuf + kBox * 128, &maps.act_small[tc.g], fb, ch, wr + kBox);
        } else {
          tma_load_2d(wbuf, wmap, &win_full[ws], ch, wr);
          if (k > 1) tma_load_2d(wbuf + kBox * 128, &maps.act_small[tc.g], &win_full[ws], ch, wr + kBox);
        }
        if (++ws == C::kWinStages) { ws = 0; wph ^= 1; }
      };
      auto load_weights = [&](const PmTile& tc, int c, int r) {
        // kTaps == 3: the row's k taps share one stage (tap s at slot s)
        const int per_stage = C::kTaps == 1 ? 1 : k;
        for (int s = 0; s < k; ++s) {
          const int sl = C::kTaps == 1 ? 0 : s;
          if (sl == 0) {
            mbar_wait(&w_empty[wst], wtph ^ 1);
            if (leader) mbar_arrive_expect_tx(&w_full[wst], NCTA * C::kWgtBytes * per_stage);
          }
          const int kx = ((r * k + s) * p.cin_chunks + c) * 64;
          const int wrow = tc.nt * N + int(rank) * (N / NCTA);  // this CTA's half of B
          uint8_t* dst = wgt + wst * C::kWgtStageBytes + sl * C::kWgtBytes;
          if constexpr (NCTA == 2)
            tma_load_2d_pair_hint(dst, &maps.wgt[tc.g], mapa_shared(&w_full[wst], 0), kx, wrow, keep);
          else
            tma_load_2d_hint(dst, &maps.wgt[tc.g], &w_full[wst], kx, wrow, keep);
          if (sl + 1 == per_stage && ++wst == C::kWgtStages) { wst = 0; wtph ^= 1; }
        }
      };
      for (int t = int(blockIdx.x) / NCTA; t < p.total_tiles; t += int(gridDim.x) / NCTA) {
        const PmTile tc = pm_decode(p, t);
        if constexpr (POOL) {
          // windows W_j = input rows y0-1+j (j = 0..3); filter row r of the
          // two output rows needs W_r (row y0) and W_r+1 (row y0+1), so its
          // weights follow W_r+1
          int y0, x0;
          pool_tile(p, tc.pt, NCTA, rank, y0, x0);
          const int row0 = tc.n * p.Hp * p.Wp + (p.P - pad) * (p.Wp + 1) + y0 * p.Wp + x0;
          for (int c = 0; c < p.cin_chunks; ++c) {
            const int ch = p.in_c_off + c * 64;
            for (int j = 0; j <= k; ++j) {
              load_window(tc, ch, row0 + j * p.Wp);
              if (j > 0) load_weights(tc, c, j - 1);
            }
          }
          continue;
        }
        const int row0 = tc.n * p.Hp * p.Wp + (p.P - pad) * (p.Wp + 1) + (tc.pt * NCTA + int(rank)) * C::kTileN;
        for (int c = 0; c < p.cin_chunks; ++c) {
          const int ch = p.in_c_off + c * 64;
          for (int r = 0; r < k; ++r) {
            // window rows: kTileN (<= 256, one box when SUBS_M == 2) + 8-row halo
            load_window(tc, ch, row0 + r * p.Wp);
            load_weights(tc, c, r);
            if (c == 0 && r == 0) AVEC_STAMP(2);
          }
        }
      }
      AVEC_STAMP(3);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (leader && elect_one()) {
      const uint32_t idesc = idesc_bf16_f32(128 * NCTA, N);
      int ws = 0, wst = 0, acc = 0;
      uint32_t wph = 0, wtph = 0, aph = 0;
      const uint32_t win_base = smem_u32(win), wgt_base = smem_u32(wgt);
      auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t accum) {
        if constexpr (NCTA == 2) mma_bf16_ss_pair(d, a, b, idesc, accum);
        else mma_bf16_ss(d, a, b, idesc, accum);
      };
      auto commit = [&](uint64_t* bar) {
        if constexpr (NCTA == 2) mma_commit_pair(bar);
        else mma_commit(bar);
      };
      for (int t = int(blockIdx.x) / NCTA; t < p.total_tiles; t += int(gridDim.x) / NCTA) {
        mbar_wait(&acc_empty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem + acc * C::kAccCols;
        bool first = true;
        if constexpr (POOL) {
          // sub-tile 0 (row y0) reads W_r, sub-tile 1 (row y0+1) reads W_r+1
          for (int c = 0; c < p.cin_chunks; ++c) {
            const int kn = c + 1 == p.cin_chunks ? p.k16_last : 4;
            mbar_wait(&win_full[ws], wph);
            tc_fence_after();
            for (int r = 0; r < k; ++r) {
              const int ns = ws + 1 == C::kWinStages ? 0 : ws + 1;
              const uint32_t nph = ws + 1 == C::kWinStages ? wph ^ 1 : wph;
              mbar_wait(&win_full[ns], nph);
              tc_fence_after();
              const uint32_t wb0 = win_base + ws * C::kWinBytes, wb1 = win_base + ns * C::kWinBytes;
              for (int s = 0; s < k; ++s) {
                mbar_wait(&w_full[wst], wtph);
                tc_fence_after();
                const uint64_t bd = desc_sw128(wgt_base + wst * C::kWgtStageBytes);
                const uint64_t a0 = desc_sw128(wb0 + s * 128), a1 = desc_sw128(wb1 + s * 128);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {  // a 32-byte K step adds 2 to a descriptor
                  if (kk >= kn) break;
                  const uint32_t accum = (first && kk == 0) ? 0u : 1u;
                  mma(d0, a0 + 2 * kk, bd + 2 * kk, accum);
                  mma(d0 + N, a1 + 2 * kk, bd + 2 * kk, accum);
                }
                first = false;
                commit(&w_empty[wst]);
                if (++wst == C::kWgtStages) { wst = 0; wtph ^= 1; }
              }
              commit(&win_empty[ws]);  // W_r is done
              ws = ns;
              wph = nph;
            }
            commit(&win_empty[ws]);  // W_k
            if (++ws == C::kWinStages) { ws = 0; wph ^= 1; }
          }
        } else {
        for (int c = 0; c < p.cin_chunks; ++c) {
          // the last chunk's zero-weight channel tail (96-channel dense blocks,
          // mapped stage inputs) is skipped in 16-channel K steps
          const int kn = c + 1 == p.cin_chunks ? p.k16_last : 4;
          for (int r = 0; r < k; ++r) {
            mbar_wait(&win_full[ws], wph);
            tc_fence_after();
            if (first) AVEC_STAMP(4);
            const uint32_t wb = win_base + ws * C::kWinBytes;
            if constexpr (C::kTaps == 3) {
              mbar_wait(&w_full[wst], wtph);
              tc_fence_after();
            }
            for (int s = 0; s < k; ++s) {
              if constexpr (C::kTaps == 1) {
                mbar_wait(&w_full[wst], wtph);
                tc_fence_after();
              }
              const uint32_t bb = wgt_base + wst * C::kWgtStageBytes + (C::kTaps == 1 ? 0 : s * C::kWgtBytes);
              // descriptors built once per tap: a 32-byte K step adds 2 to the
              // start-address field (addresses < 256 KB, so it cannot carry out)
              const uint64_t bd0 = desc_sw128(bb);
              // the K16 count as a compile-time constant: a fully unrolled
              // tap is straight-line MMAs with immediate descriptor offsets
              // (a runtime-bounded loop put a branch and a 64-bit add chain
              // on the single issuing thread between MMAs)
              auto tap = [&](auto kn_c) {
                constexpr int KN = decltype(kn_c)::value;
#pragma unroll
                for (int sub = 0; sub < SUBS_M; ++sub) {
                  const uint64_t ad0 = desc_sw128(wb + (sub * 128 + s) * 128);
#pragma unroll
                  for (int kk = 0; kk < KN; ++kk)
                    mma(d0 + sub * N, ad0 + 2 * kk, bd0 + 2 * kk, (first && kk == 0) ? 0u : 1u);
                }
              };
              switch (kn) {
                case 4: tap(std::integral_constant<int, 4>{}); break;
                case 3: tap(std::integral_constant<int, 3>{}); break;
                case 2: tap(std::integral_constant<int, 2>{}); break;
                default: tap(std::integral_constant<int, 1>{}); break;
              }
              first = false;
              if constexpr (C::kTaps == 1) {
                commit(&w_empty[wst]);
                if (++wst == C::kWgtStages) { wst = 0; wtph ^= 1; }
              }
            }
            if constexpr (C::kTaps == 3) {
              commit(&w_empty[wst]);
              if (++wst == C::kWgtStages) { wst = 0; wtph ^= 1; }
            }
            commit(&win_empty[ws]);
            if (++ws == C::kWinStages) { ws = 0; wph ^= 1; }
          }
        }
        }  // !POOL
        commit(&acc_full[acc]);
        if (++acc == C::kAccStages) { acc = 0; aph ^= 1; }
      }
      AVEC_STAMP(5);
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  } else {
    // ------------------------------------------------------------ epilogue
    // Warp q owns TMEM lanes 32q..32q+31 = pixels 32q.. of each 128-pixel
    // sub-tile. Channel slabs go TMEM -> registers (bias, activation, zero
    // outside the image, bf16) -> this warp's swizzled [32 px][64 ch] staging
    // box -> one TMA store per box, so global writes are whole 128-byte lines
    // (per-thread 16-byte stores at a 128-byte pixel stride cost 8x the L1
    // wavefronts and left the high-resolution layers store-bound).
    const uint32_t quad = warp & 3;
    const uint32_t lane = lane_id();
    const int ep = int(threadIdx.x) - 64;  // 0..127
    uint8_t* stg_w = stg + quad * (2 * C::kStgBox);
    int acc = 0, stg_i = 0;
    uint32_t aph = 0;
    const int img_rows = p.Hp * p.Wp;
    for (int t = int(blockIdx.x) / NCTA; t < p.total_tiles; t += int(gridDim.x) / NCTA) {
      const PmTile tc = pm_decode(p, t);
      const ConvGroupParams& g = p.g[tc.g];
      float* bs = sbias + acc * N;
      float* sl = sbias + (C::kAccStages + acc) * N;
      // this tile's bias / PReLU-slope slices (the acc stage's previous tile
      // finished reading them); ReLU is PReLU with slope 0, identity slope 1
      for (int i = ep; i < N; i += 128) {
        const int co = tc.nt * N + i;
        bs[i] = co < g.cout ? g.bias[co] : 0.f;
        sl[i] = g.act == 1 ? 0.f : (g.act == 2 && co < g.cout) ? g.slope[co] : 1.f;
      }
      named_bar_sync(1, 128);
      mbar_wait(&acc_full[acc], aph);
      tc_fence_after();
      if (ep == 0) AVEC_STAMP(6);
      __nv_bfloat16* out = static_cast<__nv_bfloat16*>(g.out);
      const int c_left = g.cout - tc.nt * N;  // live channels of this tile
      if constexpr (POOL) {
        // fused 2x2/2 max-pool: TMEM lane = column x0+32q+lane, sub-tile 0/1 =
        // rows y0/y0+1 at columns [0,N)/[N,2N). max over the four raw sums,
        // then bias and activation: x -> bf16(act(x + b)) is monotonic for
        // ReLU, so this equals pooling the bf16 conv outputs bit for bit.
        int y0, x0;
        pool_tile(p, tc.pt, NCTA, rank, y0, x0);
        const bool pvalid = x0 + int(quad) * 32 + int(lane) < p.W;  // W even: pairs share validity
        const uint32_t tb0 = tmem + ((quad * 32) << 16) + acc * C::kAccCols;
        const bool relu = g.act == 1;
        for (int c0 = 0; c0 < N; c0 += 64) {  // cout == N (host check)
          uint8_t* buf = stg_w + (stg_i & 1) * C::kStgBox;
          if (lane == 0) bulk_wait_read<1>();  // the store that last read `buf` is done
          __syncwarp();
#pragma unroll
          for (int hlf = 0; hlf < 2; ++hlf) {
            uint32_t va[32], vb[32];
            tmem_ld32(tb0 + c0 + 32 * hlf, va);
            tmem_ld32(tb0 + N + c0 + 32 * hlf, vb);
            tmem_ld_wait();
            uint32_t w[16];
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              float m0 = fmaxf(__uint_as_float(va[j]), __uint_as_float(vb[j]));
              float m1 = fmaxf(__uint_as_float(va[j + 1]), __uint_as_float(vb[j + 1]));
              m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
              m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
              const int c = c0 + 32 * hlf + j;
              float a = m0 + bs[c], b = m1 + bs[c + 1];
              if (relu) {
                a = fmaxf(a, 0.f);
                b = fmaxf(b, 0.f);
              } else {
                a = fmaxf(a, 0.f) + sl[c] * fminf(a, 0.f);
                b = fmaxf(b, 0.f) + sl[c + 1] * fminf(b, 0.f);
              }
              w[j / 2] = pvalid ? pack_bf16(a, b) : 0u;
            }
            if ((lane & 1) == 0) {  // even lanes hold pooled column (x0 + 32q + lane) / 2
              const uint32_t row = lane >> 1;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t qq = 4 * hlf + q;
                *reinterpret_cast<uint4*>(buf + row * 128 + ((qq ^ (row & 7)) << 4)) =
                    make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
              }
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_4d(&maps.out_pool[tc.g], buf, g.out_c_off + tc.nt * N + c0,
                         x0 / 2 + int(quad) * 16 + p.pool_P, y0 / 2 + p.pool_P, tc.n);
            bulk_commit();
          }
          ++stg_i;
        }
      } else {
        for (int sub = 0; sub < SUBS_M; ++sub) {
          const int o = (tc.pt * NCTA + int(rank)) * C::kTileN + sub * 128 + int(quad) * 32 + int(lane);
          const int hh = o / p.Wp;
          const int ww = o - hh * p.Wp;
          const bool valid = hh < p.H && ww < p.W;
          const int row_in_img = p.P * p.Wp + p.P + o;  // output row of this pixel
          const uint32_t tbase = tmem + ((quad * 32) << 16) + acc * C::kAccCols + sub * N;
          if (p.out_mode == kOutTmaBf16) {
            const int row_w = row_in_img - int(lane);  // the warp's first pixel
            // one [32 px][W ch] box: TMEM -> bias/activation/bf16 -> swizzled
            // staging (swizzle span = box row: 16-byte chunk q of row r lands at
            // q ^ (r & 7) for 128 B rows, q ^ ((r >> 1) & 3) for 64 B,
            // q ^ ((r >> 2) & 1) for 32 B; 16 B rows are unswizzled) -> TMA store
            auto box = [&](auto width, auto relu_only, int c0) {
              constexpr int W = decltype(width)::value;
              constexpr bool kRelu = decltype(relu_only)::value;
              uint32_t va[W < 16 ? 16 : W > 32 ? 32 : W], vb[W == 64 ? 32 : 1];
              if constexpr (W >= 32) {
                tmem_ld32(tbase + c0, va);
                if constexpr (W == 64) tmem_ld32(tbase + c0 + 32, vb);
              } else {
                tmem_ld16(tbase + c0, va);  // c0 + 16 <= N: N is a multiple of 16
              }
              tmem_ld_wait();
              uint8_t* buf = stg_w + (stg_i & 1) * C::kStgBox;
              if (lane == 0) bulk_wait_read<1>();  // the store that last read `buf` is done
              __syncwarp();
  #pragma unroll
              for (int q = 0; q < W / 8; ++q) {
                uint32_t w[4];
  #pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const int c = q * 8 + 2 * j;  // channel within the box
                  uint32_t x0, x1;
                  if constexpr (W == 64) {
                    x0 = q < 4 ? va[c & 31] : vb[c & 31];
                    x1 = q < 4 ? va[(c + 1) & 31] : vb[(c + 1) & 31];
                  } else {
                    x0 = va[c];
                    x1 = va[c + 1];
                  }
                  float a = __uint_as_float(x0) + bs[c0 + c];
                  float b = __uint_as_float(x1) + bs[c0 + c + 1];
                  if constexpr (kRelu) {
                    a = fmaxf(a, 0.f);
                    b = fmaxf(b, 0.f);
                  } else {  // identity (slope 1) or PReLU
                    a = fmaxf(a, 0.f) + sl[c0 + c] * fminf(a, 0.f);
                    b = fmaxf(b, 0.f) + sl[c0 + c + 1] * fminf(b, 0.f);
                  }
                  w[j] = valid ? pack_bf16(a, b) : 0u;
                }
                uint32_t off;
                if constexpr (W == 64) off = lane * 128 + ((q ^ (lane & 7)) << 4);
                else if constexpr (W == 32) off = lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4);
                else if constexpr (W == 16) off = lane * 32 + ((q ^ ((lane >> 2) & 1)) << 4);
                else off = lane * 16;
                *reinterpret_cast<uint4*>(buf + off) = make_uint4(w[0], w[1], w[2], w[3]);
              }
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                const CUtensorMap* m = W == 64 ? &maps.out[tc.g]
                                       : W == 32 ? &maps.out32[tc.g]
                                       : W == 16 ? &maps.out16[tc.g]
                                                 : &maps.out8[tc.g];
                tma_store_3d(m, buf, g.out_c_off + tc.nt * N + c0, row_w, tc.n);
                bulk_commit();
              }
              ++stg_i;
            };
            using I64 = std::integral_constant<int, 64>;
            using I32 = std::integral_constant<int, 32>;
            using I16 = std::integral_constant<int, 16>;
            using I8 = std::integral_constant<int, 8>;
            auto boxes = [&](auto relu_only) {
              if (c_left >= N) {  // full tile: compile-time box sequence
  #pragma unroll
                for (int c0 = 0; c0 + 64 <= N; c0 += 64) box(I64{}, relu_only, c0);
                if constexpr (N % 64 == 32) box(I32{}, relu_only, N - 32);
              } else {
                // round_up(live channels, 8) in boxes of 64/32/16/8 channels; the
                // channels past cout (zero weights, zero bias) store zeros
                const int c_end = (c_left + 7) & ~7;
                int c0 = 0;
                for (; c0 + 64 <= c_end; c0 += 64) box(I64{}, relu_only, c0);
                if (c0 + 32 <= c_end) { box(I32{}, relu_only, c0); c0 += 32; }
                if (c0 + 16 <= c_end) { box(I16{}, relu_only, c0); c0 += 16; }
                if (c0 + 8 <= c_end) box(I8{}, relu_only, c0);
              }
            };
            if (g.act == 1) boxes(std::true_type{});
            else boxes(std::false_type{});
            continue;
          }
          // thin heads (38/19 channels into the stage concat) and the fp32 NCHW
          // network output: per-channel stores of valid pixels only; lanes are
          // consecutive pixels, so NCHW stores coalesce along W
  #pragma unroll
          for (int c0 = 0; c0 < N; c0 += 32) {
            if (c0 >= c_left) break;
            uint32_t v[32];
            tmem_ld32(tbase + c0, v);
            tmem_ld_wait();
  #pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (valid && c0 + j < c_left) {
                float a = __uint_as_float(v[j]) + bs[c0 + j];
                a = fmaxf(a, 0.f) + sl[c0 + j] * fminf(a, 0.f);
                const int co = tc.nt * N + c0 + j;
                if (p.out_mode == kOutNchwF32)
                  static_cast<float*>(g.out)[((static_cast<size_t>(tc.n) * g.out_c_stride + g.out_c_off + co) *
                                                  p.H + hh) * p.W + ww] = a;
                else
                  out[(static_cast<size_t>(tc.n) * img_rows + row_in_img) * g.out_c_stride + g.out_c_off + co] =
                      __float2bfloat16_rn(a);
              }
            }
          }
        }
      }
      tc_fence_before();
      if constexpr (NCTA == 2) {
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(&acc_empty[acc], 0));  // the leader's barrier
      } else {
        mbar_arrive(&acc_empty[acc]);
      }
      if (++acc == C::kAccStages) { acc = 0; aph ^= 1; }
    }
    if (ep == 0) AVEC_STAMP(7);
    if (lane == 0) bulk_wait<0>();
    if (ep == 0) AVEC_STAMP(8);
  }
  tc_fence_before();
  if constexpr (NCTA == 2) cluster_sync_all();  // the leader's MMAs read peer smem until the end
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (NCTA == 2) tmem_dealloc_pair<kTmemCols>(tmem);
    else tmem_dealloc<kTmemCols>(tmem);
  }
  if (threadIdx.x == 0) AVEC_STAMP(9);
}

template <int N, int SUBS_M, int NCTA, bool POOL = false>
void launch_pm(const ConvMaps& maps, const ConvParams& p, int sm_count, cudaStream_t stream) {
  // row-wide weight stages hold one filter row's taps (tap s in slot s): a
  // wider filter would write past its stage into the next one
  if (PmCfg<N, SUBS_M, NCTA, POOL>::kTaps > 1 && p.k > PmCfg<N, SUBS_M, NCTA, POOL>::kTaps)
    fail(AVEC_ERR_UNSUPPORTED, "pixel-major conv: filter wider than the row-wide weight stage");
  const int pairs = sm_count / NCTA;
  const int grid = NCTA * (p.total_tiles < pairs ? p.total_tiles : pairs);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = PmCfg<N, SUBS_M, NCTA, POOL>::total + 1024;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (NCTA == 2) {  // the pair must share a TPC
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  check_cuda(cudaLaunchKernelEx(&cfg, conv_pm_kernel<N, SUBS_M, NCTA, POOL>, maps, p), "conv_pm launch");
}

template <int N, int SUBS_M, int NCTA, bool POOL = false>
void configure_pm() {
  check_cuda(cudaFuncSetAttribute(conv_pm_kernel<N, SUBS_M, NCTA, POOL>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(PmCfg<N, SUBS_M, NCTA, POOL>::total + 1024)),
             "conv_pm smem attribute");
}

}  // namespace

#ifdef AVEC_TRACE
void conv_pm_trace(int on, cudaStream_t st) {
  check_cuda(cudaMemcpyToSymbolAsync(g_trace_on, &on, sizeof on, 0, cudaMemcpyHostToDevice, st), "trace arm");
  check_cuda(cudaStreamSynchronize(st), "trace arm");
}
int conv_pm_trace_dump(unsigned long long* host, int n) {
  return cudaMemcpyFromSymbol(host, g_trace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 5;
}
#endif

int conv_pm_subs(int n_tile) { return n_tile == 256 ? 1 : 2; }  // 2 acc stages fit TMEM

void conv_pm_configure() {
  configure_pm<64, 2, 1>();
  configure_pm<96, 2, 1>();
  configure_pm<128, 2, 1>();
  configure_pm<256, 1, 1>();
  configure_pm<64, 2, 2>();
  configure_pm<96, 2, 2>();
  configure_pm<128, 2, 2>();
  configure_pm<256, 1, 2>();
  configure_pm<64, 2, 1, true>();
  configure_pm<128, 2, 1, true>();
  configure_pm<64, 2, 2, true>();
  configure_pm<128, 2, 2, true>();
}

int conv_pm_tile_n(int cout) { return cout <= 64 ? 64 : cout <= 96 ? 96 : cout <= 128 ? 128 : 256; }

void launch_conv_pm(const ConvMaps& maps, const ConvParams& p, int sm_count, cudaStream_t stream) {
  const bool pair = p.ncta == 2;
  if (p.pool) {
    if (p.pm_n == 64)
      pair ? launch_pm<64, 2, 2, true>(maps, p, sm_count, stream) : launch_pm<64, 2, 1, true>(maps, p, sm_count, stream);
    else if (p.pm_n == 128)
      pair ? launch_pm<128, 2, 2, true>(maps, p, sm_count, stream)
           : launch_pm<128, 2, 1, true>(maps, p, sm_count, stream);
    else
      fail(AVEC_ERR_UNSUPPORTED, "fused pooling supports 64/128-channel tiles");
    return;
  }
  switch (p.pm_n) {
    case 64: pair ? launch_pm<64, 2, 2>(maps, p, sm_count, stream) : launch_pm<64, 2, 1>(maps, p, sm_count, stream); break;
    case 96: pair ? launch_pm<96, 2, 2>(maps, p, sm_count, stream) : launch_pm<96, 2, 1>(maps, p, sm_count, stream); break;
    case 128:
      pair ? launch_pm<128, 2, 2>(maps, p, sm_count, stream) : launch_pm<128, 2, 1>(maps, p, sm_count, stream);
      break;
    case 256:
      pair ? launch_pm<256, 1, 2>(maps, p, sm_count, stream) : launch_pm<256, 1, 1>(maps, p, sm_count, stream);
      break;
    default: fail(AVEC_ERR_UNSUPPORTED, "pixel-major conv supports N tiles of 64/96/128/256");
  }
}

}  // namespace avec
