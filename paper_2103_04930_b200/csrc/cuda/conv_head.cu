// Fused stage head: Mconv6 (1x1, c6 channels, ReLU/PReLU) followed by Mconv7
// (1x1, c7 <= 64 channels, no activation) in one tcgen05 kernel (sm_100a).
//
// The c6-channel intermediate never reaches HBM: per 128-pixel tile,
//   MMA1  acc1[b] = X[128 px x cin] * W6[block]^T   (128 cols, b = block & 1)
//   epi1  acc1[b] -> bias6, act6 -> bf16 -> Y[b] in smem (SW128 K-major)
//   MMA2  acc2[128 px x 64] += Y[b] * W7[:, block]^T  (TMEM cols 256..319)
// for each 128-wide block of c6, double-buffered so MMA1 of block j+1 runs
// while the epilogue converts block j, then
//   epi2  acc2 -> bias7 -> the stage concat (bf16, 32/16/8-channel TMA boxes)
//         and/or the fp32 NCHW network output.
// On BODY_25 (c6 = 512 at 1312x736 x 32 frames) this removes a 495 MB write
// and read per stage and one launch; on COCO (c6 = 128) mostly the launch.
// Warp roles: warp 0 X/W6 TMA producer, warp 1 TMEM owner + MMA issuer,
// warps 2-9 both epilogues (two per TMEM lane quadrant, splitting the
// columns), warp 10 W7 TMA producer. Persistent over (branch, image, tile).
#include <cuda_bf16.h>

#include <type_traits>

#include "conv_tc.cuh"
#include "engine.hpp"
#include "ptx.cuh"

namespace avec {

namespace {

using namespace ptx;

constexpr int kHThreads = 352;  // X/W6 producer, MMA, 8 epilogue warps (2 per TMEM lane quadrant), W7 producer
constexpr int kHEpi = 256;
constexpr uint32_t kHTmemCols = 512;
constexpr int kAcc2Col = 256;  // acc2 lives at TMEM columns 256..319
constexpr int kNB = 128;        // c6 block width (MMA1 N)
constexpr int kXStages = 3;
constexpr int kW6Stages = 3;
constexpr int kW7Stages = 2;

struct HeadSmem {
  static constexpr int x = 0;                          // kXStages x [128 px][64 ch]
  static constexpr int w6 = x + kXStages * 16384;      // kW6Stages x [128 rows][64]
  static constexpr int y = w6 + kW6Stages * 16384;     // 2 x [128 px][128 ch] as 2 SW128 chunks each
  static constexpr int w7 = y + 2 * 32768;             // kW7Stages x [64 rows][64]
  static constexpr int stg = w7 + kW7Stages * 8192;    // 8 warps x [32 px][<=32 ch]
  static constexpr int bias = stg + 8 * 2048;          // b6/s6 per Y buffer (2 x 2 x 128) + b7 (64)
  static constexpr int bars = bias + (4 * kNB + 64) * 4;
  static constexpr int total = bars + 256;
  static_assert(total + 1024 <= 232448, "smem budget");
};

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void head_decode(const HeadParams& p, int t, int& g, int& n, int& pt) {
  const int per_group = p.n_images * p.tiles_per_image;
  g = t / per_group;
  const int rem = t - g * per_group;
  n = rem / p.tiles_per_image;
  pt = rem - n * p.tiles_per_image;
}

__global__ void __launch_bounds__(kHThreads, 1)
    conv_head_kernel(const __grid_constant__ HeadMaps maps, const __grid_constant__ HeadParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* sx = smem + HeadSmem::x;
  uint8_t* sw6 = smem + HeadSmem::w6;
  uint8_t* sy = smem + HeadSmem::y;
  uint8_t* sw7 = smem + HeadSmem::w7;
  uint8_t* stg = smem + HeadSmem::stg;
  float* sb6 = reinterpret_cast<float*>(smem + HeadSmem::bias);  // [2][128]
  float* ss6 = sb6 + 2 * kNB;                                     // [2][128]
  float* sb7 = ss6 + 2 * kNB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + HeadSmem::bars);
  uint64_t* x_full = bars;
  uint64_t* x_empty = x_full + kXStages;
  uint64_t* w6_full = x_empty + kXStages;
  uint64_t* w6_empty = w6_full + kW6Stages;
  uint64_t* w7_full = w6_empty + kW6Stages;
  uint64_t* w7_empty = w7_full + kW7Stages;
  uint64_t* a1_full = w7_empty + kW7Stages;  // [2]
  uint64_t* y_full = a1_full + 2;             // [2]
  uint64_t* y_empty = y_full + 2;             // [2]
  uint64_t* a2_full = y_empty + 2;
  uint64_t* a2_empty = a2_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a2_empty + 1);

  const uint32_t warp = warp_id();
  constexpr int NB = kNB;
  constexpr int kc_per_block = NB / 64;
  if (warp == 0 && elect_one()) {
    for (int g = 0; g < p.n_groups; ++g) {
      tma_prefetch(&maps.x[g]);
      tma_prefetch(&maps.w6[g]);
      tma_prefetch(&maps.w7[g]);
    }
    for (int i = 0; i < kXStages; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < kW6Stages; ++i) { mbar_init(&w6_full[i], 1); mbar_init(&w6_empty[i], 1); }
    for (int i = 0; i < kW7Stages; ++i) { mbar_init(&w7_full[i], 1); mbar_init(&w7_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a1_full[i], 1);
      mbar_init(&y_full[i], kHEpi);
      mbar_init(&y_empty[i], 1);
    }
    mbar_init(a2_full, 1);
    mbar_init(a2_empty, kHEpi);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kHTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      int xs = 0, w6s = 0;
      uint32_t xph = 0, w6ph = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        int g, n, pt;
        head_decode(p, t, g, n, pt);
        const int row0 = n * p.Hp * p.Wp + p.P * (p.Wp + 1) + pt * 128;
        for (int j = 0; j < p.blocks; ++j) {
          for (int c = 0; c < p.cin_chunks; ++c) {
            mbar_wait(&x_empty[xs], xph ^ 1);
            mbar_arrive_expect_tx(&x_full[xs], 16384);
            tma_load_2d(sx + xs * 16384, &maps.x[g], &x_full[xs], p.in_c_off + c * 64, row0);
            if (++xs == kXStages) { xs = 0; xph ^= 1; }
            mbar_wait(&w6_empty[w6s], w6ph ^ 1);
            mbar_arrive_expect_tx(&w6_full[w6s], NB * 128);
            tma_load_2d_hint(sw6 + w6s * 16384, &maps.w6[g], &w6_full[w6s], c * 64, j * NB, keep);
            if (++w6s == kW6Stages) { w6s = 0; w6ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 10) {
    // ------------------------------------------------------------ W7 producer
    // its own warp: W7 stages free only when MMA2 of the previous block ran,
    // which waits on the epilogue; the X/W6 stream must not stall behind it
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      int w7s = 0;
      uint32_t w7ph = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        int g, n, pt;
        head_decode(p, t, g, n, pt);
        for (int j = 0; j < p.blocks; ++j)
          for (int kc = 0; kc < kc_per_block; ++kc) {
            mbar_wait(&w7_empty[w7s], w7ph ^ 1);
            mbar_arrive_expect_tx(&w7_full[w7s], 8192);
            tma_load_2d_hint(sw7 + w7s * 8192, &maps.w7[g], &w7_full[w7s], j * NB + kc * 64, 0, keep);
            if (++w7s == kW7Stages) { w7s = 0; w7ph ^= 1; }
          }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      const uint32_t idesc1 = idesc_bf16_f32(128, NB);
      const uint32_t idesc2 = idesc_bf16_f32(128, 64);
      int xs = 0, w6s = 0, w7s = 0;
      uint32_t xph = 0, w6ph = 0, w7ph = 0, a2eph = 0;
      uint32_t yfph = 0;  // phase bit per Y buffer (bit b), kept in a register
      int bc = 0;  // running block counter: Y / acc1 buffer = bc & 1
      const uint32_t x_base = smem_u32(sx), w6_base = smem_u32(sw6), y_base = smem_u32(sy),
                     w7_base = smem_u32(sw7);
      // MMA2 of one block: acc2 (+)= Y[b] * W7[:, block]^T
      auto mma2 = [&](int jb, int b, bool first_of_tile) {
        mbar_wait(&y_full[b], (yfph >> b) & 1);  // Y[b] written (and acc1[b] drained)
        yfph ^= 1u << b;
        if (first_of_tile) {  // acc2 drained by the previous tile's epilogue
          mbar_wait(a2_empty, a2eph ^ 1);
          a2eph ^= 1;
        }
        tc_fence_after();
        for (int kc = 0; kc < kc_per_block; ++kc) {
          mbar_wait(&w7_full[w7s], w7ph);
          tc_fence_after();
          const uint64_t ya = desc_sw128(y_base + b * 32768 + kc * 16384), wb = desc_sw128(w7_base + w7s * 8192);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // a 32-byte K step adds 2 to a descriptor
            mma_bf16_ss(tmem + kAcc2Col, ya + 2 * kk, wb + 2 * kk, idesc2,
                        (first_of_tile && kc == 0 && kk == 0) ? 0u : 1u);
          mma_commit(&w7_empty[w7s]);
          if (++w7s == kW7Stages) { w7s = 0; w7ph ^= 1; }
        }
        mma_commit(&y_empty[b]);
        (void)jb;
      };
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
        for (int j = 0; j < p.blocks; ++j, ++bc) {
          const int b = bc & 1;
          // acc1[b] is free: its previous block's y_full was waited in the
          // MMA2 issued before this point
          for (int c = 0; c < p.cin_chunks; ++c) {
            mbar_wait(&x_full[xs], xph);
            mbar_wait(&w6_full[w6s], w6ph);
            tc_fence_after();
            const uint64_t xa = desc_sw128(x_base + xs * 16384), wb = desc_sw128(w6_base + w6s * 16384);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16_ss(tmem + b * NB, xa + 2 * kk, wb + 2 * kk, idesc1,
                          (c == 0 && kk == 0) ? 0u : 1u);
            mma_commit(&x_empty[xs]);
            mma_commit(&w6_empty[w6s]);
            if (++xs == kXStages) { xs = 0; xph ^= 1; }
            if (++w6s == kW6Stages) { w6s = 0; w6ph ^= 1; }
          }
          mma_commit(&a1_full[b]);
          if (j > 0) mma2(j - 1, b ^ 1, j == 1);  // the previous block, converted meanwhile
        }
        mma2(p.blocks - 1, (bc - 1) & 1, p.blocks == 1);
        mma_commit(a2_full);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogues
    const uint32_t quad = warp & 3;
    const int sub = (int(warp) - 2) >> 2;  // which half of the columns this warp converts
    const uint32_t lane = lane_id();
    const int ep = int(threadIdx.x) - 64;  // 0..255, loader index for the bias slices
    // warp w may only touch TMEM lanes 32(w%4)..+31: this thread's pixel (and
    // its TMEM lane, and its row of Y) is 32 quad + lane
    const int px = int(quad) * 32 + int(lane);
    const uint32_t lane_base = (quad * 32) << 16;
    uint8_t* stg_w = stg + (int(warp) - 2) * 2048;
    uint8_t* yrow = sy + px * 128;  // this pixel's row in every 16 KB Y chunk
    uint32_t a1ph = 0, yeph = 0, a2fph = 0;  // phase bit per buffer (bit b)
    int bc = 0;
    for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
      int gi, n, pt;
      head_decode(p, t, gi, n, pt);
      const HeadGroup& g = p.g[gi];
      const int o = pt * 128 + px;  // padded-width output position of this pixel
      const int hh = o / p.Wp;
      const int ww = o - hh * p.Wp;
      const bool valid = hh < p.H && ww < p.W;
      for (int j = 0; j < p.blocks; ++j, ++bc) {
        const int b = bc & 1;
        float* bs = sb6 + b * NB;
        float* ss = ss6 + b * NB;
        // this block's bias / slope: every epilogue warp is done with the
        // slices' previous block (and the previous tile's b7) before they change
        named_bar_sync(1, kHEpi);
        if (ep < NB) {
          const int co = j * NB + ep;
          bs[ep] = g.bias6[co];
          ss[ep] = g.act6 == 1 ? 0.f : g.act6 == 2 ? g.slope6[co] : 1.f;
        } else if (j == 0 && ep < NB + 64) {
          sb7[ep - NB] = ep - NB < g.c7 ? g.bias7[ep - NB] : 0.f;
        }
        named_bar_sync(1, kHEpi);
        mbar_wait(&y_empty[b], ((yeph >> b) & 1) ^ 1);  // MMA2 of this buffer's previous block released Y[b]
        yeph ^= 1u << b;
        mbar_wait(&a1_full[b], (a1ph >> b) & 1);
        a1ph ^= 1u << b;
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < NB / 2; cc += 32) {
          const int c0 = sub * (NB / 2) + cc;
          uint32_t v[32];
          tmem_ld32(tmem + lane_base + b * NB + c0, v);
          tmem_ld_wait();
          uint8_t* chunk = yrow + b * 32768 + (c0 >> 6) * 16384;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t w[4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const int c = c0 + q * 8 + 2 * jj;
              float x0 = __uint_as_float(v[q * 8 + 2 * jj]) + bs[c];
              float x1 = __uint_as_float(v[q * 8 + 2 * jj + 1]) + bs[c + 1];
              x0 = fmaxf(x0, 0.f) + ss[c] * fminf(x0, 0.f);
              x1 = fmaxf(x1, 0.f) + ss[c + 1] * fminf(x1, 0.f);
              w[jj] = pack2(x0, x1);
            }
            const uint32_t qq = ((c0 & 63) >> 3) + q;  // 16-byte chunk within the 128-byte row
            *reinterpret_cast<uint4*>(chunk + ((qq ^ (uint32_t(px) & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&y_full[b]);
      }
      // ---- epilogue 2: acc2 (+ b7) -> outputs; this warp: channels 32 sub .. 32 sub + 31
      mbar_wait(a2_full, a2fph);
      a2fph ^= 1;
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(tmem + lane_base + kAcc2Col + sub * 32, v);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(a2_empty);
      const int cb = sub * 32;  // first channel of this warp
      float zf[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) zf[c] = __uint_as_float(v[c]) + sb7[cb + c];
      if (g.out2 != nullptr && valid) {  // fp32 NCHW copy for the wire
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (cb + c < g.c7)
            g.out2[((static_cast<size_t>(n) * g.out2_c_stride + g.out2_c_off + cb + c) * p.H + hh) * p.W + ww] =
                zf[c];
      }
      if (g.out_mode == kOutNchwF32) {
        if (valid) {
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (cb + c < g.c7)
              static_cast<float*>(g.out)[((static_cast<size_t>(n) * g.out_c_stride + g.out_c_off + cb + c) * p.H +
                                          hh) * p.W + ww] = zf[c];
        }
        continue;
      }
      // bf16 into the stage concat: round_up(c7, 8) channels as 32/16/8-channel
      // boxes of this warp's 32 pixels (channels past c7 carry zero weights and
      // bias, so they store zeros)
      uint32_t packed[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) packed[i] = valid ? pack2(zf[2 * i], zf[2 * i + 1]) : 0u;
      const int row_w = p.P * p.Wp + p.P + pt * 128 + int(quad) * 32;
      const int c_end = (g.c7 + 7) & ~7;
      auto box = [&](auto width, auto first) {
        constexpr int W = decltype(width)::value;
        constexpr int c0 = decltype(first)::value;  // relative to this warp's first channel
        if (lane == 0) bulk_wait_read<0>();  // this warp's previous store has read the staging box
        __syncwarp();
#pragma unroll
        for (int q = 0; q < W / 8; ++q) {
          const int w0 = (c0 >> 1) + q * 4;  // packed word of channel c0 + 8q
          uint32_t w[4];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) w[jj] = packed[w0 + jj];
          uint32_t off;
          if constexpr (W == 32) off = lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4);
          else if constexpr (W == 16) off = lane * 32 + ((q ^ ((lane >> 2) & 1)) << 4);
          else off = lane * 16;
          *reinterpret_cast<uint4*>(stg_w + off) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const CUtensorMap* m = W == 32 ? &maps.out32[gi] : W == 16 ? &maps.out16[gi] : &maps.out8[gi];
          tma_store_3d(m, stg_w, g.out_c_off + cb + c0, row_w, n);
          bulk_commit();
        }
      };
      // this warp's channels: [cb, min(c_end, cb + 32)), a 32-channel box or 16/8 tails
      using I0 = std::integral_constant<int, 0>;
      using I16 = std::integral_constant<int, 16>;
      using B8 = std::integral_constant<int, 8>;
      using B16 = std::integral_constant<int, 16>;
      using B32 = std::integral_constant<int, 32>;
      switch (c_end - cb) {
        case 8: box(B8{}, I0{}); break;
        case 16: box(B16{}, I0{}); break;
        case 24: box(B16{}, I0{}); box(B8{}, I16{}); break;
        default:
          if (c_end - cb >= 32) box(B32{}, I0{});
          break;
      }
    }
    if (lane_id() == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kHTmemCols>(tmem);
  }
}

// ------------------------------------------------------------------------
// CTA-pair head (cta_group::2), for c6 >= 256 and cin <= 384 (BODY_25's
// stage heads). A 128-pixel tile per CTA, M = 256 per MMA over the pair:
//  * each CTA keeps its X tile resident for all c6 blocks (6 chunk slots,
//    each refilled with the next tile's chunk as soon as the last block's
//    MMA1 has read it), instead of re-reading it per block;
//  * each CTA loads half of every W6 block (64 of 128 rows) and half of W7
//    (32 of 64 rows), so the per-SM weight stream halves too.
// Per 128 pixels that is 96 KB of X + 192 KB of W6 + 32 KB of W7 from L2,
// against 384 + 384 + 64 KB for the single-CTA kernel (whose BODY_25 heads
// are L2-bound). Warps: 0 W6 producer, 1 MMA issuer (leader), 2-9 epilogues,
// 10 X producer, 11 W7 producer. Full barriers and the epilogue-to-MMA
// barriers live in the leader; the rest are multicast commits.
constexpr int kH2Threads = 384;
constexpr int kH2XChunks = 6;
constexpr int kH2W6Stages = 4;
constexpr int kH2W7Stages = 2;

struct Head2Smem {
  static constexpr int x = 0;                                // 6 x [128 px][64 ch]
  static constexpr int w6 = x + kH2XChunks * 16384;          // stages x [64 rows][64]
  static constexpr int y = w6 + kH2W6Stages * 8192;          // 2 x [128 px][128 ch] (2 SW128 chunks each)
  static constexpr int w7 = y + 2 * 32768;                   // stages x [32 rows][64]
  static constexpr int stg = w7 + kH2W7Stages * 4096;        // 8 warps x [32 px][<=32 ch]
  static constexpr int bias = stg + 8 * 2048;                // b6/s6 per Y buffer (2 x 2 x 128) + b7 (64)
  static constexpr int bars = bias + (4 * kNB + 64) * 4;
  static constexpr int total = bars + 512;
  static_assert(total + 1024 <= 232448, "smem budget");
};

__global__ void __launch_bounds__(kH2Threads, 1)
    conv_head2_kernel(const __grid_constant__ HeadMaps maps, const __grid_constant__ HeadParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* sx = smem + Head2Smem::x;
  uint8_t* sw6 = smem + Head2Smem::w6;
  uint8_t* sy = smem + Head2Smem::y;
  uint8_t* sw7 = smem + Head2Smem::w7;
  uint8_t* stg = smem + Head2Smem::stg;
  float* sb6 = reinterpret_cast<float*>(smem + Head2Smem::bias);  // [2][128]
  float* ss6 = sb6 + 2 * kNB;                                      // [2][128]
  float* sb7 = ss6 + 2 * kNB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Head2Smem::bars);
  uint64_t* x_full = bars;                        // [6] leader
  uint64_t* x_empty = x_full + kH2XChunks;        // [6] multicast commit
  uint64_t* w6_full = x_empty + kH2XChunks;       // leader
  uint64_t* w6_empty = w6_full + kH2W6Stages;
  uint64_t* w7_full = w6_empty + kH2W6Stages;     // leader
  uint64_t* w7_empty = w7_full + kH2W7Stages;
  uint64_t* a1_full = w7_empty + kH2W7Stages;     // [2] multicast commit
  uint64_t* y_full = a1_full + 2;                 // [2] leader, 16 warp arrivals
  uint64_t* y_empty = y_full + 2;                 // [2] multicast commit
  uint64_t* a2_full = y_empty + 2;                // multicast commit
  uint64_t* a2_empty = a2_full + 1;               // leader, 16 warp arrivals
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a2_empty + 1);

  const uint32_t warp = warp_id();
  const uint32_t rank = cluster_cta_rank();
  const bool leader = rank == 0;
  constexpr int NB = kNB;
  if (warp == 0 && elect_one()) {
    for (int g = 0; g < p.n_groups; ++g) {
      tma_prefetch(&maps.x[g]);
      tma_prefetch(&maps.w6[g]);
      tma_prefetch(&maps.w7[g]);
    }
    for (int i = 0; i < kH2XChunks; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < kH2W6Stages; ++i) { mbar_init(&w6_full[i], 1); mbar_init(&w6_empty[i], 1); }
    for (int i = 0; i < kH2W7Stages; ++i) { mbar_init(&w7_full[i], 1); mbar_init(&w7_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a1_full[i], 1);
      mbar_init(&y_full[i], 16);
      mbar_init(&y_empty[i], 1);
    }
    mbar_init(a2_full, 1);
    mbar_init(a2_empty, 16);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<kHTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int t_begin = int(blockIdx.x) / 2, t_step = int(gridDim.x) / 2;

  if (warp == 10) {
    // ------------------------------------------------------------ X producer
    if (elect_one()) {
      uint32_t xph = 0;
      for (int t = t_begin; t < p.total_tiles; t += t_step, xph ^= 1) {
        int g, n, ptp;
        head_decode(p, t, g, n, ptp);
        const int row0 = n * p.Hp * p.Wp + p.P * (p.Wp + 1) + (ptp * 2 + int(rank)) * 128;
        for (int c = 0; c < p.cin_chunks; ++c) {
          mbar_wait(&x_empty[c], xph ^ 1);  // the previous tile's last block read chunk c
          if (leader) mbar_arrive_expect_tx(&x_full[c], 2 * 16384);
          tma_load_2d_pair(sx + c * 16384, &maps.x[g], mapa_shared(&x_full[c], 0), p.in_c_off + c * 64, row0);
        }
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------ W6 producer (this CTA's half rows)
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      int s6 = 0;
      uint32_t ph = 0;
      for (int t = t_begin; t < p.total_tiles; t += t_step) {
        int g, n, ptp;
        head_decode(p, t, g, n, ptp);
        for (int j = 0; j < p.blocks; ++j)
          for (int c = 0; c < p.cin_chunks; ++c) {
            mbar_wait(&w6_empty[s6], ph ^ 1);
            if (leader) mbar_arrive_expect_tx(&w6_full[s6], 2 * 8192);
            tma_load_2d_pair_hint(sw6 + s6 * 8192, &maps.w6[g], mapa_shared(&w6_full[s6], 0), c * 64,
                                  j * NB + int(rank) * (NB / 2), keep);
            if (++s6 == kH2W6Stages) { s6 = 0; ph ^= 1; }
          }
      }
    }
  } else if (warp == 11) {
    // ------------------------------------------------------------ W7 producer (this CTA's 32 rows)
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      int s7 = 0;
      uint32_t ph = 0;
      for (int t = t_begin; t < p.total_tiles; t += t_step) {
        int g, n, ptp;
        head_decode(p, t, g, n, ptp);
        for (int j = 0; j < p.blocks; ++j)
          for (int kc = 0; kc < NB / 64; ++kc) {
            mbar_wait(&w7_empty[s7], ph ^ 1);
            if (leader) mbar_arrive_expect_tx(&w7_full[s7], 2 * 4096);
            tma_load_2d_pair_hint(sw7 + s7 * 4096, &maps.w7[g], mapa_shared(&w7_full[s7], 0), j * NB + kc * 64,
                                  int(rank) * 32, keep);
            if (++s7 == kH2W7Stages) { s7 = 0; ph ^= 1; }
          }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    if (leader && elect_one()) {
      const uint32_t idesc1 = idesc_bf16_f32(256, NB);
      const uint32_t idesc2 = idesc_bf16_f32(256, 64);
      int s6 = 0, s7 = 0;
      uint32_t ph6 = 0, ph7 = 0, xph = 0, a2eph = 0, yfph = 0;
      int bc = 0;
      const uint32_t x_base = smem_u32(sx), w6_base = smem_u32(sw6), y_base = smem_u32(sy),
                     w7_base = smem_u32(sw7);
      auto mma2 = [&](int b, bool first_of_tile) {
        mbar_wait(&y_full[b], (yfph >> b) & 1);  // both CTAs' Y[b] written, acc1[b] drained
        yfph ^= 1u << b;
        if (first_of_tile) {
          mbar_wait(a2_empty, a2eph ^ 1);
          a2eph ^= 1;
        }
        tc_fence_after();
        for (int kc = 0; kc < NB / 64; ++kc) {
          mbar_wait(&w7_full[s7], ph7);
          tc_fence_after();
          const uint64_t ya = desc_sw128(y_base + b * 32768 + kc * 16384), wb = desc_sw128(w7_base + s7 * 4096);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // a 32-byte K step adds 2 to a descriptor
            mma_bf16_ss_pair(tmem + kAcc2Col, ya + 2 * kk, wb + 2 * kk, idesc2,
                             (first_of_tile && kc == 0 && kk == 0) ? 0u : 1u);
          mma_commit_pair(&w7_empty[s7]);
          if (++s7 == kH2W7Stages) { s7 = 0; ph7 ^= 1; }
        }
        mma_commit_pair(&y_empty[b]);
      };
      for (int t = t_begin; t < p.total_tiles; t += t_step, xph ^= 1) {
        for (int j = 0; j < p.blocks; ++j, ++bc) {
          const int b = bc & 1;
          for (int c = 0; c < p.cin_chunks; ++c) {
            if (j == 0) mbar_wait(&x_full[c], xph);
            mbar_wait(&w6_full[s6], ph6);
            tc_fence_after();
            const uint64_t xa = desc_sw128(x_base + c * 16384), wb = desc_sw128(w6_base + s6 * 8192);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16_ss_pair(tmem + b * NB, xa + 2 * kk, wb + 2 * kk, idesc1,
                               (c == 0 && kk == 0) ? 0u : 1u);
            mma_commit_pair(&w6_empty[s6]);
            if (j == p.blocks - 1) mma_commit_pair(&x_empty[c]);  // the next tile may refill chunk c
            if (++s6 == kH2W6Stages) { s6 = 0; ph6 ^= 1; }
          }
          mma_commit_pair(&a1_full[b]);
          if (j > 0) mma2(b ^ 1, j == 1);  // the previous block, converted meanwhile
        }
        mma2((bc - 1) & 1, p.blocks == 1);
        mma_commit_pair(a2_full);
      }
    }
  } else if (warp >= 2 && warp <= 9) {
    // ------------------------------------------------------------ epilogues (this CTA's 128 pixels)
    const uint32_t quad = warp & 3;
    const int sub = (int(warp) - 2) >> 2;
    const uint32_t lane = lane_id();
    const int ep = int(threadIdx.x) - 64;  // 0..255
    const int px = int(quad) * 32 + int(lane);
    const uint32_t lane_base = (quad * 32) << 16;
    uint8_t* stg_w = stg + (int(warp) - 2) * 2048;
    uint8_t* yrow = sy + px * 128;
    uint32_t a1ph = 0, yeph = 0, a2fph = 0;
    const uint32_t a2_empty_leader = mapa_shared(a2_empty, 0);
    int bc = 0;
    for (int t = t_begin; t < p.total_tiles; t += t_step) {
      int gi, n, ptp;
      head_decode(p, t, gi, n, ptp);
      const int pt = ptp * 2 + int(rank);
      const HeadGroup& g = p.g[gi];
      const int o = pt * 128 + px;
      const int hh = o / p.Wp;
      const int ww = o - hh * p.Wp;
      const bool valid = hh < p.H && ww < p.W;
      for (int j = 0; j < p.blocks; ++j, ++bc) {
        const int b = bc & 1;
        float* bs = sb6 + b * NB;
        float* ss = ss6 + b * NB;
        named_bar_sync(1, 256);
        if (ep < NB) {
          const int co = j * NB + ep;
          bs[ep] = g.bias6[co];
          ss[ep] = g.act6 == 1 ? 0.f : g.act6 == 2 ? g.slope6[co] : 1.f;
        } else if (j == 0 && ep < NB + 64) {
          sb7[ep - NB] = ep - NB < g.c7 ? g.bias7[ep - NB] : 0.f;
        }
        named_bar_sync(1, 256);
        mbar_wait(&y_empty[b], ((yeph >> b) & 1) ^ 1);
        yeph ^= 1u << b;
        mbar_wait(&a1_full[b], (a1ph >> b) & 1);
        a1ph ^= 1u << b;
        tc_fence_after();
#pragma unroll
        for (int cc = 0; cc < NB / 2; cc += 32) {
          const int c0 = sub * (NB / 2) + cc;
          uint32_t v[32];
          tmem_ld32(tmem + lane_base + b * NB + c0, v);
          tmem_ld_wait();
          uint8_t* chunk = yrow + b * 32768 + (c0 >> 6) * 16384;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t w[4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const int c = c0 + q * 8 + 2 * jj;
              float x0 = __uint_as_float(v[q * 8 + 2 * jj]) + bs[c];
              float x1 = __uint_as_float(v[q * 8 + 2 * jj + 1]) + bs[c + 1];
              x0 = fmaxf(x0, 0.f) + ss[c] * fminf(x0, 0.f);
              x1 = fmaxf(x1, 0.f) + ss[c + 1] * fminf(x1, 0.f);
              w[jj] = pack2(x0, x1);
            }
            const uint32_t qq = ((c0 & 63) >> 3) + q;
            *reinterpret_cast<uint4*>(chunk + ((qq ^ (uint32_t(px) & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        // default-semantics remote arrive after fence.proxy.async, as CUTLASS's
        // ClusterBarrier: a cluster-scope release costs a MEMBAR + ERRBAR per
        // block and warp (the top stall site when measured)
        if (lane == 0) mbar_arrive_cluster(mapa_shared(&y_full[b], 0));
      }
      // ---- epilogue 2: acc2 (+ b7) -> outputs; this warp: channels 32 sub .. 32 sub + 31
      mbar_wait(a2_full, a2fph);
      a2fph ^= 1;
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(tmem + lane_base + kAcc2Col + sub * 32, v);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(a2_empty_leader);
      const int cb = sub * 32;
      float zf[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) zf[c] = __uint_as_float(v[c]) + sb7[cb + c];
      if (g.out2 != nullptr && valid) {
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (cb + c < g.c7)
            g.out2[((static_cast<size_t>(n) * g.out2_c_stride + g.out2_c_off + cb + c) * p.H + hh) * p.W + ww] =
                zf[c];
      }
      if (g.out_mode == kOutNchwF32) {
        if (valid) {
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (cb + c < g.c7)
              static_cast<float*>(g.out)[((static_cast<size_t>(n) * g.out_c_stride + g.out_c_off + cb + c) * p.H +
                                          hh) * p.W + ww] = zf[c];
        }
        continue;
      }
      uint32_t packed[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) packed[i] = valid ? pack2(zf[2 * i], zf[2 * i + 1]) : 0u;
      const int row_w = p.P * p.Wp + p.P + pt * 128 + int(quad) * 32;
      const int c_end = (g.c7 + 7) & ~7;
      auto box = [&](auto width, auto first) {
        constexpr int W = decltype(width)::value;
        constexpr int c0 = decltype(first)::value;
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
#pragma unroll
        for (int q = 0; q < W / 8; ++q) {
          const int w0 = (c0 >> 1) + q * 4;
          uint32_t w[4];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) w[jj] = packed[w0 + jj];
          uint32_t off;
          if constexpr (W == 32) off = lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4);
          else if constexpr (W == 16) off = lane * 32 + ((q ^ ((lane >> 2) & 1)) << 4);
          else off = lane * 16;
          *reinterpret_cast<uint4*>(stg_w + off) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const CUtensorMap* m = W == 32 ? &maps.out32[gi] : W == 16 ? &maps.out16[gi] : &maps.out8[gi];
          tma_store_3d(m, stg_w, g.out_c_off + cb + c0, row_w, n);
          bulk_commit();
        }
      };
      using I0 = std::integral_constant<int, 0>;
      using I16 = std::integral_constant<int, 16>;
      using B8 = std::integral_constant<int, 8>;
      using B16 = std::integral_constant<int, 16>;
      using B32 = std::integral_constant<int, 32>;
      switch (c_end - cb) {
        case 8: box(B8{}, I0{}); break;
        case 16: box(B16{}, I0{}); break;
        case 24: box(B16{}, I0{}); box(B8{}, I16{}); break;
        default:
          if (c_end - cb >= 32) box(B32{}, I0{});
          break;
      }
    }
    if (lane_id() == 0) bulk_wait<0>();
  }
  tc_fence_before();
  cluster_sync_all();  // the leader's MMAs read peer smem until the end
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<kHTmemCols>(tmem);
  }
}

}  // namespace

void conv_head_configure() {
  check_cuda(cudaFuncSetAttribute(conv_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  HeadSmem::total + 1024),
             "conv_head smem attribute");
  check_cuda(cudaFuncSetAttribute(conv_head2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  Head2Smem::total + 1024),
             "conv_head2 smem attribute");
}

int conv_head_pair_max_chunks() { return kH2XChunks; }

void launch_conv_head(const HeadMaps& maps, const HeadParams& p, int sm_count, cudaStream_t stream) {
  if (p.ncta == 2) {  // CTA pairs: p.total_tiles counts pairs of 128-pixel tiles
    const int pairs = sm_count / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (p.total_tiles < pairs ? p.total_tiles : pairs));
    cfg.blockDim = dim3(kH2Threads);
    cfg.dynamicSmemBytes = Head2Smem::total + 1024;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    check_cuda(cudaLaunchKernelEx(&cfg, conv_head2_kernel, maps, p), "conv_head2 launch");
    return;
  }
  const int grid = p.total_tiles < sm_count ? p.total_tiles : sm_count;
  conv_head_kernel<<<grid, kHThreads, HeadSmem::total + 1024, stream>>>(maps, p);
  check_cuda(cudaGetLastError(), "conv_head launch");
}

}  // namespace avec
