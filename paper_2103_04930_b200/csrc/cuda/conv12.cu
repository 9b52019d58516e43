// conv1_1 + conv1_2 + pool1 in one tcgen05 kernel (sm_100a): the 64-channel
// full-resolution conv1_1 activation never reaches HBM.
//
// Tile = output rows y0, y0+1 (y0 even) at columns x0 .. x0+125 (x0 = 126 cb):
// conv1_2 needs conv1_1 at rows y0-1 .. y0+2 and padded columns x0 .. x0+127,
// i.e. four 128-position windows — exactly one M = 128 MMA each.
//   producer  TMA of the fp32 frame patch [3 ch][rows y0-2..y0+3][132 cols from
//             (x0-2) & ~3] (zero-filled outside the frame; a TMA inner
//             coordinate must be 16-byte aligned — an unaligned one is an
//             illegal instruction, tests/native/tma3d_probe.cu); conv1_1's
//             and conv1_2's weights once per CTA (conv1_2's 72 KB stay
//             resident as [W(2,s); W(1,s); W(0,s)] per column tap s)
//   epilogue  A: im2col of the 27 taps per window position (x - 0.5, 0 outside
//                the frame) into a K = 32 SW64 im2col buffer; taps 27 and 28
//                are 1.0, against conv1_1's bias split hi + lo into its
//                weights there (engine.cu upload), so acc1 includes the bias
//   MMA       conv1_1: 4 windows x 2 MMAs (M128 N64 K16) -> acc1[4] in TMEM
//   epilogue  B: acc1 -> ReLU, 0 outside the image, bf16 -> the tile's four
//                window slots of a 6-slot ring (conv1_2's A operand, SW128
//                K-major), each once conv1_2 released the slot's last use
//   MMA       conv1_2: window w (shifted by s positions) feeds output row 0
//             with W(w,s) and output row 1 with W(w-1,s). The two middle
//             windows do both in one N = 128 MMA against the adjacent
//             [W(w,s); W(w-1,s)] rows (64 cycles, at the tensor rate), the
//             outer two one N = 64 MMA each: 224 cycles per K16 step instead of
//             six N = 64 MMAs at the 48-cycle shared-memory operand floor (288;
//             profiles/r01_tc_probe.json) -> acc2[stage]. Windows (0, 1) run
//             first, interleaved per K step, then (2, 3), so the first pair's
//             slots are released half-way through the tile
//   epilogue  C: 2x2 max of the raw sums, bias, ReLU, bf16 -> pooled row
//             y0/2, columns x0/2 .. x0/2+62 through a 4D TMA map (the 127th/
//             128th positions read past their window and are never stored)
// The MMA warp issues conv1_1(t+1) before conv1_2(t), so the im2col of tile
// t+2, the conv1_1 epilogue of tile t+1 (into the slots conv1_2(t) released
// first) and the pooled epilogue of tile t-1 all overlap conv1_2 of tile t. Same bf16
// operands as the separate conv_first + pooled conv1_2 path; the fp32 sums run
// in another tap order, so the two agree to bf16 rounding, not bit for bit.
#include <cuda_bf16.h>

#include <cstdlib>

#include "conv_tc.cuh"
#include "engine.hpp"
#include "ptx.cuh"

namespace avec {

namespace {

using namespace ptx;

// SUBS = epilogue warps per TMEM lane quadrant: 2 (default; 152 vs 156 us at
// C2, 2.52-2.58 vs 2.62-2.65 ms at C5) or 4 (AVEC_C12_SUBS=4)
template <int SUBS>
struct C12Cfg {
  static constexpr int kEpi = 128 * SUBS;
  static constexpr int kThreads = 64 + kEpi + 32;  // weights, MMA, epilogue warps, frame patches
  static constexpr int kPatchWarp = 2 + 4 * SUBS;
  static constexpr int kWinPerSub = 4 / SUBS;      // windows per epilogue warp (im2col, conv1_1 epilogue)
  static constexpr int kChPerSub = 64 / SUBS;      // pooled channels per epilogue warp
};
constexpr uint32_t kTmemCols = 512;
constexpr int kTileCols = 126;  // output columns per tile (even: whole pooled columns)
constexpr int kPatchCols = 132;
constexpr int kPatchRows = 6;
constexpr int kPatchBytes = 3 * kPatchRows * kPatchCols * 4;  // 9504
// conv1_2's weights stay resident for the CTA's lifetime (72 KB): per column
// tap s, [W(2,s); W(1,s); W(0,s)] x [64 cout][64 K] bf16 SW128, 8 KB each. A
// ring of 3 x 12 KB stages reloaded 72 KB per tile from L2 and left the MMA
// warp waiting on weights (16% of its samples); the 6-slot window ring below
// is what frees the room.
constexpr int kWBlk = 64 * 64 * 2;       // one W(r,s) block, bytes
constexpr int kW12Tap = 3 * kWBlk;       // the three filter rows of one column tap
// conv1_1 output windows: a ring of 6 slots instead of 2 x 4 buffers. conv1_2
// reads a tile's windows in order (window-outer MMAs), so a tile's first two
// slots free early and the next tile's conv1_1 epilogue reuses them.
constexpr int kWinSlots = 6;
constexpr int kAcc2Col = 256;  // acc2[2 stages] at 256..383, 384..511 (2 rows x 64 each)

struct Smem12 {
  static constexpr int win = 0;                          // kWinSlots x [128][64] bf16 SW128
  static constexpr int imc = win + kWinSlots * 16384;    // 4 windows x [128][32] bf16 SW64 (im2col)
  static constexpr int w12 = imc + 4 * 8192;             // 3 x kW12Tap, resident
  static constexpr int w11 = w12 + 3 * kW12Tap;          // [64 cout][32 K] SW64 (K 29 used)
  static constexpr int patch = w11 + 4096;               // [3][6][132] fp32 (one buffer: the
                                                         // next patch has a whole tile to land)
  static constexpr int stg = patch + 10240;              // 4 warps x [16 px][64 ch] (pooled box)
  static constexpr int bias = stg + 4 * 2048;            // conv1_2 bias (64; room for 128)
  static constexpr int bars = bias + 2 * 64 * 4;
  static constexpr int total = bars + 256;
  static_assert((2 + 2 + 1 + 1 + 1 + 1 + 2 + kWinSlots + 2 + 2) * 8 + 4 <= 256, "barrier block");
  static_assert(total + 1024 <= 232448, "smem budget");
};

// bf16x2 {relu(a), relu(b)} (a in the low half) in one cvt: rn(relu(x)) == relu(rn(x))
__device__ __forceinline__ uint32_t pack2_relu(float a, float b) {
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(b), "f"(a));
  return d;
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void tile_of(const ConvParams& p, int t, int& n, int& y0, int& x0) {
  n = t / p.tiles_per_image;
  const int rem = t - n * p.tiles_per_image;
  const int rp = rem / p.col_blocks;
  y0 = 2 * rp;
  x0 = (rem - rp * p.col_blocks) * kTileCols;
}

// maps.act_big[0]: fp32 frames [N*3][H][W], box {132, 6, 3}; maps.wgt[0]:
// conv1_2 weights, maps.wgt[1]: conv1_1 weights (box {64, 64}); maps.out_pool[0]
// / [1]: pooled 4D stores with 16 / 15-column boxes. p.g[0] = conv1_2, p.g[1] = conv1_1.
template <int SUBS>
__global__ void __launch_bounds__(C12Cfg<SUBS>::kThreads, 1)
    conv12_kernel(const __grid_constant__ ConvMaps maps, const __grid_constant__ ConvParams p) {
  using Cfg = C12Cfg<SUBS>;
  constexpr int kSubs = SUBS, kEpi = Cfg::kEpi, kPatchWarp = Cfg::kPatchWarp;
  constexpr int kWinPerSub = Cfg::kWinPerSub, kChPerSub = Cfg::kChPerSub;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* win = smem + Smem12::win;
  uint8_t* imc = smem + Smem12::imc;
  uint8_t* w12 = smem + Smem12::w12;
  uint8_t* w11 = smem + Smem12::w11;
  float* patch = reinterpret_cast<float*>(smem + Smem12::patch);
  uint8_t* stg = smem + Smem12::stg;
  float* b12 = reinterpret_cast<float*>(smem + Smem12::bias);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem12::bars);
  uint64_t* patch_full = bars;             // [2] (only [0] used)
  uint64_t* patch_empty = patch_full + 2;  // [2] 128 arrivals
  uint64_t* w11_full = patch_empty + 2;
  uint64_t* w12_full = w11_full + 1;            // the resident conv1_2 weights landed
  uint64_t* imc_full = w12_full + 1;            // 128 arrivals: im2col written
  uint64_t* a1_full = imc_full + 1;             // conv1_1 MMAs done (acc1 ready, im2col free)
  uint64_t* win_full = a1_full + 1;             // [2] by tile parity: its 4 windows written, acc1 drained
  uint64_t* slot_empty = win_full + 2;          // [kWinSlots] conv1_2 MMAs done with a window slot
  uint64_t* acc2_full = slot_empty + kWinSlots; // [2]
  uint64_t* acc2_empty = acc2_full + 2;         // [2] 128 arrivals
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc2_empty + 2);

  const uint32_t warp = warp_id();
  if (warp == 0 && elect_one()) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&patch_full[i], 1);
      mbar_init(&patch_empty[i], kEpi);
      mbar_init(&win_full[i], kEpi);
      mbar_init(&acc2_full[i], 1);
      mbar_init(&acc2_empty[i], kEpi);
    }
    for (int i = 0; i < kWinSlots; ++i) mbar_init(&slot_empty[i], 1);
    mbar_init(w11_full, 1);
    mbar_init(w12_full, 1);
    mbar_init(imc_full, kEpi);
    mbar_init(a1_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      mbar_arrive_expect_tx(w11_full, 4096);
      tma_load_2d(w11, &maps.wgt[1], w11_full, 0, 0);
      mbar_arrive_expect_tx(w12_full, 3 * kW12Tap);
      for (int s = 0; s < 3; ++s)
        for (int r = 2; r >= 0; --r)  // K index (r*3 + s)*64 + cin
          tma_load_2d(w12 + s * kW12Tap + (2 - r) * kWBlk, &maps.wgt[0], w12_full, (r * 3 + s) * 64, 0);
    }
  } else if (warp == kPatchWarp) {
    // ------------------------------------------------------------ frame patches
    // its own warp, so a patch lands as soon as its buffer frees (the im2col
    // of tile t+1 runs before conv1_2 of tile t and must not wait on HBM)
    if (elect_one()) {
      int it = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++it) {
        int n, y0, x0;
        tile_of(p, t, n, y0, x0);
        mbar_wait(&patch_empty[0], (it & 1) ^ 1);
        mbar_arrive_expect_tx(&patch_full[0], kPatchBytes);
        tma_load_3d(patch, &maps.act_big[0], &patch_full[0], (x0 - 2) & ~3, y0 - 2, n * 3);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // order per tile t: conv1_1(t+1) (once act11(t) drained acc1 and the
    // im2col of t+1 is written), then conv1_2(t) — the tensor pipe runs them
    // in issue order, so act11(t+1) overlaps conv1_2(t)
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16_f32(128, 64), idesc2 = idesc_bf16_f32(128, 128);
      const uint32_t win_base = smem_u32(win), imc_base = smem_u32(imc);
      const uint32_t w12_base = smem_u32(w12), w11_base = smem_u32(w11);
      auto conv11 = [&](uint32_t ph) {
        mbar_wait(imc_full, ph);
        tc_fence_after();
        const uint64_t bd11 = desc_sw64(w11_base);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t ad = desc_sw64(imc_base + j * 8192);
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)  // K = 32 covers the 27 taps; a 32-byte K step adds 2 to a descriptor
            mma_bf16_ss(tmem + j * 64, ad + 2 * kk, bd11 + 2 * kk, idesc, kk ? 1u : 0u);
        }
        mma_commit(a1_full);
      };
      mbar_wait(w11_full, 0);
      if (int(blockIdx.x) < p.total_tiles) conv11(0);
      mbar_wait(w12_full, 0);
      int it = 0;
      for (int t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++it) {
        const int b = it & 1;  // acc2 stage, window-written barrier
        const uint32_t bph = (it >> 1) & 1;
        mbar_wait(&win_full[b], bph);
        if (t + int(gridDim.x) < p.total_tiles) conv11((it + 1) & 1);
        mbar_wait(&acc2_empty[b], bph ^ 1);
        tc_fence_after();
        // acc2: output row 0 at columns d0 .. d0+63, row 1 at d0+64 .. d0+127.
        // Window w (shifted by s positions) feeds row 0 with W(w,s) and row 1
        // with W(w-1,s); the middle two in one N = 128 MMA against the
        // adjacent [W(w,s); W(w-1,s)] rows, the outer two N = 64. Windows 0
        // and 1 first (interleaved per K step), then 2 and 3: the first pair's
        // slots are released half-way through the tile.
        const uint32_t d0 = tmem + kAcc2Col + b * 128;
#pragma unroll 1
        for (int hp = 0; hp < 2; ++hp) {  // windows (0, 1), then (2, 3), interleaved per K step
          const int slot_a = (4 * it + 2 * hp) % kWinSlots, slot_b = (4 * it + 2 * hp + 1) % kWinSlots;
          const uint32_t wa = win_base + slot_a * 16384, wb2 = win_base + slot_b * 16384;
#pragma unroll
          for (int s = 0; s < 3; ++s) {
            // W(2,s) at +0, W(1,s) at +8 KB, W(0,s) at +16 KB (512 descriptor units each)
            const uint64_t b2 = desc_sw128(w12_base + s * kW12Tap), b1 = b2 + 512, b0 = b2 + 1024;
            const uint64_t a0 = desc_sw128(wa + s * 128), a1 = desc_sw128(wb2 + s * 128);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // a 32-byte K step adds 2 to a descriptor
              const uint64_t kb = 2 * kk;
              if (hp == 0) {
                mma_bf16_ss(d0, a0 + kb, b0 + kb, idesc, (s == 0 && kk == 0) ? 0u : 1u);  // row 0 += win0 W(0,s)
                if (s == 0 && kk == 0) {
                  mma_bf16_ss(d0, a1, b1, idesc, 1u);       // row 0 += win1 W(1,0)
                  mma_bf16_ss(d0 + 64, a1, b0, idesc, 0u);  // row 1 = win1 W(0,0): its first term
                } else {
                  mma_bf16_ss(d0, a1 + kb, b1 + kb, idesc2, 1u);  // rows 0|1 += win1 [W(1,s); W(0,s)]
                }
              } else {
                mma_bf16_ss(d0, a0 + kb, b2 + kb, idesc2, 1u);       // rows 0|1 += win2 [W(2,s); W(1,s)]
                mma_bf16_ss(d0 + 64, a1 + kb, b2 + kb, idesc, 1u);   // row 1 += win3 W(2,s)
              }
            }
          }
          mma_commit(&slot_empty[slot_a]);
          mma_commit(&slot_empty[slot_b]);
        }
        mma_commit(&acc2_full[b]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue group
    // warps 2 .. 1 + 4 kSubs: quad = TMEM lane quadrant (warp % 4), sub =
    // which windows (im2col, conv1_1 epilogue) or channels (pooled) it handles;
    // four warps per quadrant keep enough loads in flight (two left the MMA
    // waiting on the conv1_1 epilogue)
    const uint32_t quad = warp & 3;
    const int sub = (int(warp) - 2) >> 2;
    const uint32_t lane = lane_id();
    const int px = int(quad) * 32 + int(lane);  // window position / TMEM lane of this thread
    const int ep = int(threadIdx.x) - 64;
    const uint32_t lane_base = (quad * 32) << 16;
    if (ep < 64) b12[ep] = p.g[0].bias[ep];  // (conv1_1's bias rides in its weights)
    named_bar_sync(1, kEpi);
    // A: im2col of tile (t, it) into the SW64 im2col buffer (free once conv1_1
    // of the previous tile completed)
    auto im2col = [&](int t, int it) {
      int n, y0, x0;
      tile_of(p, t, n, y0, x0);
      mbar_wait(&patch_full[0], it & 1);
      const float* pp = patch;
      const int C = x0 + px - 1;  // image column of this window position
      // the patch starts at column (x0 - 2) & ~3: TMA needs 16-byte aligned inner coordinates
      const float* ppx = pp + px + ((x0 - 2) & 3);
      uint8_t* wrow = imc + px * 64;
#pragma unroll
      for (int jw = 0; jw < kWinPerSub; ++jw) {
        const int j = kWinPerSub * sub + jw;
        const int R = y0 - 1 + j;  // conv1_1 output row of window j
        float xs[32];
        xs[27] = xs[28] = 1.f;  // the bias taps
#pragma unroll
        for (int i = 29; i < 32; ++i) xs[i] = 0.f;
#pragma unroll
        for (int ci = 0; ci < 3; ++ci)
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            const int yy = R + r - 1;
            const bool rv = yy >= 0 && yy < p.H;
#pragma unroll
            for (int sx = 0; sx < 3; ++sx) {
              const int xx = C + sx - 1;
              const bool v = rv && xx >= 0 && xx < p.W;
              // patch row j + r = image row y0 - 2 + j + r; image col x0 - 2 + px + sx
              xs[ci * 9 + r * 3 + sx] = v ? ppx[(ci * kPatchRows + j + r) * kPatchCols + sx] - 0.5f : 0.f;
            }
          }
        uint32_t packed[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) packed[i] = pack2(xs[2 * i], xs[2 * i + 1]);
        uint8_t* row = wrow + j * 8192;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<uint4*>(row + ((q ^ ((px >> 1) & 3)) << 4)) =
              make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
      }
      fence_proxy_async_smem();
      mbar_arrive(&patch_empty[0]);
      mbar_arrive(imc_full);
    };
    // B: conv1_1 accumulators (bias included) -> ReLU, zero outside the image, bf16 ->
    // the tile's window buffer (conv1_2's A operand, SW128 K-major)
    auto act11 = [&](int t, int it) {
      int n, y0, x0;
      tile_of(p, t, n, y0, x0);
      const int b = it & 1;
      const int C = x0 + px - 1;
#pragma unroll
      for (int jw = 0; jw < kWinPerSub; ++jw) {
        const int j = kWinPerSub * sub + jw;
        // window j of this tile is use u of ring slot u % kWinSlots: wait
        // until conv1_2 released the slot's previous use
        const int u = 4 * it + j;
        const int slot = u % kWinSlots;
        mbar_wait(&slot_empty[slot], ((u / kWinSlots) & 1) ^ 1);
        uint8_t* row = win + slot * 16384 + px * 128;
        const int R = y0 - 1 + j;
        const bool valid = R >= 0 && R < p.H && C >= 0 && C < p.W;
        uint32_t va[32], vb[32];
        tmem_ld32(tmem + lane_base + j * 64, va);
        tmem_ld32(tmem + lane_base + j * 64 + 32, vb);
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          uint32_t w[4];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int c = q * 8 + 2 * jj;
            w[jj] = valid ? pack2_relu(__uint_as_float(q < 4 ? va[c & 31] : vb[c & 31]),
                                       __uint_as_float(q < 4 ? va[(c + 1) & 31] : vb[(c + 1) & 31]))
                          : 0u;
          }
          *reinterpret_cast<uint4*>(row + ((q ^ (px & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&win_full[b]);
    };
    // C: pooled conv1_2 epilogue of tile (t, it)
    auto pooled = [&](int t, int it) {
      int n, y0, x0;
      tile_of(p, t, n, y0, x0);
      const int b = it & 1;
      const uint32_t bph = (it >> 1) & 1;
      mbar_wait(&acc2_full[b], bph);
      tc_fence_after();
      const bool pvalid = px < kTileCols && x0 + px < p.W;
      const uint32_t tb0 = tmem + lane_base + kAcc2Col + b * 128;
      uint8_t* buf = stg + quad * 2048;
      if (sub == 0 && lane == 0) bulk_wait_read<0>();
      named_bar_sync(2 + quad, 32 * kSubs);  // the quad's previous store has read the staging box
      {
        constexpr int kH = kChPerSub / 2;
        const int cb = kChPerSub * sub;
        uint32_t va[kChPerSub], vb[kChPerSub];
        if constexpr (kChPerSub == 16) {
          tmem_ld16(tb0 + cb, va);
          tmem_ld16(tb0 + 64 + cb, vb);
        } else {
          tmem_ld32(tb0 + cb, va);
          tmem_ld32(tb0 + 64 + cb, vb);
        }
        tmem_ld_wait();
        // vertical max in registers; the horizontal pair (lanes 2i, 2i+1)
        // splits the channels: the even lane finishes the lower half, the odd the upper
        const bool odd = lane & 1;
        float m[kH];
#pragma unroll
        for (int k = 0; k < kH; ++k) {
          const float lo = fmaxf(__uint_as_float(va[k]), __uint_as_float(vb[k]));
          const float hi = fmaxf(__uint_as_float(va[kH + k]), __uint_as_float(vb[kH + k]));
          const float other = __shfl_xor_sync(0xffffffffu, odd ? lo : hi, 1);
          m[k] = fmaxf(odd ? hi : lo, other);
        }
        const int c0 = cb + (odd ? kH : 0);
        uint32_t w[kH / 2];
#pragma unroll
        for (int k = 0; k < kH / 2; ++k) {
          const float2 bias = *reinterpret_cast<const float2*>(b12 + c0 + 2 * k);
          w[k] = pvalid ? pack2_relu(m[2 * k] + bias.x, m[2 * k + 1] + bias.y) : 0u;
        }
        const uint32_t row = lane >> 1;
#pragma unroll
        for (int q = 0; q < kH / 8; ++q) {
          const uint32_t qq = c0 / 8 + q;
          *reinterpret_cast<uint4*>(buf + row * 128 + ((qq ^ (row & 7)) << 4)) =
              make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(&acc2_empty[b]);
      fence_proxy_async_smem();
      named_bar_sync(2 + quad, 32 * kSubs);
      if (sub == 0 && lane == 0) {
        // warp 3's 16th pooled column is the next tile's first: 15-column box
        tma_store_4d(quad == 3 ? &maps.out_pool[1] : &maps.out_pool[0], buf, p.g[0].out_c_off,
                     x0 / 2 + int(quad) * 16 + p.pool_P, y0 / 2 + p.pool_P, n);
        bulk_commit();
      }
    };
    const int g0 = blockIdx.x, gs = gridDim.x;
    if (g0 < p.total_tiles) im2col(g0, 0);
    int it = 0;
    for (int t = g0; t < p.total_tiles; t += gs, ++it) {
      mbar_wait(a1_full, it & 1);  // conv1_1(t) done: acc1 holds it, the im2col buffer is free
      tc_fence_after();
      if (t + gs < p.total_tiles) im2col(t + gs, it + 1);
      act11(t, it);
      if (it > 0) pooled(t - gs, it - 1);
    }
    if (it > 0) pooled(g0 + (it - 1) * gs, it - 1);
    if (sub == 0 && lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

}  // namespace

void conv12_configure() {
  check_cuda(cudaFuncSetAttribute(conv12_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem12::total + 1024),
             "conv12 smem attribute");
  check_cuda(cudaFuncSetAttribute(conv12_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem12::total + 1024),
             "conv12 smem attribute");
}

int conv12_tile_cols() { return kTileCols; }
int conv12_wgt_k() { return 64; }  // resident W(r,s) blocks: [64 cout][64 K] SW128

void launch_conv12(const ConvMaps& maps, const ConvParams& p, int sm_count, cudaStream_t stream) {
  const int grid = p.total_tiles < sm_count ? p.total_tiles : sm_count;
  static const int subs = [] {
    const char* e = std::getenv("AVEC_C12_SUBS");
    return e && e[0] == '4' ? 4 : 2;
  }();
  if (subs == 2)
    conv12_kernel<2><<<grid, C12Cfg<2>::kThreads, Smem12::total + 1024, stream>>>(maps, p);
  else
    conv12_kernel<4><<<grid, C12Cfg<4>::kThreads, Smem12::total + 1024, stream>>>(maps, p);
  check_cuda(cudaGetLastError(), "conv12 launch");
}

}  // namespace avec
