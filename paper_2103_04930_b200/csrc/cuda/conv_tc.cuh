// Implicit-GEMM convolution on tcgen05 (sm_100a), the pose network's hot op.
//
// Layout ("padded-flat NHWC"): every activation tensor of one pyramid level is
// a bf16 buffer [N][Hp][Wp][C] with a zero border of P pixels (Hp = H + 2P,
// Wp = W + 2P) and C a multiple of 64. Flattening (h, w) of image n over the
// padded width turns every filter tap (r, s) of a stride-1 "same" convolution
// into a constant row shift r*Wp + s of the same 2D [rows][C] matrix, so:
//
//   out[o][co] = sum_{r,s,ci} act[base_n + o + r*Wp + s][ci] * W[co][r][s][ci]
//
// for o over the image's output positions laid out on the padded width (the
// Wp-W columns per row that fall in the border are computed, then written as
// ZERO, which keeps the output's border valid padding for the next layer).
//
// GEMM mapping (swap-AB): M = 128 output channels (weights are operand A),
// N = 256 pixels per MMA (activations are operand B; N=256 keeps the SS-mode
// smem operand traffic under the measured 128 B/clk, see tests/native/tc_probe.cu),
// K = 64 channels of one tap per k-block.
//
// Two tile shapes (template SUBS):
//  * SUBS = 2: 128 Cout x 512 pixels; both N=256 MMAs share every weight
//    k-block (halves L2 weight traffic); accumulators fill all 512 TMEM
//    columns. Used for large-K layers (7x7 stages) where the mainloop dwarfs
//    the epilogue.
//  * SUBS = 1: 128 x 256 with TWO accumulator stages in TMEM, so the epilogue
//    of tile i overlaps the mainloop of tile i+1. Only reachable through the
//    AVEC_TC3 experiment (3x3 layers on this kernel); the short-K layers run
//    on the pixel-major kernel (conv_pm.cu).
//
// Activation reuse: for each (channel chunk, filter row r) the producer loads
// ONE window of 256*SUBS + 8 rows; the k taps s = 0..k-1 are MMA descriptors
// offset by s rows into that window (the hardware swizzles on absolute smem
// address bits, validated by tests/native/tc_probe.cu), so a 7x7 conv reads
// its input 7x, not 49x, from L2.
//
// Epilogue: TMEM -> registers (bias, ReLU/PReLU, zero outside the image, bf16) ->
// 128B-swizzled smem staging -> TMA bulk-tensor store of [32 px][64 ch] boxes
// into the output's 3D view [N][Hp*Wp][C] (rows past the image are clipped by
// the tensor bounds). Outputs that are not 64-channel slabs (the 38/19-channel
// branch heads) and the fp32 NCHW network output use a direct-store path.
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 TMEM owner + MMA
// issuer, warps 2-5 epilogue. Persistent: grid = min(tiles, SMs).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace avec {

constexpr int kConvMaxGroups = 2;

enum ConvOutMode : int {
  kOutTmaBf16 = 0,   // bf16 padded-flat NHWC via TMA store (64-channel slabs)
  kOutDirectBf16 = 1,  // bf16 padded-flat NHWC, per-element stores
  kOutNchwF32 = 2,   // fp32 NCHW [n][c][H][W] (network output)
};

struct ConvGroupParams {
  const float* bias;   // [m_tiles * 128], zero padded
  void* out;           // destination base
  int out_c_off;       // channel offset inside the destination
  int out_c_stride;    // channels of the destination buffer (NHWC) / total channels (NCHW)
  int cout;            // real output channels written
  int act;             // 0 none, 1 ReLU, 2 PReLU (pixel-major kernel only)
  const float* slope;  // PReLU slopes [m_tiles * 128]
};

struct ConvParams {
  int k;               // filter size (1, 3, 7), stride 1, pad k/2
  int cin_chunks;      // input channels / 64 (padded)
  int k16_last;        // pixel-major: 16-channel K steps with nonzero weights in the last chunk (1..4)
  int in_c_off;        // first input channel inside the source buffer
  int n_images;
  int H, W;            // output = input spatial size
  int Hp, Wp, P;       // buffer geometry (input and output share it)
  int out_mode;        // ConvOutMode
  int subs;            // swap-AB: 1 or 2 (tile width 256 * subs pixels)
  int pixel_major;     // 1: conv_pm.cu orientation (M = pixels, N = pm_n channels)
  int pm_n;            // pixel-major channel tile: 64, 96, 128 or 256
  int ncta;            // pixel-major: 1, or 2 = CTA pair (cta_group::2, M = 256 pixels per MMA)
  // pixel-major with a fused 2x2/2 max-pool: tiles are [2 rows x 128 columns]
  // per CTA (sub-tile = row), the epilogue writes the pooled row through
  // maps.out_pool into the next level's buffer (padding pool_P)
  int pool;
  int pool_P;
  int col_blocks;      // pool: ceil(W / 128)
  int m_tiles;         // channel tiles: ceil(cout / 128), or ceil(cout / pm_n)
  int tiles_per_image; // ceil(H*Wp / pixels per tile)
  int tile_px;         // swap-AB regular tiles: pixels per tile (<= 256 * subs, multiple of 32)
  int n_groups;
  int total_tiles;
  // swap-AB balanced partition (0 = regular tiles): 32-position units over the
  // n_groups * n_images segments of units_per_seg units each
  int balanced_units;
  int units_per_seg;
  // swap-AB split-K (small grids: C1, frame groups): each tile's window
  // iterations (cin_chunks * k of them) are cut into `splits` contiguous ranges
  // computed by different CTAs; they store raw fp32 partials to `ws`
  // ([tile][split][tile_px][128]) and conv_tc_reduce_kernel sums them in split
  // order (deterministic) and applies the epilogue. 1 = off.
  int splits;
  int tf32;            // conv_first: tf32 operands (kind::tf32) instead of bf16
  float* ws;
  ConvGroupParams g[kConvMaxGroups];
};

struct ConvMaps {
  CUtensorMap act_big[kConvMaxGroups];    // 2D [rows][C_in], box {64 ch, 256 rows}
  CUtensorMap act_small[kConvMaxGroups];  // 2D, box {64 ch, 8 rows}
  CUtensorMap act_mid[kConvMaxGroups];    // 2D, box {64 ch, 128 rows}
  CUtensorMap wgt[kConvMaxGroups];        // 2D [cout_pad][k*k*cin_pad], box {64, 128 (or pm_n) rows}
  CUtensorMap out[kConvMaxGroups];        // 3D [N][Hp*Wp][C_out], box {64 ch, 32 rows, 1}, SW128
  // narrower boxes of the same view for the pixel-major kernel's channel tails
  // (96-wide layers, 52/38/26/19-channel heads): 32 ch SW64, 16 ch SW32, 8 ch
  CUtensorMap out32[kConvMaxGroups];
  CUtensorMap out16[kConvMaxGroups];
  CUtensorMap out8[kConvMaxGroups];
  CUtensorMap out_pool[kConvMaxGroups];   // 4D [N][Hp'][Wp'][C] of the pooled level, box {64, 16, 1, 1}
};

// Fused stage head (conv_head.cu): Mconv6 (1x1 -> c6, act6) then Mconv7
// (1x1 -> c7 <= 64, no activation) per 128-pixel tile, c6 in NB-wide blocks.
struct HeadGroup {
  const float* bias6;
  const float* slope6;
  int act6;
  const float* bias7;
  int c7;
  void* out;            // bf16 padded-flat slab (kOutTmaBf16) or fp32 NCHW (kOutNchwF32)
  int out_mode;
  int out_c_off, out_c_stride;
  float* out2;          // optional second destination: fp32 NCHW (BODY_25's last PAF stage)
  int out2_c_off, out2_c_stride;
};

struct HeadParams {
  int n_images, H, W, Hp, Wp, P;
  int in_c_off, cin_chunks;
  int nb, blocks;       // c6 = nb * blocks, nb = 128
  int tiles_per_image, total_tiles, n_groups;  // ncta == 2: tiles = pairs of 128-pixel tiles
  int ncta;                                     // 1, or 2 for the CTA-pair kernel (conv_head2)
  HeadGroup g[kConvMaxGroups];
};

struct HeadMaps {
  CUtensorMap x[kConvMaxGroups];    // input, box {64 ch, 128 rows}
  CUtensorMap w6[kConvMaxGroups];   // [c6_pad][cin_pad], box {64, 128 rows}
  CUtensorMap w7[kConvMaxGroups];   // [c7_pad][c6], box {64, 64 rows}
  CUtensorMap out32[kConvMaxGroups], out16[kConvMaxGroups], out8[kConvMaxGroups];
};

// host side
// per device, before the first launch (sets the dynamic smem limits)
void conv_configure();
void launch_conv_tc(const ConvMaps& maps, const ConvParams& p, int sm_count, cudaStream_t stream);
// split-K count for a swap-AB launch of `tiles` tiles with `windows` window
// iterations each on `sm_count` SMs (1 = no split; AVEC_SPLITK=0 disables)
int conv_tc_splits(int tiles, int windows, int sm_count);
// pixel-major variant (conv_pm.cu)
void conv_pm_configure();
int conv_pm_subs(int n_tile);   // 128-pixel M sub-tiles per tile for a channel tile
int conv_pm_tile_n(int cout);   // channel tile (MMA N) for a layer's output width
void launch_conv_pm(const ConvMaps& maps, const ConvParams& p, int sm_count, cudaStream_t stream);
// first layer fused with the input conversion (conv_first.cu): fp32 NCHW frames
// -> 3x3x3 taps built in smem -> tcgen05 -> 64-channel padded-flat NHWC output
void conv_first_configure();
void conv_head_configure();
int conv_head_pair_max_chunks();  // input chunks the pair head keeps resident
// conv1_1 + conv1_2 + pool1 (conv12.cu)
void conv12_configure();
int conv12_tile_cols();
int conv12_wgt_k();  // K columns per conv1_2 weight box (the stage's swizzle span / 2)
void launch_conv12(const ConvMaps& maps, const ConvParams& p, int sm_count, cudaStream_t stream);
void launch_conv_head(const HeadMaps& maps, const HeadParams& p, int sm_count, cudaStream_t stream);
void launch_conv_first(const ConvMaps& maps, const ConvParams& p, const float* frames, int sm_count,
                       cudaStream_t stream);

}  // namespace avec
