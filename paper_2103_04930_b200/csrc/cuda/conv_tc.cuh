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
// Wp-W columns per row that fall in the border are computed and discarded).
//
// GEMM mapping (swap-AB): M = 128 output channels (weights are operand A),
// N = 256 pixels per MMA (activations are operand B), K = 64 channels of one
// tap per k-block. A CTA tile is 128 Cout x 512 pixels (two N=256 MMAs that
// share every weight k-block); both accumulators fill the 512 TMEM columns.
//
// Activation reuse: for each (channel chunk, filter row r) the producer loads
// ONE window of 512 + k - 1 rows; the k taps s = 0..k-1 are MMA descriptors
// offset by s rows into that window (validated by tests/native/tc_probe.cu), so
// a 7x7 conv reads its input 7x, not 49x, from L2.
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 TMEM owner + MMA
// issuer, warps 2-5 epilogue (TMEM -> bias/ReLU -> bf16 NHWC or fp32 NCHW).
// Persistent: grid = min(tiles, SMs); tiles strided by gridDim.x.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace avec {

constexpr int kConvMaxGroups = 2;

struct ConvGroupParams {
  const float* bias;   // [m_tiles * 128], zero padded
  void* out;           // bf16 padded-flat NHWC buffer, or fp32 NCHW output
  int out_c_off;       // channel offset inside the destination
  int out_c_stride;    // channels of the destination buffer (NHWC) / total channels (NCHW)
  int cout;            // real output channels written
  int relu;
};

struct ConvParams {
  int k;               // filter size (1, 3, 7), stride 1, pad k/2
  int cin_chunks;      // input channels / 64 (padded)
  int in_c_off;        // first input channel inside the source buffer
  int n_images;
  int H, W;            // output = input spatial size
  int Hp, Wp, P;       // input buffer geometry
  int out_Hp, out_Wp, out_P;  // output buffer geometry (NHWC mode)
  int out_nchw_f32;    // 1: write fp32 NCHW [n][c][H][W] (final outputs)
  int m_tiles;         // ceil(cout / 128)
  int tiles_per_image; // ceil(H*Wp / 512)
  int n_groups;
  int total_tiles;
  ConvGroupParams g[kConvMaxGroups];
};

struct ConvMaps {
  CUtensorMap act_big[kConvMaxGroups];    // box {64 ch, 256 rows}
  CUtensorMap act_small[kConvMaxGroups];  // box {64 ch, 8 rows}
  CUtensorMap wgt[kConvMaxGroups];        // box {64, 128 rows}
};

// host side
size_t conv_smem_bytes();
// per device, before the first launch (sets the dynamic smem limit)
void conv_configure();
void launch_conv_tc(const ConvMaps& maps, const ConvParams& p, int sm_count, cudaStream_t stream);

}  // namespace avec
