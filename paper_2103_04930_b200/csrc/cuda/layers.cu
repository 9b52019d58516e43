// Streaming layers of the pose net: input conversion fused with the first
// (3-channel) convolution, 2x2 max-pool, and an unpad/convert helper.
// All are HBM-bound; loads/stores are 16-byte vectors over channels.
#include <cuda_bf16.h>

#include "engine.hpp"

namespace avec {

namespace {

// conv1_1 has 3 input channels (K = 27), too thin to feed the tensor cores
// directly. This streaming kernel fuses the wire-format conversion with an
// im2col: fp32 NCHW frame -> (x - 0.5) -> bf16 (the net's input precision) ->
// one 64-channel row per pixel holding the 27 taps (ci*9 + r*3 + s) and 37
// zeros, in the level-0 padded-flat layout. conv1_1 then runs as a 1x1
// tcgen05 conv over those 64 channels (weights packed to match).
// HBM-bound: 12 B read + 128 B written per pixel.
__global__ void __launch_bounds__(128) im2col_first_kernel(const float* __restrict__ in, int n,
                                                           int H, int W,
                                                           __nv_bfloat16* __restrict__ out, int P) {
  const long long pix = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long total = static_cast<long long>(n) * H * W;
  if (pix >= total) return;
  const int x = static_cast<int>(pix % W);
  const int y = static_cast<int>((pix / W) % H);
  const int b = static_cast<int>(pix / (static_cast<long long>(W) * H));
  uint32_t packed[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) packed[i] = 0;
#pragma unroll
  for (int ci = 0; ci < 3; ++ci) {
    const float* plane = in + (static_cast<size_t>(b) * 3 + ci) * H * W;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int yy = y + r - 1, xx = x + s - 1;
        float v = 0.f;
        if (yy >= 0 && yy < H && xx >= 0 && xx < W) v = __ldg(plane + yy * W + xx) - 0.5f;
        const int t = ci * 9 + r * 3 + s;
        const uint32_t bits = __bfloat16_as_ushort(__float2bfloat16_rn(v));
        packed[t >> 1] |= (t & 1) ? (bits << 16) : bits;
      }
    }
  }
  uint4* dst = reinterpret_cast<uint4*>(
      out + ((static_cast<size_t>(b) * (H + 2 * P) + y + P) * (W + 2 * P) + x + P) * 64);
#pragma unroll
  for (int q = 0; q < 8; ++q)
    dst[q] = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
}

__global__ void maxpool2_kernel(const __nv_bfloat16* __restrict__ in, int n, int H, int W,
                                int P_in, int C, __nv_bfloat16* __restrict__ out, int P_out) {
  const int Ho = H / 2, Wo = W / 2, C8 = C / 8;
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long total = static_cast<long long>(n) * Ho * Wo * C8;
  if (idx >= total) return;
  const int c8 = static_cast<int>(idx % C8);
  long long rest = idx / C8;
  const int xo = static_cast<int>(rest % Wo);
  rest /= Wo;
  const int yo = static_cast<int>(rest % Ho);
  const int b = static_cast<int>(rest / Ho);
  const int Wp_in = W + 2 * P_in, Hp_in = H + 2 * P_in;
  const size_t row = (static_cast<size_t>(b) * Hp_in + 2 * yo + P_in) * Wp_in + 2 * xo + P_in;
  const uint4* p = reinterpret_cast<const uint4*>(in + row * C) + c8;
  const size_t step = static_cast<size_t>(C) / 8;
  uint4 a = __ldg(p), bb = __ldg(p + step), c = __ldg(p + Wp_in * step),
        d = __ldg(p + (Wp_in + 1) * step);
  uint4 r;
  const __nv_bfloat162* A = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* B = reinterpret_cast<const __nv_bfloat162*>(&bb);
  const __nv_bfloat162* Cc = reinterpret_cast<const __nv_bfloat162*>(&c);
  const __nv_bfloat162* D = reinterpret_cast<const __nv_bfloat162*>(&d);
  __nv_bfloat162* R = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
  for (int j = 0; j < 4; ++j) R[j] = __hmax2(__hmax2(A[j], B[j]), __hmax2(Cc[j], D[j]));
  const int Wp_out = Wo + 2 * P_out, Hp_out = Ho + 2 * P_out;
  const size_t orow = (static_cast<size_t>(b) * Hp_out + yo + P_out) * Wp_out + xo + P_out;
  reinterpret_cast<uint4*>(out + orow * C)[c8] = r;
}

__global__ void unpad_kernel(const __nv_bfloat16* __restrict__ in, int n, int H, int W, int P,
                             int C_stride, int c_off, int c, float* __restrict__ out) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long total = static_cast<long long>(n) * H * W * c;
  if (idx >= total) return;
  const int ch = static_cast<int>(idx % c);
  long long rest = idx / c;
  const int x = static_cast<int>(rest % W);
  rest /= W;
  const int y = static_cast<int>(rest % H);
  const int b = static_cast<int>(rest / H);
  const size_t row = (static_cast<size_t>(b) * (H + 2 * P) + y + P) * (W + 2 * P) + x + P;
  out[idx] = __bfloat162float(in[row * C_stride + c_off + ch]);
}

unsigned blocks_for(long long total, int threads) {
  return static_cast<unsigned>((total + threads - 1) / threads);
}

}  // namespace

void launch_im2col_first(const float* d_in, int n, int H, int W, void* d_out, int P,
                         cudaStream_t stream) {
  const long long total = static_cast<long long>(n) * H * W;
  im2col_first_kernel<<<blocks_for(total, 128), 128, 0, stream>>>(
      d_in, n, H, W, static_cast<__nv_bfloat16*>(d_out), P);
  check_cuda(cudaGetLastError(), "im2col_first launch");
}

void launch_maxpool2(const void* d_in, int n, int H, int W, int P_in, int C, void* d_out,
                     int P_out, cudaStream_t stream) {
  const long long total = static_cast<long long>(n) * (H / 2) * (W / 2) * (C / 8);
  maxpool2_kernel<<<blocks_for(total, 256), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(d_in), n, H, W, P_in, C,
      static_cast<__nv_bfloat16*>(d_out), P_out);
  check_cuda(cudaGetLastError(), "maxpool launch");
}

void launch_unpad_to_f32(const void* d_in, int n, int H, int W, int P, int C_stride, int c_off,
                         int c, float* d_out, cudaStream_t stream) {
  const long long total = static_cast<long long>(n) * H * W * c;
  unpad_kernel<<<blocks_for(total, 256), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(d_in), n, H, W, P, C_stride, c_off, c, d_out);
  check_cuda(cudaGetLastError(), "unpad launch");
}

}  // namespace avec
