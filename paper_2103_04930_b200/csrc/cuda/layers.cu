// Streaming layers of the pose net: input conversion fused with the first
// (3-channel) convolution, 2x2 max-pool, and an unpad/convert helper.
// All are HBM-bound; loads/stores are 16-byte vectors over channels.
#include <cuda_bf16.h>

#include "engine.hpp"

namespace avec {

namespace {

// conv1_1: 3 input channels make a K=27 GEMM — too thin for the tensor cores,
// so it runs on the FP32 pipes, fused with the wire-format conversion:
// fp32 NCHW frame -> (x - 0.5) -> bf16 (the net's input precision) -> 3x3 conv
// -> +bias -> ReLU -> bf16 NHWC (64 ch, one 128-byte row per pixel).
__global__ void __launch_bounds__(128) conv_first_kernel(const float* __restrict__ in, int n,
                                                         int H, int W,
                                                         const float* __restrict__ w27x64,
                                                         const float* __restrict__ bias,
                                                         __nv_bfloat16* __restrict__ out, int P) {
  __shared__ float sw[27 * 64];
  __shared__ float sb[64];
  for (int i = threadIdx.x; i < 27 * 64; i += blockDim.x) sw[i] = w27x64[i];
  if (threadIdx.x < 64) sb[threadIdx.x] = bias[threadIdx.x];
  __syncthreads();
  const long long pix = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long total = static_cast<long long>(n) * H * W;
  if (pix >= total) return;
  const int x = static_cast<int>(pix % W);
  const int y = static_cast<int>((pix / W) % H);
  const int b = static_cast<int>(pix / (static_cast<long long>(W) * H));
  float xin[27];
#pragma unroll
  for (int ci = 0; ci < 3; ++ci) {
    const float* plane = in + (static_cast<size_t>(b) * 3 + ci) * H * W;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int yy = y + r - 1, xx = x + s - 1;
        float v = 0.f;
        if (yy >= 0 && yy < H && xx >= 0 && xx < W)
          v = __bfloat162float(__float2bfloat16_rn(__ldg(plane + yy * W + xx) - 0.5f));
        xin[ci * 9 + r * 3 + s] = v;
      }
    }
  }
  __nv_bfloat16* dst =
      out + ((static_cast<size_t>(b) * (H + 2 * P) + y + P) * (W + 2 * P) + x + P) * 64;
#pragma unroll
  for (int c8 = 0; c8 < 8; ++c8) {
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
#pragma unroll
    for (int t = 0; t < 27; ++t) {
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = fmaf(xin[t], sw[t * 64 + c8 * 8 + j], acc[j]);
    }
    uint32_t packed[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float a = fmaxf(acc[2 * j] + sb[c8 * 8 + 2 * j], 0.f);
      float c = fmaxf(acc[2 * j + 1] + sb[c8 * 8 + 2 * j + 1], 0.f);
      __nv_bfloat162 h2 = __floats2bfloat162_rn(a, c);
      packed[j] = *reinterpret_cast<uint32_t*>(&h2);
    }
    reinterpret_cast<uint4*>(dst)[c8] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
  }
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

void launch_conv_first(const float* d_in, int n, int H, int W, const float* w_fp32_27x64,
                       const float* bias64, void* d_out, int P, cudaStream_t stream) {
  const long long total = static_cast<long long>(n) * H * W;
  conv_first_kernel<<<blocks_for(total, 128), 128, 0, stream>>>(
      d_in, n, H, W, w_fp32_27x64, bias64, static_cast<__nv_bfloat16*>(d_out), P);
  check_cuda(cudaGetLastError(), "conv_first launch");
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
