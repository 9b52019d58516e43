// Streaming layers of the pose net: 2x2 max-pool and an unpad/convert helper
// (the input conversion is fused into the first convolution, conv_first.cu).
// All are HBM-bound; loads/stores are 16-byte vectors over channels.
#include <cuda_bf16.h>

#include "engine.hpp"

namespace avec {

namespace {

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
