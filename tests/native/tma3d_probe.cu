// TMA probe for fp32 multi-plane patch loads (test program, not product code):
// loads one box of a [planes][H][W] fp32 tensor at (c0, c1, c2) into shared
// memory (SWIZZLE_NONE, zero fill outside the tensor) and compares it with the
// host's expectation. One configuration per process (a faulting TMA kills the
// context):  tma3d_probe W H planes box0 box1 box2 c0 c1 c2 dst_off
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2103_04930_b200/csrc/cuda/ptx.cuh"

using namespace avec::ptx;

#define CK(x)                                                                                               \
  do {                                                                                                      \
    cudaError_t e = (x);                                                                                    \
    if (e != cudaSuccess) {                                                                                 \
      std::printf("{\"ok\": false, \"error\": \"%s at line %d\"}\n", cudaGetErrorString(e), __LINE__);     \
      std::exit(1);                                                                                         \
    }                                                                                                       \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void probe(const __grid_constant__ CUtensorMap map, float* out, int n, int c0, int c1, int c2,
                      int dst_off, int bytes) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  float* dst = reinterpret_cast<float*>(smem + dst_off);
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, bytes);
    tma_load_3d(dst, &map, &bar, c0, c1, c2);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = dst[i];
}

int main(int argc, char** argv) {
  if (argc != 11) {
    std::printf("usage: W H planes box0 box1 box2 c0 c1 c2 dst_off\n");
    return 2;
  }
  int a[10];
  for (int i = 0; i < 10; ++i) a[i] = std::atoi(argv[i + 1]);
  const int W = a[0], H = a[1], P = a[2], b0 = a[3], b1 = a[4], b2 = a[5], c0 = a[6], c1 = a[7], c2 = a[8];
  const int dst_off = a[9];
  std::vector<float> h(size_t(W) * H * P);
  for (size_t i = 0; i < h.size(); ++i) h[i] = float(i % 100003) + 1.f;
  float *d, *o;
  CK(cudaMalloc(&d, h.size() * 4));
  CK(cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  const int n = b0 * b1 * b2;
  CK(cudaMalloc(&o, n * 4));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q));
  CUtensorMap m;
  cuuint64_t dims[3] = {cuuint64_t(W), cuuint64_t(H), cuuint64_t(P)};
  cuuint64_t strides[2] = {cuuint64_t(W) * 4, cuuint64_t(W) * H * 4};
  cuuint32_t box[3] = {cuuint32_t(b0), cuuint32_t(b1), cuuint32_t(b2)};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = reinterpret_cast<EncodeTiledFn>(fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es,
                                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::printf("{\"ok\": false, \"error\": \"encode %d\"}\n", int(r));
    return 1;
  }
  const int smem = 1024 + dst_off + n * 4;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe<<<1, 128, smem>>>(m, o, n, c0, c1, c2, dst_off, n * 4);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> got(n);
  CK(cudaMemcpy(got.data(), o, n * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int z = 0; z < b2; ++z)
    for (int y = 0; y < b1; ++y)
      for (int x = 0; x < b0; ++x) {
        const int X = c0 + x, Y = c1 + y, Z = c2 + z;
        const bool in = X >= 0 && X < W && Y >= 0 && Y < H && Z >= 0 && Z < P;
        const float want = in ? h[(size_t(Z) * H + Y) * W + X] : 0.f;
        bad += got[(size_t(z) * b1 + y) * b0 + x] != want;
      }
  std::printf("{\"ok\": %s, \"mismatches\": %d}\n", bad ? "false" : "true", bad);
  return bad ? 1 : 0;
}
