// Pose-net post-processing: heatmap/PAF bilinear upsample and 3x3 peak NMS.
// Arithmetic uses explicit _rn intrinsics in the exact order of the CPU oracle
// (oracle/post_oracle.c, compiled with -ffp-contract=off): bit-exact parity.
#include <cstdint>

#include "engine.hpp"

namespace avec {

namespace {

__device__ __forceinline__ float src_coord(int o, int scale, int n, int& i0, int& i1) {
  float f = __fsub_rn(__fdiv_rn(__fadd_rn(static_cast<float>(o), 0.5f), static_cast<float>(scale)),
                      0.5f);
  if (f < 0.0f) f = 0.0f;
  int a = static_cast<int>(f);
  if (a > n - 1) a = n - 1;
  i0 = a;
  i1 = (a + 1 < n) ? a + 1 : n - 1;
  return __fsub_rn(f, static_cast<float>(a));
}

__device__ __forceinline__ float lerp2(float a, float b, float t) {
  return __fadd_rn(__fmul_rn(__fsub_rn(1.0f, t), a), __fmul_rn(t, b));
}

// one thread per 4 consecutive output pixels of a row (float4 store)
__global__ void upsample_kernel(const float* __restrict__ in, int planes, int h, int w, int scale,
                                float* __restrict__ out) {
  const int wo = w * scale, ho = h * scale;
  const int wq = wo / 4;
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long total = static_cast<long long>(planes) * ho * wq;
  if (idx >= total) return;
  const int q = static_cast<int>(idx % wq);
  long long rest = idx / wq;
  const int oy = static_cast<int>(rest % ho);
  const int pl = static_cast<int>(rest / ho);
  const float* src = in + static_cast<size_t>(pl) * h * w;
  int y0, y1;
  const float ly = src_coord(oy, scale, h, y0, y1);
  float r[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int x0, x1;
    const float lx = src_coord(q * 4 + j, scale, w, x0, x1);
    const float top = lerp2(__ldg(src + y0 * w + x0), __ldg(src + y0 * w + x1), lx);
    const float bot = lerp2(__ldg(src + y1 * w + x0), __ldg(src + y1 * w + x1), lx);
    r[j] = lerp2(top, bot, ly);
  }
  reinterpret_cast<float4*>(out + (static_cast<size_t>(pl) * ho + oy) * wo)[q] =
      make_float4(r[0], r[1], r[2], r[3]);
}

// Peak test for the pixel this lane owns in row y; neighbours come from the
// lanes on either side (warp shuffles) and rows y-1 / y+1 loaded per lane.
__device__ __forceinline__ bool lane_peak(const float* __restrict__ pl, int H, int W, int y, int x,
                                          float threshold, float& v) {
  const bool inb = x < W;
  const float NEG = -__int_as_float(0x7f800000);
  v = inb ? __ldg(pl + static_cast<size_t>(y) * W + x) : NEG;
  const float up = (inb && y > 0) ? __ldg(pl + static_cast<size_t>(y - 1) * W + x) : NEG;
  const float dn = (inb && y + 1 < H) ? __ldg(pl + static_cast<size_t>(y + 1) * W + x) : NEG;
  const int lane = threadIdx.x & 31;
  // left column (x-1): from lane-1, lane 0 loads it
  float lv = __shfl_up_sync(0xffffffffu, v, 1), lu = __shfl_up_sync(0xffffffffu, up, 1),
        ld = __shfl_up_sync(0xffffffffu, dn, 1);
  float rv = __shfl_down_sync(0xffffffffu, v, 1), ru = __shfl_down_sync(0xffffffffu, up, 1),
        rd = __shfl_down_sync(0xffffffffu, dn, 1);
  if (lane == 0) {
    const bool ok = inb && x > 0;
    lv = ok ? __ldg(pl + static_cast<size_t>(y) * W + x - 1) : NEG;
    lu = (ok && y > 0) ? __ldg(pl + static_cast<size_t>(y - 1) * W + x - 1) : NEG;
    ld = (ok && y + 1 < H) ? __ldg(pl + static_cast<size_t>(y + 1) * W + x - 1) : NEG;
  }
  if (lane == 31) {
    const bool ok = x + 1 < W;
    rv = ok ? __ldg(pl + static_cast<size_t>(y) * W + x + 1) : NEG;
    ru = (ok && y > 0) ? __ldg(pl + static_cast<size_t>(y - 1) * W + x + 1) : NEG;
    rd = (ok && y + 1 < H) ? __ldg(pl + static_cast<size_t>(y + 1) * W + x + 1) : NEG;
  }
  if (x + 1 >= W) rv = ru = rd = NEG;  // right neighbour outside the plane
  if (!inb || !(v > threshold)) return false;
  // out-of-plane neighbours are -inf, so "strictly greater" ignores them
  return v > lv && v > lu && v > ld && v > rv && v > ru && v > rd && v > up && v > dn;
}

// pass 1: per (plane, row) peak counts
__global__ void nms_count_kernel(const float* __restrict__ in, int H, int W, float threshold,
                                 int* __restrict__ row_counts) {
  const int y = blockIdx.x, pl = blockIdx.y;
  const float* p = in + static_cast<size_t>(pl) * H * W;
  __shared__ int warp_tot[32];
  int cnt = 0;
  const int span = (W + 31) / 32 * 32;
  for (int x = threadIdx.x; x < span; x += blockDim.x) {
    float v;
    const bool pk = lane_peak(p, H, W, y, x, threshold, v);
    cnt += __popc(__ballot_sync(0xffffffffu, pk));
  }
  if ((threadIdx.x & 31) == 0) warp_tot[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += warp_tot[i];
    row_counts[static_cast<size_t>(pl) * H + y] = t;
  }
}

// pass 2: per-plane exclusive scan of the row counts (one block per plane)
__global__ void nms_scan_kernel(const int* __restrict__ row_counts, int H, int max_peaks,
                                int* __restrict__ row_offsets, int* __restrict__ counts) {
  const int pl = blockIdx.x;
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int y = 0; y < H; ++y) {
      row_offsets[static_cast<size_t>(pl) * H + y] = acc;
      acc += row_counts[static_cast<size_t>(pl) * H + y];
    }
    counts[pl] = acc < max_peaks ? acc : max_peaks;
  }
}

// pass 3: write peaks in raster order (row offset + rank inside the row)
__global__ void nms_write_kernel(const float* __restrict__ in, int H, int W, float threshold,
                                 int max_peaks, const int* __restrict__ row_offsets,
                                 float* __restrict__ peaks) {
  const int y = blockIdx.x, pl = blockIdx.y;
  const float* p = in + static_cast<size_t>(pl) * H * W;
  int base = row_offsets[static_cast<size_t>(pl) * H + y];
  if (base >= max_peaks) return;
  __shared__ int warp_cnt[32];
  const int span = (W + 31) / 32 * 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int x0 = 0; x0 < span; x0 += blockDim.x) {
    const int x = x0 + threadIdx.x;
    float v = 0.f;
    const bool pk = (x < span) ? lane_peak(p, H, W, y, x, threshold, v) : false;
    const unsigned m = __ballot_sync(0xffffffffu, pk);
    if (lane == 0) warp_cnt[wid] = __popc(m);
    __syncthreads();
    int before = 0, total = 0;
    for (int i = 0; i < nw; ++i) {
      if (i < wid) before += warp_cnt[i];
      total += warp_cnt[i];
    }
    if (pk) {
      const int idx = base + before + __popc(m & ((1u << lane) - 1u));
      if (idx < max_peaks) {
        float sw = 0.0f, sx = 0.0f, sy = 0.0f;
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const int yy = y + dy, xx = x + dx;
            if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
            const float s = __ldg(p + static_cast<size_t>(yy) * W + xx);
            sw = __fadd_rn(sw, s);
            sx = __fadd_rn(sx, __fmul_rn(static_cast<float>(xx), s));
            sy = __fadd_rn(sy, __fmul_rn(static_cast<float>(yy), s));
          }
        float* o = peaks + (static_cast<size_t>(pl) * max_peaks + idx) * 5;
        o[0] = static_cast<float>(x);
        o[1] = static_cast<float>(y);
        o[2] = __fdiv_rn(sx, sw);
        o[3] = __fdiv_rn(sy, sw);
        o[4] = v;
      }
    }
    base += total;
    __syncthreads();
    if (base >= max_peaks) return;
  }
}

}  // namespace

void launch_upsample(const float* d_in, int planes, int h, int w, int scale, float* d_out,
                     cudaStream_t stream) {
  if ((w * scale) % 4 != 0) fail(AVEC_ERR_UNSUPPORTED, "upsample needs output width % 4 == 0");
  const long long total = static_cast<long long>(planes) * h * scale * (w * scale / 4);
  upsample_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream>>>(
      d_in, planes, h, w, scale, d_out);
  check_cuda(cudaGetLastError(), "upsample launch");
}

size_t nms_scratch_bytes(int planes, int H, int /*W*/) {
  return 2 * static_cast<size_t>(planes) * H * sizeof(int);
}

void launch_nms(const float* d_in, int planes, int H, int W, float threshold, int max_peaks,
                int* d_counts, float* d_peaks, void* d_scratch, size_t scratch_bytes,
                cudaStream_t stream) {
  if (scratch_bytes < nms_scratch_bytes(planes, H, W)) fail(AVEC_ERR_INVALID_ARGUMENT, "nms scratch");
  if (H > 65535 || planes > 65535) fail(AVEC_ERR_UNSUPPORTED, "nms grid limits");
  int* row_counts = static_cast<int*>(d_scratch);
  int* row_offsets = row_counts + static_cast<size_t>(planes) * H;
  dim3 grid(H, planes);
  nms_count_kernel<<<grid, 256, 0, stream>>>(d_in, H, W, threshold, row_counts);
  nms_scan_kernel<<<planes, 32, 0, stream>>>(row_counts, H, max_peaks, row_offsets, d_counts);
  nms_write_kernel<<<grid, 256, 0, stream>>>(d_in, H, W, threshold, max_peaks, row_offsets,
                                              d_peaks);
  check_cuda(cudaGetLastError(), "nms launch");
}

}  // namespace avec
