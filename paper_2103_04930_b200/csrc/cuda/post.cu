// Pose-net post-processing: heatmap/PAF bilinear upsample and 3x3 peak NMS.
// Arithmetic uses explicit _rn intrinsics in the exact order of the CPU oracle
// (oracle/post_oracle.c, compiled with -ffp-contract=off): bit-exact parity.
#include <algorithm>
#include <cstdint>

#include <cstdlib>

#include "engine.hpp"
#include "ptx.cuh"

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

// Power-of-two scales (the pose net's x8): (o + 0.5) / scale is exact as a
// multiply by 1/scale, so the coordinates match src_coord bit for bit without
// the division.
__device__ __forceinline__ float src_coord_pow2(int o, float inv_scale, int n, int& i0, int& i1) {
  float f = __fsub_rn(__fmul_rn(__fadd_rn(static_cast<float>(o), 0.5f), inv_scale), 0.5f);
  if (f < 0.0f) f = 0.0f;
  int a = static_cast<int>(f);
  if (a > n - 1) a = n - 1;
  i0 = a;
  i1 = (a + 1 < n) ? a + 1 : n - 1;
  return __fsub_rn(f, static_cast<float>(a));
}

// x8 upsample. Interior 8-output groups (1 <= g < w - 1): outputs 8g+j sit
// at f = g - 1 + (j + 4.5) / 8 (j < 4: between source columns g-1, g; j >= 4:
// between g, g+1). Every step of src_coord is exact in fp32 there, so lx is
// the constant (j + 4.5) / 8 mod 1 and the result equals the general
// kernel's bit for bit; the groups at the row ends (clamped columns) take the
// general coordinates in the block's last warp.
// A thread computes one float4 of outputs (4 columns: they all lie between
// the same two source columns) for the 4 output rows of a quad (oy = 4q ..
// 4q+3 share one pair of source rows: rows 8k..8k+3 sit between source rows
// k-1 and k, rows 8k+4..8k+7 between k and k+1, clamped alike at the
// borders). The 4 source values and 8 horizontal lerps are done once per
// quad, the vertical lerp per row, with the same op sequence per output as
// the general kernel (bit for bit). Consecutive lanes store consecutive 16-byte
// chunks, so each store instruction writes whole sectors: the previous
// 8-columns-per-thread layout wrote 32-byte strided halves and moved twice the
// bytes through L1 -> L2 (the write path at 83%; with a separate row-end
// kernel 106 + 10 us at C2, now 79 us).
__global__ void upsample8_kernel(const float* __restrict__ in, int h, int w, float* __restrict__ out) {
  const int wo = w * 8, ho = h * 8;
  const int n_in = 2 * (w - 2);  // interior float4s per output row (threads 0 .. n_in-1)
  const int oy0 = blockIdx.y * 4;
  const int pl = blockIdx.z;
  const float* src = in + static_cast<size_t>(pl) * h * w;
  const int tid = threadIdx.x;
  if (tid >= blockDim.x - 32) {
    // the block's last warp: the row ends (the 8-output groups 0 and w-1,
    // clamped source columns) of its 4 rows on the general per-column
    // coordinates, one float4 of one row per lane, so no interior warp waits
    const int l = tid - (blockDim.x - 32);
    if (l >= 16) return;
    const int oy = oy0 + (l >> 2), k = l & 3;
    const int f = k < 2 ? k : 2 * w - 4 + k;
    int y0, y1;
    const float ly = src_coord_pow2(oy, 0.125f, h, y0, y1);
    const float* r0 = src + static_cast<size_t>(y0) * w;
    const float* r1 = src + static_cast<size_t>(y1) * w;
    float r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int x0, x1;
      const float lx = src_coord_pow2(4 * f + j, 0.125f, w, x0, x1);
      r[j] = lerp2(lerp2(__ldg(r0 + x0), __ldg(r0 + x1), lx), lerp2(__ldg(r1 + x0), __ldg(r1 + x1), lx), ly);
    }
    reinterpret_cast<float4*>(out + (static_cast<size_t>(pl) * ho + oy) * wo)[f] = make_float4(r[0], r[1], r[2], r[3]);
    return;
  }
  if (tid >= n_in) return;
  const int f = 2 + tid;  // float4 index of the output row
  const int g = f >> 1, half = f & 1;
  constexpr float kLx[8] = {0.5625f, 0.6875f, 0.8125f, 0.9375f, 0.0625f, 0.1875f, 0.3125f, 0.4375f};
  const int c = g - 1 + half;  // left source column of these 4 outputs
  int py0 = -1, py1 = -1;
  float top[4], bot[4];
#pragma unroll
  for (int dy = 0; dy < 4; ++dy) {
    const int oy = oy0 + dy;
    int y0, y1;
    const float ly = src_coord_pow2(oy, 0.125f, h, y0, y1);
    if (y0 != py0 || y1 != py1) {  // once per quad (the rows share their source rows)
      const float* r0 = src + static_cast<size_t>(y0) * w + c;
      const float* r1 = src + static_cast<size_t>(y1) * w + c;
      const float a0 = __ldg(r0), a1 = __ldg(r0 + 1);
      const float b0 = __ldg(r1), b1 = __ldg(r1 + 1);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float lx = kLx[half * 4 + j];
        top[j] = lerp2(a0, a1, lx);
        bot[j] = lerp2(b0, b1, lx);
      }
      py0 = y0;
      py1 = y1;
    }
    reinterpret_cast<float4*>(out + (static_cast<size_t>(pl) * ho + oy) * wo)[f] =
        make_float4(lerp2(top[0], bot[0], ly), lerp2(top[1], bot[1], ly), lerp2(top[2], bot[2], ly),
                    lerp2(top[3], bot[3], ly));
  }
}

// one 8-output group: the general path of the pow2 kernels
__device__ __forceinline__ void upsample_group(const float* __restrict__ in, int h, int w, int scale, float inv_scale,
                                               float* __restrict__ out, int pl, int oy, int g) {
  const int wo = w * scale, ho = h * scale;
  const float* src = in + static_cast<size_t>(pl) * h * w;
  int y0, y1;
  const float ly = src_coord_pow2(oy, inv_scale, h, y0, y1);
  int c0, c0b;
  src_coord_pow2(g * 8, inv_scale, w, c0, c0b);  // first output's left source column
  const int c1 = c0 + 1 < w ? c0 + 1 : w - 1, c2 = c0 + 2 < w ? c0 + 2 : w - 1;
  const float* r0 = src + static_cast<size_t>(y0) * w;
  const float* r1 = src + static_cast<size_t>(y1) * w;
  const float a0 = __ldg(r0 + c0), a1 = __ldg(r0 + c1), a2 = __ldg(r0 + c2);
  const float b0 = __ldg(r1 + c0), b1 = __ldg(r1 + c1), b2 = __ldg(r1 + c2);
  float r[8];
  float4* o4 = reinterpret_cast<float4*>(out + (static_cast<size_t>(pl) * ho + oy) * wo) + 2 * g;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    int x0, x1;
    const float lx = src_coord_pow2(g * 8 + j, inv_scale, w, x0, x1);
    // x0 - c0 and x1 - c0 are in {0, 1, 2} (clamped columns alias)
    const int d0 = x0 - c0, d1 = x1 - c0;
    const float ta = d0 == 0 ? a0 : d0 == 1 ? a1 : a2, tb = d1 == 0 ? a0 : d1 == 1 ? a1 : a2;
    const float ba = d0 == 0 ? b0 : d0 == 1 ? b1 : b2, bb = d1 == 0 ? b0 : d1 == 1 ? b1 : b2;
    const float top = lerp2(ta, tb, lx);
    const float bot = lerp2(ba, bb, lx);
    r[j] = lerp2(top, bot, ly);
  }
  o4[0] = make_float4(r[0], r[1], r[2], r[3]);
  o4[1] = make_float4(r[4], r[5], r[6], r[7]);
}

// grid (column groups, output rows, planes): no integer division per thread
__global__ void upsample_pow2_kernel(const float* __restrict__ in, int planes, int h, int w, int scale,
                                     float inv_scale, float* __restrict__ out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= w * scale / 8) return;
  upsample_group(in, h, w, scale, inv_scale, out, blockIdx.z, blockIdx.y, g);
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

// ---- tiled variant (W % 4 == 0): a block stages rows y0-1 .. y0+R of one
// plane in shared memory with coalesced float4 loads (many in flight), then
// each thread tests four columns per row from the tile. Rows and columns
// outside the plane read as -inf, so "strictly greater" ignores them.
constexpr int kNmsRows = 8;      // two-pass kernels
constexpr int kNmsRows1 = 8;     // one-pass tiles (16 measured slower: 119 vs 100 us; masks hold <= 16 rows)

__device__ __forceinline__ void nms_stage_tile(float* tile, const float* __restrict__ p, int H, int W, int y0,
                                               int rows) {
  const float NEG = -__int_as_float(0x7f800000);
  const int W4 = W >> 2;
  const int n = (rows + 2) * W4;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int rr = i / W4, c4 = i - rr * W4;
    const int y = y0 - 1 + rr;
    const float4 v = (y >= 0 && y < H) ? __ldg(reinterpret_cast<const float4*>(p + static_cast<size_t>(y) * W) + c4)
                                       : make_float4(NEG, NEG, NEG, NEG);
    reinterpret_cast<float4*>(tile + rr * W)[c4] = v;
  }
}

// peak mask of columns 4*x4 .. 4*x4+3 of tile row r+1 (= image row y0 + r)
__device__ __forceinline__ unsigned nms_tile_peaks(const float* tile, int W, int r, int x4, float threshold,
                                                   float (&mid)[4]) {
  const float NEG = -__int_as_float(0x7f800000);
  if (x4 >= (W >> 2)) return 0u;
  float row[3][6];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float* t = tile + (r + k) * W + 4 * x4;
    const float4 c = reinterpret_cast<const float4*>(t)[0];
    row[k][0] = x4 > 0 ? t[-1] : NEG;
    row[k][1] = c.x; row[k][2] = c.y; row[k][3] = c.z; row[k][4] = c.w;
    row[k][5] = 4 * x4 + 4 < W ? t[4] : NEG;
  }
  // "strictly greater than all 8 neighbours" as one comparison with their
  // maximum, built from shared pairwise maxima; max.NaN propagates a NaN
  // neighbour so it still blocks the peak, as in the oracle's comparisons
  auto mx = [](float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
  };
  float h0[4], h2[4];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float* a = row[2 * k];
    float pr[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) pr[i] = mx(a[i], a[i + 1]);
    float* h = k ? h2 : h0;
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = mx(pr[i], a[i + 2]);
  }
  unsigned m = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float v = row[1][i + 1];
    mid[i] = v;
    const float nb = mx(mx(h0[i], h2[i]), mx(row[1][i], row[1][i + 2]));
    m |= (v > threshold && v > nb) ? (1u << i) : 0u;
  }
  return m;
}

__global__ void nms4_count_kernel(const float* __restrict__ in, int H, int W, float threshold,
                                  int* __restrict__ row_counts) {
  extern __shared__ __align__(16) float tile[];
  __shared__ int rows_cnt[kNmsRows];
  const int y0 = blockIdx.x * kNmsRows, pl = blockIdx.y;
  const int rows = y0 + kNmsRows < H ? kNmsRows : H - y0;
  const float* p = in + static_cast<size_t>(pl) * H * W;
  if (threadIdx.x < kNmsRows) rows_cnt[threadIdx.x] = 0;
  nms_stage_tile(tile, p, H, W, y0, rows);
  __syncthreads();
  for (int r = 0; r < rows; ++r) {
    int cnt = 0;
    for (int x4 = threadIdx.x; x4 < (W >> 2); x4 += blockDim.x) {
      float mid[4];
      cnt += __popc(nms_tile_peaks(tile, W, r, x4, threshold, mid));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&rows_cnt[r], cnt);
  }
  __syncthreads();
  if (threadIdx.x < rows) row_counts[static_cast<size_t>(pl) * H + y0 + threadIdx.x] = rows_cnt[threadIdx.x];
}

// one pass over a row per iteration: blockDim covers W / 4 columns
__global__ void nms4_write_kernel(const float* __restrict__ in, int H, int W, float threshold, int max_peaks,
                                  const int* __restrict__ row_offsets, float* __restrict__ peaks) {
  extern __shared__ __align__(16) float tile[];
  __shared__ int warp_cnt[32];
  const int y0 = blockIdx.x * kNmsRows, pl = blockIdx.y;
  const int rows = y0 + kNmsRows < H ? kNmsRows : H - y0;
  const float* p = in + static_cast<size_t>(pl) * H * W;
  if (row_offsets[static_cast<size_t>(pl) * H + y0] >= max_peaks) return;
  nms_stage_tile(tile, p, H, W, y0, rows);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int x4 = threadIdx.x;
  for (int r = 0; r < rows; ++r) {
    const int y = y0 + r;
    const int base = row_offsets[static_cast<size_t>(pl) * H + y];
    if (base >= max_peaks) return;  // uniform: later rows start later
    float mid[4];
    const unsigned m = nms_tile_peaks(tile, W, r, x4, threshold, mid);
    // raster rank: peaks of earlier lanes / warps, then earlier columns of this thread
    const int mine = __popc(m);
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_cnt[wid] = incl;
    __syncthreads();
    int before = 0;
    for (int i = 0; i < wid; ++i) before += warp_cnt[i];
    int idx = base + before + incl - mine;
    for (int i = 0; i < 4; ++i) {
      if (!((m >> i) & 1u)) continue;
      if (idx < max_peaks) {
        const int x = 4 * x4 + i;
        float sw = 0.0f, sx = 0.0f, sy = 0.0f;
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const int yy = y + dy, xx = x + dx;
            if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
            const float sv = tile[(r + 1 + dy) * W + xx];
            sw = __fadd_rn(sw, sv);
            sx = __fadd_rn(sx, __fmul_rn(static_cast<float>(xx), sv));
            sy = __fadd_rn(sy, __fmul_rn(static_cast<float>(yy), sv));
          }
        float* o = peaks + (static_cast<size_t>(pl) * max_peaks + idx) * 5;
        o[0] = static_cast<float>(x);
        o[1] = static_cast<float>(y);
        o[2] = __fdiv_rn(sx, sw);
        o[3] = __fdiv_rn(sy, sw);
        o[4] = mid[i];
      }
      ++idx;
    }
    __syncthreads();  // warp_cnt is rewritten for the next row
  }
}

// Single pass (W % 4 == 0): every block takes the next 8-row tile in launch
// order (atomic ticket, so every earlier tile has started), counts its peaks,
// publishes the count, and finds the number of peaks before it in raster
// order by looking back over the earlier tiles of its plane (decoupled
// look-back: a tile whose inclusive prefix is already published ends the
// walk). It then writes its peaks at those offsets from its staged rows, so
// the heatmaps are read once instead of twice. Peak test and refinement are
// the same code as the two-pass kernels (bit-exact against the oracle).
constexpr unsigned long long kNmsAgg = 1ull << 62, kNmsPrefix = 1ull << 63;

__global__ void nms4_onepass_kernel(const float* __restrict__ in, int H, int W, float threshold, int max_peaks,
                                    int tiles_per_plane, unsigned long long* __restrict__ status,
                                    int* __restrict__ ticket, int* __restrict__ counts, float* __restrict__ peaks) {
  extern __shared__ __align__(16) float tile[];
  __shared__ int s_id, s_prefix, warp_cnt[32], row_tot[kNmsRows1];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    s_id = atomicAdd(ticket, 1);
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  if (threadIdx.x < kNmsRows1) row_tot[threadIdx.x] = 0;
  __syncthreads();
  const int id = s_id;
  const int pl = id / tiles_per_plane, tt = id - pl * tiles_per_plane;
  const int y0 = tt * kNmsRows1;
  const int rows = y0 + kNmsRows1 < H ? kNmsRows1 : H - y0;
  const float* p = in + static_cast<size_t>(pl) * H * W;
  // stage rows y0-1 .. y0+rows: the in-plane ones are contiguous in memory,
  // one bulk async copy (the whole tile in flight at once); the out-of-plane
  // halo rows read as -inf
  const int ya = y0 > 0 ? y0 - 1 : 0, yb = y0 + rows < H ? y0 + rows + 1 : H;  // [ya, yb) in the plane
  if (threadIdx.x == 0) {
    const uint32_t bytes = static_cast<uint32_t>(yb - ya) * W * 4;
    ptx::mbar_arrive_expect_tx(&bar, bytes);
    ptx::bulk_load(tile + (ya - (y0 - 1)) * W, p + static_cast<size_t>(ya) * W, bytes, &bar);
  }
  {
    const float NEG = -__int_as_float(0x7f800000);
    if (y0 == 0)
      for (int i = threadIdx.x; i < W; i += blockDim.x) tile[i] = NEG;
    if (y0 + rows == H)
      for (int i = threadIdx.x; i < W; i += blockDim.x) tile[(rows + 1) * W + i] = NEG;
  }
  ptx::mbar_wait(&bar, 0);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int x4 = threadIdx.x;  // blockDim covers W / 4 columns
  uint64_t masks = 0;          // 4 columns x kNmsRows1 rows of peak bits
  for (int r = 0; r < rows; ++r) {
    float mid[4];
    const unsigned m = nms_tile_peaks(tile, W, r, x4, threshold, mid);
    masks |= static_cast<uint64_t>(m) << (4 * r);
    int cnt = __popc(m);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0 && cnt) atomicAdd(&row_tot[r], cnt);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    // warp 0: publish this tile's count, then look back 32 tiles at a time
    int total = 0;
    for (int r = 0; r < rows; ++r) total += row_tot[r];
    unsigned long long* st = status + static_cast<size_t>(pl) * tiles_per_plane;
    if (lane == 0) atomicExch(&st[tt], (tt == 0 ? kNmsPrefix : kNmsAgg) | static_cast<unsigned>(total));
    int prefix = 0;
    for (int j = tt - 1; j >= 0; j -= 32) {
      const int idx = j - lane;  // lane k looks at tile j - k; before the plane: a prefix of 0
      unsigned long long v = idx >= 0 ? 0ull : kNmsPrefix;
      while (!__all_sync(0xffffffffu, (v & (kNmsAgg | kNmsPrefix)) != 0))
        if (!(v & (kNmsAgg | kNmsPrefix))) v = atomicAdd(&st[idx], 0ull);
      const unsigned pm = __ballot_sync(0xffffffffu, (v & kNmsPrefix) != 0);
      const int first = pm ? __ffs(pm) - 1 : 32;  // nearest tile whose inclusive prefix is known
      int c = lane <= first ? static_cast<int>(v & 0xffffffffu) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      prefix += c;
      if (pm) break;
    }
    if (lane == 0) {
      if (tt > 0) {
        __threadfence();
        atomicExch(&st[tt], kNmsPrefix | static_cast<unsigned>(prefix + total));
      }
      if (tt + 1 == tiles_per_plane) counts[pl] = prefix + total < max_peaks ? prefix + total : max_peaks;
      s_prefix = prefix;
    }
  }
  __syncthreads();
  int base = s_prefix;
  for (int r = 0; r < rows; ++r) {
    if (base >= max_peaks) return;  // uniform across the block
    const int y = y0 + r;
    const unsigned m = static_cast<unsigned>(masks >> (4 * r)) & 15u;
    const int mine = __popc(m);
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_cnt[wid] = incl;
    __syncthreads();
    int before = 0;
    for (int i = 0; i < wid; ++i) before += warp_cnt[i];
    int idx = base + before + incl - mine;
    for (int i = 0; i < 4; ++i) {
      if (!((m >> i) & 1u)) continue;
      if (idx < max_peaks) {
        const int x = 4 * x4 + i;
        float sw = 0.0f, sx = 0.0f, sy = 0.0f;
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const int yy = y + dy, xx = x + dx;
            if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
            const float sv = tile[(r + 1 + dy) * W + xx];
            sw = __fadd_rn(sw, sv);
            sx = __fadd_rn(sx, __fmul_rn(static_cast<float>(xx), sv));
            sy = __fadd_rn(sy, __fmul_rn(static_cast<float>(yy), sv));
          }
        float* o = peaks + (static_cast<size_t>(pl) * max_peaks + idx) * 5;
        o[0] = static_cast<float>(x);
        o[1] = static_cast<float>(y);
        o[2] = __fdiv_rn(sx, sw);
        o[3] = __fdiv_rn(sy, sw);
        o[4] = tile[(r + 1) * W + x];
      }
      ++idx;
    }
    base += row_tot[r];
    __syncthreads();  // warp_cnt is rewritten for the next row
  }
}

// Tile-compact NMS (W % 4 == 0, default). Pass 1 reads the heatmaps once:
// every 8-row tile (one bulk async copy) finds its peaks and writes the
// first `cap` of them, in raster order, to its own slot of a scratch list
// together with its peak count -- no block ever waits for another. Pass 2
// (one small block per plane) scans the tile counts and gathers the plane's
// first max_peaks peaks in raster order, refining each from its 3x3
// neighbourhood. Same peak test and refinement arithmetic as the two-pass
// kernels (bit-exact against the oracle).
struct NmsPeak {
  int x, y;
  float score;
};

__global__ void nms4_tiles_kernel(const float* __restrict__ in, int H, int W, float threshold, int cap,
                                  int* __restrict__ tile_counts, NmsPeak* __restrict__ tile_peaks) {
  extern __shared__ __align__(16) float tile[];
  __shared__ int wbase[kNmsRows1][32];
  __shared__ __align__(8) uint64_t bar;
  const int tiles = gridDim.x, tt = blockIdx.x, pl = blockIdx.y;
  const int y0 = tt * kNmsRows1;
  const int rows = y0 + kNmsRows1 < H ? kNmsRows1 : H - y0;
  const float* p = in + static_cast<size_t>(pl) * H * W;
  const int ya = y0 > 0 ? y0 - 1 : 0, yb = y0 + rows < H ? y0 + rows + 1 : H;  // in-plane rows [ya, yb)
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t bytes = static_cast<uint32_t>(yb - ya) * W * 4;
    ptx::mbar_arrive_expect_tx(&bar, bytes);
    ptx::bulk_load(tile + (ya - (y0 - 1)) * W, p + static_cast<size_t>(ya) * W, bytes, &bar);
  }
  {
    const float NEG = -__int_as_float(0x7f800000);
    if (y0 == 0)
      for (int i = threadIdx.x; i < W; i += blockDim.x) tile[i] = NEG;
    if (y0 + rows == H)
      for (int i = threadIdx.x; i < W; i += blockDim.x) tile[(rows + 1) * W + i] = NEG;
  }
  ptx::mbar_wait(&bar, 0);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int x4 = threadIdx.x;  // blockDim covers W / 4 columns
  uint64_t masks = 0;
  for (int r = 0; r < rows; ++r) {
    float mid[4];
    const unsigned m = nms_tile_peaks(tile, W, r, x4, threshold, mid);
    masks |= static_cast<uint64_t>(m) << (4 * r);
    int c = __popc(m);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) wbase[r][wid] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // raster order = row-major over (row, warp)
    int acc = 0;
    for (int r = 0; r < rows; ++r)
      for (int w = 0; w < nw; ++w) {
        const int c = wbase[r][w];
        wbase[r][w] = acc;
        acc += c;
      }
    tile_counts[static_cast<size_t>(pl) * tiles + tt] = acc;
  }
  __syncthreads();
  NmsPeak* out = tile_peaks + (static_cast<size_t>(pl) * tiles + tt) * cap;
  for (int r = 0; r < rows; ++r) {
    const unsigned m = static_cast<unsigned>(masks >> (4 * r)) & 15u;
    if (!__any_sync(0xffffffffu, m)) continue;  // typical heatmaps: most warp rows have no peak
    const int mine = __popc(m);
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    int idx = wbase[r][wid] + incl - mine;
    for (int i = 0; i < 4 && idx < cap; ++i) {
      if (!((m >> i) & 1u)) continue;
      const int x = 4 * x4 + i;
      out[idx] = NmsPeak{x, y0 + r, tile[(r + 1) * W + x]};
      ++idx;
    }
  }
}

// NMS pass 1 (W % 8 == 0, W <= 2048; the default): same per-tile peak lists
// as nms4_tiles_kernel. The tile's R + 2 rows land in shared memory by one
// bulk copy (all bytes in flight at once, no registers held for them); then
// each thread owns 8 columns and walks the rows top to bottom, reading every
// row ONCE (two conflict-free 16-byte loads), taking the neighbour columns
// from the adjacent lanes by shuffle (the warp's edge lanes read one scalar),
// and forming each row's horizontal 3-max and left/right max once for the
// rows above and below. nms4_tiles_kernel read every row three times with
// 4-way-conflicting scalar neighbour loads (~40 instructions per pixel,
// issue-bound). Same peak test (strictly greater than the max.NaN of the 8
// neighbours; max is associative and commutative, so the regrouping cannot
// change a comparison) and the same raster-ordered lists for nms_gather_kernel.
constexpr int kNms8Rows = 5;  // tile height, measured on C2 planes (stress / sparse threshold, us): 4: 44.4 / 41.9, 5: 39.9 / 38.3, 6: 40.5 / 38.5, 8: 42.3 / 39.0, 12: 47.6 / 44.5, 16: 49.6 / 46.9

// One tile per block (a persistent, double-buffered variant in which each
// block prefetched its next tile measured slower, 67 us: fewer resident
// warps for the compute).
template <int R>
__global__ void __launch_bounds__(256) nms8_tiles_kernel(const float* __restrict__ in, int H, int W, float threshold,
                                                         int cap, int tiles, int* __restrict__ tile_counts,
                                                         NmsPeak* __restrict__ tile_peaks) {
  extern __shared__ __align__(16) float tile[];  // rows y0-1 .. y0+R (-inf outside the plane)
  __shared__ int wbase[R][8];
  __shared__ uint8_t pmask[R][256];
  __shared__ __align__(8) uint64_t bar;
  const float NEG = -__int_as_float(0x7f800000);
  const int x8 = threadIdx.x, c0 = 8 * x8;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool col_ok = c0 < W;
  const int t = blockIdx.x;  // = plane * tiles + tile index
  const int pl = t / tiles, y0 = (t - pl * tiles) * R;
  const int rows = y0 + R < H ? R : H - y0;
  const int ya = y0 > 0 ? y0 - 1 : 0, yb = y0 + rows < H ? y0 + rows + 1 : H;  // in-plane rows [ya, yb)
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_barrier_init();
    const uint32_t bytes = static_cast<uint32_t>(yb - ya) * W * 4;
    ptx::mbar_arrive_expect_tx(&bar, bytes);
    ptx::bulk_load(tile + (ya - (y0 - 1)) * W, in + static_cast<size_t>(pl) * H * W + static_cast<size_t>(ya) * W,
                   bytes, &bar);
  }
  if (y0 == 0)
    for (int i = threadIdx.x; i < W; i += blockDim.x) tile[i] = NEG;
  if (y0 + rows == H)
    for (int i = threadIdx.x; i < W; i += blockDim.x) tile[(rows + 1) * W + i] = NEG;
  __syncthreads();  // (also orders the barrier's init before the other threads' waits)
  ptx::mbar_wait(&bar, 0);
  auto mx = [](float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
  };
  struct Row {
    float4 a, b;
    float el, er;  // lane 0: column c0 - 1; lane 31: column c0 + 8
  };
  {
    auto load = [&](int k) {  // tile row k = image row y0 - 1 + k
      Row r;
      const float* rp = tile + k * W + c0;
      const float4 n4 = make_float4(NEG, NEG, NEG, NEG);
      r.a = col_ok ? reinterpret_cast<const float4*>(rp)[0] : n4;
      r.b = col_ok ? reinterpret_cast<const float4*>(rp)[1] : n4;
      r.el = (lane == 0 && col_ok && c0 > 0) ? rp[-1] : NEG;
      r.er = (lane == 31 && c0 + 8 < W) ? rp[8] : NEG;
      return r;
    };
    // hm: max of the 3 columns around each of mine; lr: max of left and right
    auto horiz = [&](const Row& r, float (&v)[8], float (&lr)[8], float (&hm)[8]) {
      float left = __shfl_up_sync(0xffffffffu, r.b.w, 1);
      float right = __shfl_down_sync(0xffffffffu, r.a.x, 1);
      if (lane == 0) left = r.el;
      if (lane == 31) right = r.er;
      const float e[10] = {left, r.a.x, r.a.y, r.a.z, r.a.w, r.b.x, r.b.y, r.b.z, r.b.w, right};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[i] = e[i + 1];
        lr[i] = mx(e[i], e[i + 2]);
        hm[i] = mx(lr[i], e[i + 1]);
      }
    };
    float v_cur[8], lr_cur[8], hm_cur[8], hm_prev[8];
    {
      float vd[8], lrd[8];
      const Row r0 = load(0), r1 = load(1);
      horiz(r0, vd, lrd, hm_prev);
      horiz(r1, v_cur, lr_cur, hm_cur);
    }
    Row nxt = load(2);
    // unrolled over all R rows with no branch (a short last tile computes the
    // rows past its end from stale shared memory and masks them), so the
    // row-to-row rotation of the per-thread values is register renaming
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float v_n[8], lr_n[8], hm_n[8];
      horiz(nxt, v_n, lr_n, hm_n);  // row y0 + r + 1
      if (r + 3 <= R + 1) nxt = load(r + 3);
      unsigned m = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        // v > threshold and v > every neighbour, as one comparison with
        // max.NaN(neighbours, threshold): a NaN anywhere still fails it
        const float lim = mx(mx(mx(hm_prev[i], hm_n[i]), lr_cur[i]), threshold);
        m |= v_cur[i] > lim ? (1u << i) : 0u;
      }
      if (!col_ok || r >= rows) m = 0;
      pmask[r][threadIdx.x] = static_cast<uint8_t>(m);
      const int c = __reduce_add_sync(0xffffffffu, __popc(m));
      if (lane == 0) wbase[r][wid] = c;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        hm_prev[i] = hm_cur[i];
        hm_cur[i] = hm_n[i];
        lr_cur[i] = lr_n[i];
        v_cur[i] = v_n[i];
      }
    }
    __syncthreads();
    if (wid == 0) {
      // exclusive prefix over (row, warp) in raster order: lane l sums a run
      // of the rows * nw counts, then one warp scan
      const int n = rows * nw, per = (n + 31) / 32, beg = lane * per;
      int run = 0;
      for (int e = beg; e < beg + per && e < n; ++e) run += wbase[e / nw][e % nw];
      int incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int q = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += q;
      }
      int acc = incl - run;
      for (int e = beg; e < beg + per && e < n; ++e) {
        const int c = wbase[e / nw][e % nw];
        wbase[e / nw][e % nw] = acc;
        acc += c;
      }
      if (lane == 31) tile_counts[t] = incl;  // t = pl * tiles + tile index
    }
    __syncthreads();
    NmsPeak* out = tile_peaks + static_cast<size_t>(t) * cap;
    for (int r = 0; r < rows; ++r) {
      if (wbase[r][0] >= cap) break;  // the tile's list is full (uniform: shared offsets only grow)
      const unsigned m = pmask[r][threadIdx.x];
      if (!__any_sync(0xffffffffu, m)) continue;  // typical heatmaps: most warp rows have no peak
      const int mine = __popc(m);
      int incl = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int q = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += q;
      }
      int idx = wbase[r][wid] + incl - mine;
      for (int i = 0; i < 8 && idx < cap; ++i) {
        if (!((m >> i) & 1u)) continue;
        const int x = c0 + i;
        out[idx] = NmsPeak{x, y0 + r, tile[(r + 1) * W + x]};
        ++idx;
      }
    }
  }
}

__global__ void nms_gather_kernel(const float* __restrict__ in, int H, int W, int tiles, int cap, int max_peaks,
                                  const int* __restrict__ tile_counts, const NmsPeak* __restrict__ tile_peaks,
                                  int* __restrict__ counts, float* __restrict__ peaks) {
  extern __shared__ int base[];  // tiles + 1 exclusive prefix
  const int pl = blockIdx.x;
  if (threadIdx.x < 32) {
    // warp 0: lane l loads and sums a contiguous run of the tile counts
    // (all loads in flight at once), then one warp scan
    const int lane = threadIdx.x, per = (tiles + 31) / 32, beg = lane * per;
    const int* tc = tile_counts + static_cast<size_t>(pl) * tiles;
    int run = 0;
    for (int t = beg; t < beg + per && t < tiles; ++t) run += tc[t];
    int incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int q = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += q;
    }
    int acc = incl - run;
    for (int t = beg; t < beg + per && t < tiles; ++t) {
      base[t] = acc;
      acc += tc[t];
    }
    if (lane == 31) {
      base[tiles] = incl;
      if (blockIdx.y == 0) counts[pl] = incl < max_peaks ? incl : max_peaks;
    }
  }
  __syncthreads();
  const int n = base[tiles] < max_peaks ? base[tiles] : max_peaks;
  const float* p = in + static_cast<size_t>(pl) * H * W;
  // blockIdx.y: this block's slice of the plane's first max_peaks peaks
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < n; i += gridDim.y * blockDim.x) {
    int lo = 0, hi = tiles;  // the tile holding peak i: base[lo] <= i < base[lo + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (base[mid] <= i) lo = mid;
      else hi = mid;
    }
    const NmsPeak pk = tile_peaks[(static_cast<size_t>(pl) * tiles + lo) * cap + (i - base[lo])];
    float sw = 0.0f, sx = 0.0f, sy = 0.0f;
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int yy = pk.y + dy, xx = pk.x + dx;
        if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
        const float sv = __ldg(p + static_cast<size_t>(yy) * W + xx);
        sw = __fadd_rn(sw, sv);
        sx = __fadd_rn(sx, __fmul_rn(static_cast<float>(xx), sv));
        sy = __fadd_rn(sy, __fmul_rn(static_cast<float>(yy), sv));
      }
    float* o = peaks + (static_cast<size_t>(pl) * max_peaks + i) * 5;
    o[0] = static_cast<float>(pk.x);
    o[1] = static_cast<float>(pk.y);
    o[2] = __fdiv_rn(sx, sw);
    o[3] = __fdiv_rn(sy, sw);
    o[4] = pk.score;
  }
}

// Fused x8 upsample + NMS pass 1 (avec_upsample_nms_device): the heatmap
// planes NMS reads are the ones upsample just wrote, so the pair re-read them
// from HBM (C2: 139 MB written, then 139 MB read back). Here a block owns one
// source-row period of a plane, output rows 8k .. 8k+7 (all of which lie
// between source rows k-1, k, k+1), and thread g owns the 8-output group of
// source column g. It computes output rows 8k-1 .. 8k+8 in registers with the
// op sequence of upsample8_kernel (bit for bit: interior groups at the
// constant lx of kLx, the two row-end groups at the clamped coordinates the
// general src_coord_pow2 yields for them, written out below), stores rows
// 8k .. 8k+7, and runs nms8_tiles_kernel's comparisons on the values as they
// are produced: the plane is written once and never read back (only the few
// peak values are, from L2). Same per-tile raster lists for nms_gather_kernel
// (tiles = h per plane). Instruction-bound rather than HBM-bound (~11 ops per
// output pixel: vertical lerp, 3x3 maxima, test); staging the stores through
// shared memory for whole-sector store instructions measured slower (56-58
// vs 52-54 us on C2's 144 planes).
// Row-end groups, from src_coord_pow2(8g + j, 1/8, w): g = 0, j < 4 clamps to
// f = 0 (columns 0, 1 at lx = 0), j >= 4 sits at 0 + (j - 3.5)/8; g = w - 1,
// j < 4 sits between w - 2 and w - 1 at kLx[j], j >= 4 at column w - 1 with
// x1 clamped to w - 1. So every group is "left half between columns (L0, L1)
// at lxL[j], right half between (R0, R1) at kLx[4 + j]", with (L0, L1, R0, R1)
// = (g-1, g, g, g+1) inside, (0, 1, 0, 1) at g = 0, (w-2, w-1, w-1, w-1) at w-1.
__global__ void __launch_bounds__(256, 3) ups8_nms_kernel(const float* __restrict__ in, int h, int w, float threshold,
                                                       int cap, float* __restrict__ out, int* __restrict__ tile_counts,
                                                       NmsPeak* __restrict__ tile_peaks) {
  constexpr int R = 8;
  __shared__ int wbase[R * 8];                  // per (row, warp) counts, then offsets, raster order r * nw + warp
  __shared__ uint8_t pmask[R][256];
  constexpr float kLx[8] = {0.5625f, 0.6875f, 0.8125f, 0.9375f, 0.0625f, 0.1875f, 0.3125f, 0.4375f};
  const float NEG = -__int_as_float(0x7f800000);
  const int H = 8 * h, W = 8 * w;
  const int g = threadIdx.x, c0 = 8 * g;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool col_ok = g < w;
  const int t = blockIdx.x;  // = plane * h + k
  const int pl = t / h, k = t - pl * h, y0 = 8 * k;
  const float* src = in + static_cast<size_t>(pl) * h * w;
  float* dst = out + static_cast<size_t>(pl) * H * W;
  const int gc = col_ok ? g : w - 1;  // idle lanes load in-range columns (their values are never used)
  const int L0 = gc > 0 ? gc - 1 : 0, L1 = gc > 0 ? gc : 1, R0 = gc, R1 = gc + 1 < w ? gc + 1 : w - 1;
  // Source rows: output rows 8k-1 .. 8k+3 lie between the pair src_coord_pow2
  // gives row 8k (k-1, k; (0, 1) at k = 0, where row -1 is outside), rows
  // 8k+4 .. 8k+8 between the pair of row 8k+4 (k, k+1; clamped at k = h-1,
  // where row 8k+8 is outside). Both pairs' source values load up front.
  int ya0, ya1, yb0, yb1;
  src_coord_pow2(y0, 0.125f, h, ya0, ya1);
  src_coord_pow2(y0 + 4, 0.125f, h, yb0, yb1);
  float A[8], B[8];  // (L0, L1, R0, R1) of the pair's top row, then of its bottom row
  {
    const float* a0 = src + static_cast<size_t>(ya0) * w;
    const float* a1 = src + static_cast<size_t>(ya1) * w;
    const float* b0 = src + static_cast<size_t>(yb0) * w;
    const float* b1 = src + static_cast<size_t>(yb1) * w;
    A[0] = __ldg(a0 + L0), A[1] = __ldg(a0 + L1), A[2] = __ldg(a0 + R0), A[3] = __ldg(a0 + R1);
    A[4] = __ldg(a1 + L0), A[5] = __ldg(a1 + L1), A[6] = __ldg(a1 + R0), A[7] = __ldg(a1 + R1);
    B[0] = __ldg(b0 + L0), B[1] = __ldg(b0 + L1), B[2] = __ldg(b0 + R0), B[3] = __ldg(b0 + R1);
    B[4] = __ldg(b1 + L0), B[5] = __ldg(b1 + L1), B[6] = __ldg(b1 + R0), B[7] = __ldg(b1 + R1);
  }
  float lxL[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) lxL[j] = gc > 0 ? kLx[j] : 0.0f;
  auto mx = [](float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
  };
  // horizontal lerps of the current pair (tp: its top row, bt: its bottom row)
  float tp[8], bt[8], tEl, bEl, tEr, bEr;
  auto hsetup = [&](const float (&S)[8]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      tp[j] = lerp2(S[0], S[1], lxL[j]);
      bt[j] = lerp2(S[4], S[5], lxL[j]);
      tp[4 + j] = lerp2(S[2], S[3], kLx[4 + j]);
      bt[4 + j] = lerp2(S[6], S[7], kLx[4 + j]);
    }
    // column c0 - 1 = group g - 1's last output (between g - 1 and g at kLx[7]);
    // column c0 + 8 = group g + 1's first (between g and g + 1 at kLx[0])
    tEl = lerp2(S[0], S[1], kLx[7]);
    bEl = lerp2(S[4], S[5], kLx[7]);
    tEr = lerp2(S[2], S[3], kLx[0]);
    bEr = lerp2(S[6], S[7], kLx[0]);
  };
  struct Row {
    float v[8];
    float el, er;  // columns c0 - 1 and c0 + 8 (-inf outside the plane)
  };
  // output row y0 + rr (rr = -1 .. 8): its values, and its store for rr = 0 .. 7
  auto make = [&](int rr) {
    Row r;
    const int oy = y0 + rr;
    if (oy < 0 || oy >= H) {  // block-uniform: the halo row above the first / below the last tile
#pragma unroll
      for (int j = 0; j < 8; ++j) r.v[j] = NEG;
      r.el = r.er = NEG;
      return r;
    }
    int ys0, ys1;
    const float ly = src_coord_pow2(oy, 0.125f, h, ys0, ys1);
#pragma unroll
    for (int j = 0; j < 8; ++j) r.v[j] = lerp2(tp[j], bt[j], ly);
    r.el = col_ok && g > 0 ? lerp2(tEl, bEl, ly) : NEG;
    r.er = g + 1 < w ? lerp2(tEr, bEr, ly) : NEG;
    if (rr >= 0 && rr < R && col_ok) {  // two float4 per lane (a warp's stores are one contiguous 1 KB span)
      float4* d = reinterpret_cast<float4*>(dst + static_cast<size_t>(oy) * W + c0);
      d[0] = make_float4(r.v[0], r.v[1], r.v[2], r.v[3]);
      d[1] = make_float4(r.v[4], r.v[5], r.v[6], r.v[7]);
    }
    return r;
  };
  // hm: max of the 3 columns around each of mine; lr: max of left and right.
  // Lanes past the plane (g >= w) hold values of column w - 1 that no one
  // may see: the plane's last group takes its right neighbour from r.er.
  auto horiz = [&](const Row& r, float (&v)[8], float (&lr)[8], float (&hm)[8]) {
    float left = __shfl_up_sync(0xffffffffu, r.v[7], 1);
    float right = __shfl_down_sync(0xffffffffu, r.v[0], 1);
    if (lane == 0) left = r.el;
    if (lane == 31 || g + 1 >= w) right = r.er;
    const float e[10] = {left, r.v[0], r.v[1], r.v[2], r.v[3], r.v[4], r.v[5], r.v[6], r.v[7], right};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i] = e[i + 1];
      lr[i] = mx(e[i], e[i + 2]);
      hm[i] = mx(lr[i], e[i + 1]);
    }
  };
  float v_cur[8], lr_cur[8], hm_cur[8], hm_prev[8];
  hsetup(A);
  {
    float vd[8], lrd[8];
    horiz(make(-1), vd, lrd, hm_prev);
    horiz(make(0), v_cur, lr_cur, hm_cur);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (r + 1 == 4) hsetup(B);  // rows 8k+4 .. 8k+8
    float v_n[8], lr_n[8], hm_n[8];
    horiz(make(r + 1), v_n, lr_n, hm_n);
    unsigned m = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      // nms8_tiles_kernel's test: v > max.NaN(8 neighbours, threshold)
      const float lim = mx(mx(mx(hm_prev[i], hm_n[i]), lr_cur[i]), threshold);
      m |= v_cur[i] > lim ? (1u << i) : 0u;
    }
    if (!col_ok) m = 0;
    pmask[r][threadIdx.x] = static_cast<uint8_t>(m);
    const int c = __reduce_add_sync(0xffffffffu, __popc(m));
    if (lane == 0) wbase[r * nw + wid] = c;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      hm_prev[i] = hm_cur[i];
      hm_cur[i] = hm_n[i];
      lr_cur[i] = lr_n[i];
      v_cur[i] = v_n[i];
    }
  }
  __syncthreads();  // also makes this block's stores of its rows visible to the peak writes below
  if (wid == 0) {
    const int n = R * nw;  // <= 64: lanes l and l + 32
    const int c_a = lane < n ? wbase[lane] : 0, c_b = lane + 32 < n ? wbase[lane + 32] : 0;
    int incl = c_a;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int q = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += q;
    }
    const int tot_a = __shfl_sync(0xffffffffu, incl, 31);
    int incl_b = c_b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int q = __shfl_up_sync(0xffffffffu, incl_b, o);
      if (lane >= o) incl_b += q;
    }
    if (lane < n) wbase[lane] = incl - c_a;
    if (lane + 32 < n) wbase[lane + 32] = tot_a + incl_b - c_b;
    if (lane == 31) tile_counts[t] = tot_a + incl_b;
  }
  __syncthreads();
  NmsPeak* outp = tile_peaks + static_cast<size_t>(t) * cap;
  for (int r = 0; r < R; ++r) {
    if (wbase[r * nw] >= cap) break;  // the tile's list is full (uniform: offsets only grow)
    const unsigned m = pmask[r][threadIdx.x];
    if (!__any_sync(0xffffffffu, m)) continue;
    const int mine = __popc(m);
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int q = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += q;
    }
    int idx = wbase[r * nw + wid] + incl - mine;
    const float* vrow = dst + static_cast<size_t>(y0 + r) * W + c0;  // written above by this block
    float pv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) pv[i] = (m >> i) & 1u ? vrow[i] : 0.0f;  // all loads in flight at once
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (!((m >> i) & 1u) || idx >= cap) continue;
      outp[idx] = NmsPeak{c0 + i, y0 + r, pv[i]};
      ++idx;
    }
  }
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
  const bool pow2 = scale >= 8 && scale <= 64 && (scale & (scale - 1)) == 0;
  if (pow2 && h * scale <= 65535 && planes <= 65535) {  // 8 outputs per thread: <= 3 source columns each side
    const int wg = w * scale / 8;
    const float inv = 1.0f / static_cast<float>(scale);
    if (scale == 8 && w >= 3 && w <= 498) {
      // a block per 4 output rows: a float4 x 4 rows per thread for the
      // interior, then one warp for the row ends (general coordinates)
      const int n = 2 * (w - 2);
      const int tpb = (n + 31) / 32 * 32 + 32;
      upsample8_kernel<<<dim3(1, h * 2, planes), tpb, 0, stream>>>(d_in, h, w, d_out);
    } else {
      const int tpb = wg >= 128 ? 128 : (wg + 31) / 32 * 32;
      upsample_pow2_kernel<<<dim3((wg + tpb - 1) / tpb, h * scale, planes), tpb, 0, stream>>>(
          d_in, planes, h, w, scale, inv, d_out);
    }
    check_cuda(cudaGetLastError(), "upsample launch");
    return;
  }
  if ((w * scale) % 4 != 0) fail(AVEC_ERR_UNSUPPORTED, "upsample needs output width % 4 == 0");
  const long long total = static_cast<long long>(planes) * h * scale * (w * scale / 4);
  upsample_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream>>>(
      d_in, planes, h, w, scale, d_out);
  check_cuda(cudaGetLastError(), "upsample launch");
}

size_t nms_scratch_bytes(int planes, int H, int /*W*/, int max_peaks) {
  // two-pass row counts/offsets, or the tile-compact path's counts + peak lists
  const int rmin = kNmsRows1 < kNms8Rows ? kNmsRows1 : kNms8Rows;  // the smaller tile height of the two paths
  const size_t tiles = (static_cast<size_t>(H) + rmin - 1) / rmin;
  const size_t compact = static_cast<size_t>(planes) * tiles * (sizeof(int) + sizeof(NmsPeak) * max_peaks) + 64;
  return std::max(2 * static_cast<size_t>(planes) * H * sizeof(int), compact);
}

void launch_nms(const float* d_in, int planes, int H, int W, float threshold, int max_peaks,
                int* d_counts, float* d_peaks, void* d_scratch, size_t scratch_bytes,
                cudaStream_t stream) {
  if (scratch_bytes < nms_scratch_bytes(planes, H, W, max_peaks)) fail(AVEC_ERR_INVALID_ARGUMENT, "nms scratch");
  if (H > 65535 || planes > 65535) fail(AVEC_ERR_UNSUPPORTED, "nms grid limits");
  int* row_counts = static_cast<int*>(d_scratch);
  int* row_offsets = row_counts + static_cast<size_t>(planes) * H;
  dim3 grid(H, planes);
  if (W % 4 == 0 && W <= 4096) {  // row tiles in smem, four columns per thread
    const int threads = ((W / 4) + 31) / 32 * 32;
    const size_t tile_bytes = static_cast<size_t>(kNmsRows + 2) * W * sizeof(float);
    if (tile_bytes > 48 * 1024) {  // wide planes (C5's 1312 columns): opt in to the larger carve-out
      check_cuda(cudaFuncSetAttribute(nms4_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(tile_bytes)), "nms smem");
      check_cuda(cudaFuncSetAttribute(nms4_write_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(tile_bytes)), "nms smem");
    }
    const int tiles = (H + kNmsRows - 1) / kNmsRows;
    const int tiles1 = (H + kNmsRows1 - 1) / kNmsRows1;
    const size_t tile1_bytes = static_cast<size_t>(kNmsRows1 + 2) * W * sizeof(float);
    static const bool two_pass = [] {
      const char* e = std::getenv("AVEC_NMS_TWOPASS");
      return e && e[0] == '1';
    }();
    static const int mode = [] {  // 0 tile-compact (default), 1 one-pass look-back
      const char* e = std::getenv("AVEC_NMS_LOOKBACK");
      return e && e[0] == '1' ? 1 : 0;
    }();
    static const bool staged = [] {  // AVEC_NMS_STAGED=1: the shared-memory tile pass 1
      const char* e = std::getenv("AVEC_NMS_STAGED");
      return e && e[0] == '1';
    }();
    if (!two_pass && mode == 0 && !staged && W % 8 == 0 && W <= 2048 &&
        (reinterpret_cast<uintptr_t>(d_in) & 15) == 0 && max_peaks > 0) {
      const int tiles_s = (H + kNms8Rows - 1) / kNms8Rows;
      const int threads8 = ((W / 8) + 31) / 32 * 32;
      int* tile_counts = static_cast<int*>(d_scratch);
      auto* tile_peaks = reinterpret_cast<NmsPeak*>(
          reinterpret_cast<uintptr_t>(tile_counts + static_cast<size_t>(planes) * tiles_s + 15) & ~uintptr_t(15));
      const size_t tile8_bytes = static_cast<size_t>(kNms8Rows + 2) * W * sizeof(float);
      static bool configured = false;
      if (!configured) {  // up to W = 2048 (+ ~2.3 KB of static tables)
        check_cuda(cudaFuncSetAttribute(nms8_tiles_kernel<kNms8Rows>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (kNms8Rows + 2) * 2048 * 4), "nms smem");
        configured = true;
      }
      const int total = tiles_s * planes;
      nms8_tiles_kernel<kNms8Rows><<<total, threads8, tile8_bytes, stream>>>(d_in, H, W, threshold, max_peaks, tiles_s,
                                                                           tile_counts, tile_peaks);
      // a block per (plane, 64 peaks): the refinement's 9 loads per peak in flight on many SMs
      nms_gather_kernel<<<dim3(planes, (max_peaks + 63) / 64), 64, (tiles_s + 1) * sizeof(int), stream>>>(
          d_in, H, W, tiles_s, max_peaks, max_peaks, tile_counts, tile_peaks, d_counts, d_peaks);
      check_cuda(cudaGetLastError(), "nms launch");
      return;
    }
    if (!two_pass && mode == 0 && (reinterpret_cast<uintptr_t>(d_in) & 15) == 0 && max_peaks > 0) {
      if (tile1_bytes > 48 * 1024)
        check_cuda(cudaFuncSetAttribute(nms4_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(tile1_bytes)), "nms smem");
      int* tile_counts = static_cast<int*>(d_scratch);
      auto* tile_peaks = reinterpret_cast<NmsPeak*>(
          reinterpret_cast<uintptr_t>(tile_counts + static_cast<size_t>(planes) * tiles1 + 15) & ~uintptr_t(15));
      nms4_tiles_kernel<<<dim3(tiles1, planes), threads, tile1_bytes, stream>>>(d_in, H, W, threshold, max_peaks,
                                                                                 tile_counts, tile_peaks);
      nms_gather_kernel<<<dim3(planes, (max_peaks + 63) / 64), 64, (tiles1 + 1) * sizeof(int), stream>>>(
          d_in, H, W, tiles1, max_peaks, max_peaks, tile_counts, tile_peaks, d_counts, d_peaks);
      check_cuda(cudaGetLastError(), "nms launch");
      return;
    }
    if (!two_pass && (reinterpret_cast<uintptr_t>(d_in) & 15) == 0) {
      if (tile1_bytes > 48 * 1024)
        check_cuda(cudaFuncSetAttribute(nms4_onepass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(tile1_bytes)), "nms smem");
      // look-back status words + the tile ticket, zeroed for this launch
      auto* status = reinterpret_cast<unsigned long long*>(d_scratch);
      int* ticket = reinterpret_cast<int*>(status + static_cast<size_t>(planes) * tiles1);
      check_cuda(cudaMemsetAsync(d_scratch, 0, static_cast<size_t>(planes) * tiles1 * 8 + 4, stream), "nms status");
      nms4_onepass_kernel<<<tiles1 * planes, threads, tile1_bytes, stream>>>(d_in, H, W, threshold, max_peaks, tiles1,
                                                                              status, ticket, d_counts, d_peaks);
      check_cuda(cudaGetLastError(), "nms launch");
      return;
    }
    dim3 grid4(tiles, planes);
    nms4_count_kernel<<<grid4, threads, tile_bytes, stream>>>(d_in, H, W, threshold, row_counts);
    nms_scan_kernel<<<planes, 32, 0, stream>>>(row_counts, H, max_peaks, row_offsets, d_counts);
    nms4_write_kernel<<<grid4, threads, tile_bytes, stream>>>(d_in, H, W, threshold, max_peaks, row_offsets,
                                                              d_peaks);
    check_cuda(cudaGetLastError(), "nms launch");
    return;
  }
  nms_count_kernel<<<grid, 256, 0, stream>>>(d_in, H, W, threshold, row_counts);
  nms_scan_kernel<<<planes, 32, 0, stream>>>(row_counts, H, max_peaks, row_offsets, d_counts);
  nms_write_kernel<<<grid, 256, 0, stream>>>(d_in, H, W, threshold, max_peaks, row_offsets,
                                              d_peaks);
  check_cuda(cudaGetLastError(), "nms launch");
}

void launch_upsample_nms(const float* d_in, int planes, int h, int w, float threshold, int max_peaks, float* d_out,
                         int* d_counts, float* d_peaks, void* d_scratch, size_t scratch_bytes, cudaStream_t stream) {
  static const bool split = [] {  // AVEC_UPSNMS_SPLIT=1: the two separate launches (A/B)
    const char* e = std::getenv("AVEC_UPSNMS_SPLIT");
    return e && e[0] == '1';
  }();
  const size_t tiles = static_cast<size_t>(planes) * h;
  const size_t need = tiles * sizeof(int) + 16 + tiles * max_peaks * sizeof(NmsPeak);
  if (!split && w >= 3 && w <= 256 && tiles <= 0x7fffffff && planes <= 65535 && max_peaks > 0 &&
      (reinterpret_cast<uintptr_t>(d_out) & 15) == 0 && need <= scratch_bytes) {
    int* tile_counts = static_cast<int*>(d_scratch);
    auto* tile_peaks = reinterpret_cast<NmsPeak*>(reinterpret_cast<uintptr_t>(tile_counts + tiles + 15) & ~uintptr_t(15));
    const int threads = (w + 31) / 32 * 32;
    // registers capped for 3 blocks of 256 threads per SM (80, no spills): 50 vs 54 us uncapped (94)
    ups8_nms_kernel<<<static_cast<unsigned>(tiles), threads, 0, stream>>>(d_in, h, w, threshold, max_peaks, d_out,
                                                                         tile_counts, tile_peaks);
    nms_gather_kernel<<<dim3(planes, (max_peaks + 63) / 64), 64, (h + 1) * sizeof(int), stream>>>(
        d_out, 8 * h, 8 * w, h, max_peaks, max_peaks, tile_counts, tile_peaks, d_counts, d_peaks);
    check_cuda(cudaGetLastError(), "upsample+nms launch");
    return;
  }
  launch_upsample(d_in, planes, h, w, 8, d_out, stream);
  launch_nms(d_out, planes, 8 * h, 8 * w, threshold, max_peaks, d_counts, d_peaks, d_scratch, scratch_bytes, stream);
}

}  // namespace avec
