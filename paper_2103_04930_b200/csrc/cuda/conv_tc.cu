// tcgen05 implicit-GEMM convolution — see conv_tc.cuh for the design.
#include <cuda_bf16.h>

#include <cstdlib>

#include "conv_tc.cuh"
#include "engine.hpp"
#include "ptx.cuh"
#include "trace.cuh"

namespace avec {

namespace {

using namespace ptx;

constexpr int kTileM = 128;   // output channels per tile (MMA M)
constexpr int kSubN = 256;    // pixels per MMA (MMA N)
constexpr int kWgtBytes = kTileM * 128;  // 128 rows x 64 bf16
constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 512;
constexpr int kChunk = 32;                      // epilogue pixels per TMEM load / TMA store
constexpr int kStageBytes = 2 * kChunk * 128;   // two 64-channel halves of 32 rows x 128 B
constexpr int kEpiThreads = 128;
constexpr int kEpiBar = 1;                      // named barrier id for the 4 epilogue warps

template <int SUBS>
struct Cfg {
  static constexpr int kTileN = kSubN * SUBS;
  static constexpr int kWinRows = kTileN + 8;   // + (k-1) <= 7 halo rows, 8-aligned
  static constexpr int kWinBytes = kWinRows * 128;
  static constexpr int kWinStages = 2;
  static constexpr int kAccStages = 2 / SUBS;   // TMEM holds 512 fp32 columns
  // the wide tiles trade the second epilogue staging buffer for a 5th weight
  // stage: deeper weight prefetch matters more than epilogue overlap there
  static constexpr int kStgBufs = SUBS == 2 ? 1 : 2;
  static constexpr int kWgtStages = SUBS == 2 ? 5 : 8;
  static constexpr int win = 0;
  static constexpr int wgt = win + kWinStages * kWinBytes;
  static constexpr int stg = wgt + kWgtStages * kWgtBytes;
  static constexpr int bars = stg + kStgBufs * kStageBytes;
  static constexpr int total = bars + 256;
  static_assert(kWinBytes % 1024 == 0 && wgt % 1024 == 0 && stg % 1024 == 0,
                "SW128 operands need 1024 B alignment");
  static_assert(total + 1024 <= 232448, "smem budget");
};

struct TileCoord {
  int g, n, pt, mt;
};

__device__ __forceinline__ TileCoord decode_tile(const ConvParams& p, int t) {
  TileCoord c;
  const int per_group = p.n_images * p.tiles_per_image * p.m_tiles;
  c.g = t / per_group;
  int rem = t - c.g * per_group;
  c.mt = rem % p.m_tiles;
  rem /= p.m_tiles;
  c.pt = rem % p.tiles_per_image;
  c.n = rem / p.tiles_per_image;
  return c;
}

// One unit of work: output positions [o0, o0+len) of image n, branch g, channel
// tile mt; with split-K, window iterations [w0, w1) of tile t's K loop only.
struct Work {
  int g, n, mt, o0, len;
  int t, ks;
};

// Iterates this CTA's work. Regular mode: fixed tiles strided by gridDim.x.
// Balanced mode (p.balanced_units > 0): the (branch, image) segments are cut
// into 32-position units and every CTA takes an equal contiguous run of them,
// split at segment ends and at kMaxLen positions, so all SMs finish together
// instead of 128 tiles leaving 20 of 148 SMs idle. Runs that end mid-chunk
// overlap a neighbour's first chunk; both CTAs compute bit-identical values
// for those positions, so the duplicate stores are benign.
struct WorkIter {
  int cur, end;
  __device__ explicit WorkIter(const ConvParams& p) {
    if (p.balanced_units > 0) {
      cur = int(static_cast<long long>(blockIdx.x) * p.balanced_units / gridDim.x);
      end = int(static_cast<long long>(blockIdx.x + 1) * p.balanced_units / gridDim.x);
    } else {
      cur = blockIdx.x;
      end = p.total_tiles * (p.splits > 1 ? p.splits : 1);
    }
  }
  template <int kMaxLen>
  __device__ bool next(const ConvParams& p, Work& w) {
    if (cur >= end) return false;
    if (p.balanced_units > 0) {
      const int U = p.units_per_seg;
      const int seg = cur / U, off = cur - seg * U;
      const int take = min(min(end, (seg + 1) * U) - cur, kMaxLen / 32);
      w.g = seg / p.n_images;
      w.n = seg - w.g * p.n_images;
      w.mt = 0;
      w.o0 = off * 32;
      w.len = take * 32;
      cur += take;
    } else {
      // the splits of one tile are adjacent units: they run side by side and
      // share the tile's activation windows in L2
      const int S = p.splits > 1 ? p.splits : 1;
      w.t = cur / S;
      w.ks = cur - w.t * S;
      const TileCoord tc = decode_tile(p, w.t);
      w.g = tc.g;
      w.n = tc.n;
      w.mt = tc.mt;
      w.o0 = tc.pt * p.tile_px;
      w.len = p.tile_px;
      cur += gridDim.x;
    }
    return true;
  }
};

// window iterations (channel chunk c, filter row r; index c * k + r) of a unit
__device__ __forceinline__ void unit_windows(const ConvParams& p, const Work& w, int& w0, int& w1) {
  const int nw = p.cin_chunks * p.k;
  if (p.balanced_units > 0 || p.splits <= 1) {
    w0 = 0;
    w1 = nw;
  } else {
    w0 = w.ks * nw / p.splits;
    w1 = (w.ks + 1) * nw / p.splits;
  }
}

// Branch-free activation: max(x,0) + neg*min(x,0) with neg = 1 (none),
// 0 (ReLU, +0 for negatives) or the channel's PReLU slope (lane = channel).
__device__ __forceinline__ float activate(uint32_t bits, float bias, float neg) {
  const float x = __uint_as_float(bits) + bias;
  return fmaxf(x, 0.f) + neg * fminf(x, 0.f);
}

template <int SUBS>
__global__ void __launch_bounds__(kThreads, 1)
    conv_tc_kernel(const __grid_constant__ ConvMaps maps, const __grid_constant__ ConvParams p) {
  using C = Cfg<SUBS>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* win = smem + C::win;
  uint8_t* wgt = smem + C::wgt;
  uint8_t* stg = smem + C::stg;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::bars);
  uint64_t* win_full = bars;
  uint64_t* win_empty = win_full + C::kWinStages;
  uint64_t* w_full = win_empty + C::kWinStages;
  uint64_t* w_empty = w_full + C::kWgtStages;
  uint64_t* acc_full = w_empty + C::kWgtStages;
  uint64_t* acc_empty = acc_full + C::kAccStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + C::kAccStages);

  const uint32_t warp = warp_id();
  if (threadIdx.x == 0) AVEC_STAMP(0);
  if (warp == 0 && elect_one()) {
    for (int g = 0; g < p.n_groups; ++g) {
      tma_prefetch(&maps.act_big[g]);
      tma_prefetch(&maps.act_small[g]);
      tma_prefetch(&maps.wgt[g]);
      if (p.out_mode == kOutTmaBf16) tma_prefetch(&maps.out[g]);
    }
    for (int i = 0; i < C::kWinStages; ++i) {
      mbar_init(&win_full[i], 1);
      mbar_init(&win_empty[i], 1);
    }
    for (int i = 0; i < C::kWgtStages; ++i) {
      mbar_init(&w_full[i], 1);
      mbar_init(&w_empty[i], 1);
    }
    for (int i = 0; i < C::kAccStages; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], kEpiThreads);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Programmatic dependent launch: everything above overlapped the previous
  // layer's tail; from here on we read its output and overwrite buffers it
  // may still read, so wait for it to complete. The next layer is released
  // only once this CTA has issued its last MMA (see below), so its CTAs do
  // not park on SMs another stream could use.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) AVEC_STAMP(1);

  const int k = p.k;
  const int pad = k / 2;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      const uint64_t keep = policy_evict_last();
      int ws = 0, wst = 0;
      uint32_t wph = 0, wtph = 0;
      const uint32_t win_tx = (C::kTileN + (k > 1 ? 8 : 0)) * 128;
      WorkIter it(p);
      Work tc;
      while (it.next<C::kTileN>(p, tc)) {
        const int row0 = tc.n * p.Hp * p.Wp + (p.P - pad) * (p.Wp + 1) + tc.o0;
        int w0, w1;
        unit_windows(p, tc, w0, w1);
        for (int wi = w0; wi < w1; ++wi) {
          const int c = wi / k, r = wi - c * k;
          const int ch = p.in_c_off + c * 64;
          {
            mbar_wait(&win_empty[ws], wph ^ 1);
            mbar_arrive_expect_tx(&win_full[ws], win_tx);
            uint8_t* wbuf = win + ws * C::kWinBytes;
            const int wr = row0 + r * p.Wp;
#pragma unroll
            for (int b = 0; b < SUBS; ++b)
              tma_load_2d(wbuf + b * kSubN * 128, &maps.act_big[tc.g], &win_full[ws], ch, wr + b * kSubN);
            if (k > 1)
              tma_load_2d(wbuf + C::kTileN * 128, &maps.act_small[tc.g], &win_full[ws], ch,
                          wr + C::kTileN);
            if (++ws == C::kWinStages) { ws = 0; wph ^= 1; }
            for (int s = 0; s < k; ++s) {
              mbar_wait(&w_empty[wst], wtph ^ 1);
              mbar_arrive_expect_tx(&w_full[wst], kWgtBytes);
              tma_load_2d_hint(wgt + wst * kWgtBytes, &maps.wgt[tc.g], &w_full[wst],
                               ((r * k + s) * p.cin_chunks + c) * 64, tc.mt * kTileM, keep);
              if (++wst == C::kWgtStages) { wst = 0; wtph ^= 1; }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      int ws = 0, wst = 0, acc = 0;
      uint32_t wph = 0, wtph = 0, aph = 0;
      const uint32_t win_base = smem_u32(win), wgt_base = smem_u32(wgt);
      WorkIter it(p);
      Work tc;
      while (it.next<C::kTileN>(p, tc)) {
        // MMA N per sub-tile: 256, or the (32-multiple) remainder of a short run
        uint32_t idesc[SUBS];
        int nsub = 0;
#pragma unroll
        for (int sub = 0; sub < SUBS; ++sub) {
          const int n_cols = min(kSubN, tc.len - sub * kSubN);
          idesc[sub] = n_cols > 0 ? idesc_bf16_f32(kTileM, n_cols) : 0u;
          nsub += n_cols > 0;
        }
        mbar_wait(&acc_empty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d0 = tmem + acc * C::kTileN;
        bool first = true;
        int w0, w1;
        unit_windows(p, tc, w0, w1);
        for (int wi = w0; wi < w1; ++wi) {
          {
            mbar_wait(&win_full[ws], wph);
            tc_fence_after();
            if (wi == w0) AVEC_STAMP(4);
            const uint32_t wb = win_base + ws * C::kWinBytes;
            for (int s = 0; s < k; ++s) {
              mbar_wait(&w_full[wst], wtph);
              tc_fence_after();
              // descriptors once per tap; a 32-byte K step adds 2 to each
              const uint64_t ad = desc_sw128(wgt_base + wst * kWgtBytes);
#pragma unroll
              for (int sub = 0; sub < SUBS; ++sub) {
                if (sub < nsub) {
                  const uint64_t bd = desc_sw128(wb + (sub * kSubN + s) * 128);
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk)
                    mma_bf16_ss(d0 + sub * kSubN, ad + 2 * kk, bd + 2 * kk, idesc[sub], (first && kk == 0) ? 0u : 1u);
                }
              }
              first = false;
              mma_commit(&w_empty[wst]);
              if (++wst == C::kWgtStages) { wst = 0; wtph ^= 1; }
            }
            mma_commit(&win_empty[ws]);
            if (++ws == C::kWinStages) { ws = 0; wph ^= 1; }
          }
        }
        mma_commit(&acc_full[acc]);
        if (++acc == C::kAccStages) { acc = 0; aph ^= 1; }
      }
      AVEC_STAMP(5);
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  } else {
    // ------------------------------------------------------------ epilogue
    const uint32_t quad = warp & 3;  // TMEM lane quadrant this warp may touch
    const uint32_t lane = lane_id();
    const int co_local = quad * 32 + lane;
    const bool leader = threadIdx.x == 64;
    int acc = 0, stg_i = 0;
    uint32_t aph = 0;
    WorkIter it(p);
    Work tc;
    while (it.next<C::kTileN>(p, tc)) {
      const ConvGroupParams& g = p.g[tc.g];
      const int co = tc.mt * kTileM + co_local;
      const int cout_m = min(kTileM, g.cout - tc.mt * kTileM);  // channels of this m-tile
      const bool live = co_local < cout_m;
      const float bias = live ? g.bias[co] : 0.f;
      const float neg = g.act == 1 ? 0.f : (live && g.act == 2) ? g.slope[co] : 1.f;
      mbar_wait(&acc_full[acc], aph);
      tc_fence_after();
      if (threadIdx.x == 64) AVEC_STAMP(6);
      if (p.splits > 1) {
        // split-K partial: raw fp32 sums to the workspace, [px][128 channels]
        // per unit, one 128-byte line per pixel and warp (conv_tc_reduce_kernel
        // adds the splits in order and applies the epilogue)
        float* dst = p.ws + (static_cast<size_t>(tc.t) * p.splits + tc.ks) * p.tile_px * kTileM + co_local;
        for (int c0 = 0; c0 < tc.len; c0 += kChunk) {
          uint32_t v[32];
          tmem_ld32(tmem + ((quad * 32) << 16) + acc * C::kTileN + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < kChunk; ++j) dst[static_cast<size_t>(c0 + j) * kTileM] = __uint_as_float(v[j]);
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[acc]);
        if (++acc == C::kAccStages) { acc = 0; aph ^= 1; }
        continue;
      }
      for (int sub = 0; sub < SUBS; ++sub) {
        for (int ch = 0; ch < kSubN / kChunk; ++ch) {
          if (sub * kSubN + ch * kChunk >= tc.len) break;  // uniform across the epilogue warps
          const int o0 = tc.o0 + sub * kSubN + ch * kChunk;
          uint32_t v[32];
          tmem_ld32(tmem + ((quad * 32) << 16) + acc * C::kTileN + sub * kSubN + ch * kChunk, v);
          tmem_ld_wait();
          // pixel (o0 + lane) validity, shared by the warp as a bit mask
          const int pos = o0 + int(lane);
          const int hh = pos / p.Wp;
          const int ww = pos - hh * p.Wp;
          const uint32_t mask = __ballot_sync(0xffffffffu, hh < p.H && ww < p.W);
          if (p.out_mode == kOutTmaBf16) {
            uint8_t* buf = stg + (stg_i % C::kStgBufs) * kStageBytes;
            // the store that last used `buf` must have read it
            if (leader) {
              if (C::kStgBufs == 2) bulk_wait_read<1>();
              else bulk_wait_read<0>();
            }
            named_bar_sync(kEpiBar, kEpiThreads);
            {
              // channels past cout (zero weights and bias) store zeros: a
              // 96-channel layer's second box ends 32 channels into the
              // destination's next slice, which a later layer overwrites
              uint8_t* half = buf + (co_local >> 6) * (kChunk * 128);
              const uint32_t cb = (co_local & 63) * 2;
#pragma unroll
              for (int j = 0; j < kChunk; ++j) {
                const float x = live && ((mask >> j) & 1u) ? activate(v[j], bias, neg) : 0.f;
                *reinterpret_cast<__nv_bfloat16*>(half + j * 128 + ((((cb >> 4) ^ (j & 7)) << 4) | (cb & 15))) =
                    __float2bfloat16_rn(x);
              }
            }
            fence_proxy_async_smem();
            named_bar_sync(kEpiBar, kEpiThreads);
            if (leader) {
              const int row = p.P * p.Wp + p.P + o0;
              const int c0 = g.out_c_off + tc.mt * kTileM;
              tma_store_3d(&maps.out[tc.g], buf, c0, row, tc.n);
              if (cout_m > 64) tma_store_3d(&maps.out[tc.g], buf + kChunk * 128, c0 + 64, row, tc.n);
              bulk_commit();
            }
            ++stg_i;
          } else if (live && mask) {
            int h = o0 / p.Wp;
            int w = o0 - h * p.Wp;
#pragma unroll
            for (int j = 0; j < kChunk; ++j) {
              if ((mask >> j) & 1u) {
                const float x = activate(v[j], bias, neg);
                if (p.out_mode == kOutNchwF32) {
                  static_cast<float*>(g.out)[((static_cast<size_t>(tc.n) * g.out_c_stride + g.out_c_off + co) *
                                                  p.H + h) * p.W + w] = x;
                } else {
                  static_cast<__nv_bfloat16*>(g.out)[(static_cast<size_t>(tc.n * p.Hp + h + p.P) * p.Wp + w + p.P) *
                                                         g.out_c_stride + g.out_c_off + co] =
                      __float2bfloat16_rn(x);
                }
              }
              if (++w == p.Wp) { w = 0; ++h; }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[acc]);
      if (++acc == C::kAccStages) { acc = 0; aph ^= 1; }
    }
    if (leader) AVEC_STAMP(7);
    if (leader) bulk_wait<0>();
    if (leader) AVEC_STAMP(8);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
  if (threadIdx.x == 0) AVEC_STAMP(9);
}

// Split-K fix-up: out = act(sum_{s in split order} partial_s + bias), zero
// outside the image, bf16 into the padded-flat NHWC destination. Block =
// 8 positions x 32 threads of 4 channels: a warp reads one 512-byte line per
// split and writes 256 contiguous bytes; the split loop issues 4 loads ahead
// of its (in-order) adds so the L2 latency is not paid per split.
__global__ void __launch_bounds__(256) conv_tc_reduce_kernel(const __grid_constant__ ConvParams p) {
  const int t = blockIdx.x;
  const int px = blockIdx.y * 8 + int(threadIdx.x >> 5);
  const int cq = int(threadIdx.x & 31) * 4;
  if (px >= p.tile_px) return;
  const TileCoord tc = decode_tile(p, t);
  const ConvGroupParams& g = p.g[tc.g];
  const int o = tc.pt * p.tile_px + px;
  const int row = p.P * p.Wp + p.P + o;  // position inside the padded image
  if (row >= p.Hp * p.Wp) return;        // past the image's buffer (clipped like the TMA store)
  const int hh = o / p.Wp, ww = o - hh * p.Wp;
  const bool valid = hh < p.H && ww < p.W;
  const int cout_m = min(kTileM, g.cout - tc.mt * kTileM);
  if (cq >= cout_m) return;
  const size_t split_stride = static_cast<size_t>(p.tile_px) * kTileM;
  const float* src = p.ws + (static_cast<size_t>(t) * p.splits * p.tile_px + px) * kTileM + cq;
  float4 acc = __ldcg(reinterpret_cast<const float4*>(src));
  int s = 1;
  for (; s + 4 <= p.splits; s += 4) {
    const float4 a = __ldcg(reinterpret_cast<const float4*>(src + s * split_stride));
    const float4 b = __ldcg(reinterpret_cast<const float4*>(src + (s + 1) * split_stride));
    const float4 c = __ldcg(reinterpret_cast<const float4*>(src + (s + 2) * split_stride));
    const float4 d = __ldcg(reinterpret_cast<const float4*>(src + (s + 3) * split_stride));
    acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
    acc.x += b.x; acc.y += b.y; acc.z += b.z; acc.w += b.w;
    acc.x += c.x; acc.y += c.y; acc.z += c.z; acc.w += c.w;
    acc.x += d.x; acc.y += d.y; acc.z += d.z; acc.w += d.w;
  }
  for (; s < p.splits; ++s) {
    const float4 a = __ldcg(reinterpret_cast<const float4*>(src + s * split_stride));
    acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
  }
  const float v[4] = {acc.x, acc.y, acc.z, acc.w};
  __align__(8) __nv_bfloat16 out[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = cq + i;
    float x = 0.f;
    if (valid && c < cout_m) {
      const int co = tc.mt * kTileM + c;
      const float neg = g.act == 1 ? 0.f : g.act == 2 ? g.slope[co] : 1.f;
      x = activate(__float_as_uint(v[i]), g.bias[co], neg);
    }
    out[i] = __float2bfloat16_rn(x);
  }
  __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(g.out) +
                       (static_cast<size_t>(tc.n) * p.Hp * p.Wp + row) * g.out_c_stride + g.out_c_off +
                       tc.mt * kTileM + cq;
  if (cq + 4 <= cout_m && ((g.out_c_stride | g.out_c_off) & 3) == 0)
    *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(out);
  else
    for (int i = 0; i < 4 && cq + i < cout_m; ++i) dst[i] = out[i];
}

template <int SUBS>
constexpr size_t smem_bytes() {
  return Cfg<SUBS>::total + 1024;
}

}  // namespace

#ifdef AVEC_TRACE
void conv_tc_trace(int on, cudaStream_t st) {
  check_cuda(cudaMemcpyToSymbolAsync(g_trace_on, &on, sizeof on, 0, cudaMemcpyHostToDevice, st), "trace arm");
  check_cuda(cudaStreamSynchronize(st), "trace arm");
}
int conv_tc_trace_dump(unsigned long long* host, int n) {
  return cudaMemcpyFromSymbol(host, g_trace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 5;
}
#endif

bool pdl_enabled() {
  static const bool on = [] {
    // Off by default: measured +1% on one stream but -22% with two slots in
    // flight (dependents park on SMs the other stream needs). AVEC_PDL=1 enables.
    const char* e = std::getenv("AVEC_PDL");
    return e && e[0] == '1';
  }();
  return on;
}

void conv_configure() {
  check_cuda(cudaFuncSetAttribute(conv_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem_bytes<1>())),
             "conv smem attribute");
  check_cuda(cudaFuncSetAttribute(conv_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem_bytes<2>())),
             "conv smem attribute");
}

int conv_tc_splits(int tiles, int windows, int sm_count) {
  static const bool on = [] {
    const char* e = std::getenv("AVEC_SPLITK");
    return !(e && e[0] == '0');
  }();
  static const int cap = [] {
    const char* e = std::getenv("AVEC_SPLITK_MAX");
    return e ? std::atoi(e) : 1 << 20;
  }();
  if (!on || tiles <= 0 || 2 * tiles > sm_count) return 1;
  int s = sm_count / tiles;
  if (s > windows) s = windows;
  return s < cap ? s : (cap > 1 ? cap : 1);
}

void launch_conv_tc(const ConvMaps& maps, const ConvParams& p, int sm_count, cudaStream_t stream) {
  if (p.splits > 1 && (p.balanced_units > 0 || !p.ws || p.out_mode == kOutNchwF32))
    fail(AVEC_ERR_UNSUPPORTED, "conv_tc split-K needs regular tiles, a workspace and a bf16 destination");
  const int work = p.balanced_units > 0 ? p.balanced_units : p.total_tiles * (p.splits > 1 ? p.splits : 1);
  const int grid = work < sm_count ? work : sm_count;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = p.subs == 1 ? smem_bytes<1>() : smem_bytes<2>();
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  if (p.subs == 1)
    check_cuda(cudaLaunchKernelEx(&cfg, conv_tc_kernel<1>, maps, p), "conv_tc launch");
  else
    check_cuda(cudaLaunchKernelEx(&cfg, conv_tc_kernel<2>, maps, p), "conv_tc launch");
  if (p.splits > 1) {
    conv_tc_reduce_kernel<<<dim3(p.total_tiles, (p.tile_px + 7) / 8), 256, 0, stream>>>(p);
    check_cuda(cudaGetLastError(), "conv_tc reduce launch");
  }
}

}  // namespace avec
