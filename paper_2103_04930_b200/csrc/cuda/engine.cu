// B200 engine: device handle table, execution slots with pinned double-buffered
// staging, the segment-mean (reference MockPose) path and the pose-net plan
// executor (tcgen05 convolutions captured into a CUDA graph per shape).
//
// Reference counterparts: MockPoseBackend::register_model / forward
// (proj/src/backend.cpp:69-96) and the dispatch call site in
// Server::dispatch_loop (proj/src/server.cpp:84-111).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "engine_impl.hpp"
#include "trace.cuh"

namespace avec {

// ------------------------------------------------------------------ memory
DevMem::~DevMem() { reset(); }
void DevMem::reset() {
  if (p) {
    int cur = -1;
    cudaGetDevice(&cur);
    if (device >= 0 && cur != device) cudaSetDevice(device);
    cudaFree(p);
    if (device >= 0 && cur != device) cudaSetDevice(cur);
  }
  p = nullptr;
  bytes = 0;
}
void DevMem::ensure(size_t n, int dev) {
  if (n <= bytes && p) return;
  reset();
  check_cuda(cudaMalloc(&p, n), "cudaMalloc");
  bytes = n;
  device = dev;
}

PinnedMem::~PinnedMem() {
  if (p) cudaFreeHost(p);
}
void PinnedMem::ensure(size_t n) {
  if (n <= bytes && p) return;
  if (p) cudaFreeHost(p);
  p = nullptr;
  check_cuda(cudaHostAlloc(&p, n, cudaHostAllocPortable), "cudaHostAlloc");
  bytes = n;
}

Plan::~Plan() {
  if (graph) cudaGraphExecDestroy(graph);
}

namespace {

constexpr size_t kStageChunk = size_t(8) << 20;  // pinned staging chunk (bytes)

uint16_t bf16_bits(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return uint16_t((u >> 16) | ((u & 0xffff) ? 0x40 : 0));
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}
// fp32 -> tf32 bit pattern, round to nearest, ties away from zero (= cvt.rna.tf32.f32)
float tf32_value(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}
float bf16_value(float x) {
  uint32_t u = uint32_t(bf16_bits(x)) << 16;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// ---- TMA descriptors (driver entry point, no -lcuda link) ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    check_cuda(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000,
                                                cudaEnableDefault, &q),
               "cuTensorMapEncodeTiled entry point");
    if (!f || q != cudaDriverEntryPointSuccess) fail(AVEC_ERR_CUDA, "cuTensorMapEncodeTiled missing");
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// 2D bf16 [rows][cols] row-major, box {box_cols, box_rows}; the swizzle span
// equals the box row (64 cols: 128 B, 32 cols: 64 B, 16 cols: 32 B)
CUtensorMap make_map_2d(const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows, uint32_t box_cols = 64) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           box_cols == 16   ? CU_TENSOR_MAP_SWIZZLE_32B
                           : box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                            : CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(AVEC_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

// 2D fp32 [rows][cols] row-major, box {32 cols = 128 B, box_rows}, 128-byte swizzle
CUtensorMap make_map_2d_f32(const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(AVEC_ERR_CUDA, "cuTensorMapEncodeTiled (f32) failed: " + std::to_string(int(r)));
  return m;
}

// 3D bf16 [n][rows][cols] (the padded-flat buffer seen per image), box {64, 32, 1}
// [32 rows][box_c channels] store boxes; the swizzle span equals the box row
// (64 ch: 128 B, 32 ch: 64 B, 16 ch: 32 B, 8 ch: none)
CUtensorMap make_map_3d_store(const void* base, uint64_t cols, uint64_t rows, uint64_t n, uint32_t box_c = 64) {
  CUtensorMap m;
  cuuint64_t dims[3] = {cols, rows, n};
  cuuint64_t strides[2] = {cols * 2, rows * cols * 2};
  cuuint32_t box[3] = {box_c, 32, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           box_c == 64   ? CU_TENSOR_MAP_SWIZZLE_128B
                           : box_c == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                           : box_c == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                         : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(AVEC_ERR_CUDA, "cuTensorMapEncodeTiled (store) failed: " + std::to_string(int(r)));
  return m;
}

// [N][Hp][Wp][C] with [16 px][64 ch] boxes along one padded row (the fused
// pool's output rows; boxes are clipped at the row end)
CUtensorMap make_map_4d_store(const void* base, uint64_t C, uint64_t Wp, uint64_t Hp, uint64_t n,
                              uint32_t box_px = 16) {
  CUtensorMap m;
  cuuint64_t dims[4] = {C, Wp, Hp, n};
  cuuint64_t strides[3] = {C * 2, Wp * C * 2, Hp * Wp * C * 2};
  cuuint32_t box[4] = {64, box_px, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
                           es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(AVEC_ERR_CUDA, "cuTensorMapEncodeTiled (4d store) failed: " + std::to_string(int(r)));
  return m;
}

// fp32 frames [N*3][H][W] (the wire layout), box {132 columns, 6 rows, 3 channels}
CUtensorMap make_map_frames(const void* base, uint64_t W, uint64_t H, uint64_t planes) {
  CUtensorMap m;
  cuuint64_t dims[3] = {W, H, planes};
  cuuint64_t strides[2] = {W * 4, H * W * 4};
  cuuint32_t box[3] = {132, 6, 3};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(AVEC_ERR_CUDA, "cuTensorMapEncodeTiled (frames) failed: " + std::to_string(int(r)));
  return m;
}

int round_up(int x, int m) { return (x + m - 1) / m * m; }

// ------------------------------------------------------------------ slots
struct SlotLease {
  avec_ctx* ctx;
  int idx;
  explicit SlotLease(avec_ctx* c) : ctx(c), idx(-1) {
    std::unique_lock<std::mutex> lk(ctx->slot_m);
    ctx->slot_cv.wait(lk, [&] {
      for (size_t i = 0; i < ctx->slot_busy.size(); ++i)
        if (!ctx->slot_busy[i]) return true;
      return false;
    });
    // round-robin over free slots: back-to-back asynchronous calls on
    // alternating streams land on alternating slots and overlap
    const size_t n = ctx->slot_busy.size();
    for (size_t k = 0; k < n; ++k) {
      const size_t i = (ctx->next_slot + k) % n;
      if (!ctx->slot_busy[i]) {
        idx = int(i);
        ctx->slot_busy[i] = true;
        ctx->next_slot = (i + 1) % n;
        break;
      }
    }
  }
  ~SlotLease() {
    {
      std::lock_guard<std::mutex> lk(ctx->slot_m);
      ctx->slot_busy[idx] = false;
    }
    ctx->slot_cv.notify_one();
  }
  Slot* slot() const { return ctx->slots[idx].get(); }
  // order this use of the slot after its previous asynchronous forward
  void after_pending(cudaStream_t st) const {
    Slot* s = slot();
    if (!s->pending) return;
    if (st) check_cuda(cudaStreamWaitEvent(st, s->done, 0), "wait slot");
    else check_cuda(cudaEventSynchronize(s->done), "wait slot");
    s->pending = false;
  }
};

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// H2D through the slot's two pinned chunks: the CPU fills chunk i+1 while the
// copy engine drains chunk i.
void stage_h2d(Slot* s, void* d_dst, const void* h_src, size_t bytes) {
  if (is_pinned(h_src)) {
    check_cuda(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, s->stream), "H2D");
    return;
  }
  size_t off = 0;
  int i = 0;
  while (off < bytes) {
    const size_t len = std::min(kStageChunk, bytes - off);
    const int b = i & 1;
    check_cuda(cudaEventSynchronize(s->stage_ev[b]), "stage wait");
    std::memcpy(s->stage[b].p, static_cast<const char*>(h_src) + off, len);
    check_cuda(cudaMemcpyAsync(static_cast<char*>(d_dst) + off, s->stage[b].p, len,
                               cudaMemcpyHostToDevice, s->stream),
               "H2D chunk");
    check_cuda(cudaEventRecord(s->stage_ev[b], s->stream), "stage record");
    off += len;
    ++i;
  }
}

// D2H mirror: chunk i+1 is in flight while the CPU copies chunk i out.
void stage_d2h(Slot* s, void* h_dst, const void* d_src, size_t bytes) {
  if (is_pinned(h_dst)) {
    check_cuda(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, s->stream), "D2H");
    check_cuda(cudaEventRecord(s->ev1, s->stream), "ev1");
    check_cuda(cudaStreamSynchronize(s->stream), "D2H sync");
    return;
  }
  const size_t n = (bytes + kStageChunk - 1) / kStageChunk;
  auto issue = [&](size_t i) {
    const size_t off = i * kStageChunk, len = std::min(kStageChunk, bytes - off);
    check_cuda(cudaMemcpyAsync(s->stage[i & 1].p, static_cast<const char*>(d_src) + off, len,
                               cudaMemcpyDeviceToHost, s->stream),
               "D2H chunk");
    check_cuda(cudaEventRecord(s->stage_ev[i & 1], s->stream), "stage record");
  };
  if (n) issue(0);
  for (size_t i = 0; i < n; ++i) {
    if (i + 1 < n) issue(i + 1);
    if (i + 1 == n) check_cuda(cudaEventRecord(s->ev1, s->stream), "ev1");
    check_cuda(cudaEventSynchronize(s->stage_ev[i & 1]), "stage wait");
    const size_t off = i * kStageChunk, len = std::min(kStageChunk, bytes - off);
    std::memcpy(static_cast<char*>(h_dst) + off, s->stage[i & 1].p, len);
  }
  check_cuda(cudaStreamSynchronize(s->stream), "D2H sync");
}

// ------------------------------------------------------------------ pose net
std::shared_ptr<PoseNet> upload_posenet(int device, PoseFamily fam, const float* weights) {
  auto net = std::make_shared<PoseNet>();
  net->fam = std::move(fam);
  const PoseFamily& f = net->fam;
  // per layer: bf16 W [cout_pad][k*k][cin_pad] + fp32 bias, 1 KB aligned
  std::vector<size_t> w_off(f.convs.size()), b_off(f.convs.size());
  size_t total = 0;
  auto take = [&](size_t bytes) {
    size_t o = total;
    total += (bytes + 1023) / 1024 * 1024;
    return o;
  };
  net->layers.resize(f.convs.size());
  for (size_t i = 0; i < f.convs.size(); ++i) {
    ConvLayerDev& L = net->layers[i];
    L.def = f.convs[i];
    // the 3-channel first layer: one 64-wide K row of its 27 taps (conv_first.cu)
    L.exec_k = i == 0 ? 1 : L.def.k;
    L.cin_pad = i == 0 ? 64 : L.def.cin_pad ? L.def.cin_pad : round_up(L.def.cin, 64);
    L.cout_pad = round_up(L.def.cout, 128);
    w_off[i] = take(size_t(L.cout_pad) * L.exec_k * L.exec_k * L.cin_pad * 2);
    b_off[i] = take(size_t(L.cout_pad) * 4 * 2);  // bias, then PReLU slopes
  }
  // "input tf32": the first layer's weights again, as tf32 [cout_pad][32]
  const size_t tf32_off = f.input_tf32 ? take(size_t(net->layers[0].cout_pad) * 32 * 4) : 0;
  std::vector<uint8_t> host(total, 0);
  const float* src = weights;
  for (size_t i = 0; i < f.convs.size(); ++i) {
    ConvLayerDev& L = net->layers[i];
    const ConvDef& d = L.def;
    const int k = d.k;
    if (i == 0) {
      if (d.cin != 3 || k != 3) fail(AVEC_ERR_INVALID_MODEL, "first layer must be 3x3 over 3 channels");
      uint16_t* w = reinterpret_cast<uint16_t*>(host.data() + w_off[i]);
      for (int co = 0; co < d.cout; ++co)
        for (int t = 0; t < 27; ++t)  // t = ci*9 + r*3 + s, the im2col channel order
          w[size_t(co) * 64 + t] = bf16_bits(src[size_t(co) * 27 + t]);
      if (f.input_tf32) {
        float* wt = reinterpret_cast<float*>(host.data() + tf32_off);
        for (int co = 0; co < d.cout; ++co)
          for (int t = 0; t < 27; ++t) wt[size_t(co) * 32 + t] = tf32_value(src[size_t(co) * 27 + t]);
      }
      src += size_t(d.cout) * 27;
    } else {
      // Caffe input channel ci -> internal channel of the layer's input window
      if (!d.cin_map.empty() && int(d.cin_map.size()) != d.cin)
        fail(AVEC_ERR_INVALID_MODEL, "bad input channel map for " + d.name);
      uint16_t* w = reinterpret_cast<uint16_t*>(host.data() + w_off[i]);
      for (int co = 0; co < d.cout; ++co)
        for (int ci = 0; ci < d.cin; ++ci) {
          const int cint = d.cin_map.empty() ? ci : d.cin_map[ci];
          if (cint < 0 || cint >= L.cin_pad) fail(AVEC_ERR_INVALID_MODEL, "channel map out of range");
          for (int r = 0; r < k; ++r)
            for (int s = 0; s < k; ++s)
              w[(size_t(co) * k * k + r * k + s) * L.cin_pad + cint] =
                  bf16_bits(src[((size_t(co) * d.cin + ci) * k + r) * k + s]);
        }
      src += size_t(d.cout) * d.cin * k * k;
    }
    std::memcpy(host.data() + b_off[i], src, d.cout * 4);
    if (i == 0) {
      // conv12 folds conv1_1's bias into its MMA: im2col taps 27 and 28 are
      // 1.0, weights there bias = hi + lo (two bf16 parts, 2^-17 relative);
      // conv_first's im2col keeps them 0
      uint16_t* w = reinterpret_cast<uint16_t*>(host.data() + w_off[i]);
      for (int co = 0; co < d.cout; ++co) {
        w[size_t(co) * 64 + 27] = bf16_bits(src[co]);
        w[size_t(co) * 64 + 28] = bf16_bits(src[co] - bf16_value(src[co]));
      }
    }
    src += d.cout;
    if (d.act == kActPrelu) {
      std::memcpy(host.data() + b_off[i] + size_t(L.cout_pad) * 4, src, d.cout * 4);
      src += d.cout;
    }
  }
  check_cuda(cudaSetDevice(device), "cudaSetDevice");
  net->mem.ensure(total, device);
  // on a private stream, synchronised: a pageable cudaMemcpy may return before
  // the DMA lands, and the slots' non-blocking streams do not order after the
  // legacy stream
  cudaStream_t up = nullptr;
  check_cuda(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking), "upload stream");
  cudaError_t e = cudaMemcpyAsync(net->mem.p, host.data(), total, cudaMemcpyHostToDevice, up);
  if (e == cudaSuccess) e = cudaStreamSynchronize(up);
  cudaStreamDestroy(up);
  check_cuda(e, "weights H2D");
  char* base = net->mem.as<char>();
  for (size_t i = 0; i < f.convs.size(); ++i) {
    net->layers[i].w = base + w_off[i];
    net->layers[i].bias = reinterpret_cast<float*>(base + b_off[i]);
    net->layers[i].slope = reinterpret_cast<float*>(base + b_off[i]) + net->layers[i].cout_pad;
  }
  if (f.input_tf32) net->layers[0].w_tf32 = reinterpret_cast<float*>(base + tf32_off);
  return net;
}

// CTA pairs: M = 256 MMAs whose B half is read once per SM, relieving the
// shared-memory operand path (tests/native/tc2_probe.cu: N = 96 runs 49
// instead of 56 cycles). Measured per layer class: a win for 3x3 convs with
// K >= 1152 and N >= 96 (C5 dense blocks -11..-22%, VGG conv2_2/conv3_x
// -6..-10%), a loss for the short-K ones (conv2_1 from 64 channels, the 1x1
// heads: +8..+18%). AVEC_PM2: 0 off, 1 that rule (default), 2 every
// pixel-major layer.
int pm_ncta(int pm_n, int exec_k, int cin_chunks) {
  static const int pm2 = [] {
    const char* e = std::getenv("AVEC_PM2");
    return e ? std::atoi(e) : 1;
  }();
  const bool long_k = exec_k == 3 && cin_chunks >= 2;
  return (pm2 == 2 || (pm2 == 1 && pm_n >= 96 && long_k)) ? 2 : 1;
}

struct PlanBuilder {
  Plan& plan;
  const PoseNet& net;
  int device;
  cudaStream_t stream;  // the building slot's stream

  int sm_count() const {
    int n = 0;
    check_cuda(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device), "SM count");
    return n;
  }

  int buffer(int level, int C) {
    const Geometry& g = plan.geo[level];
    auto m = std::make_unique<DevMem>();
    const size_t bytes = size_t(plan.n) * g.Hp() * g.Wp() * C * 2;
    m->ensure(bytes, device);
    // zero border + pad channels, on the slot stream (get_plan synchronises it
    // before the plan is used on any stream)
    check_cuda(cudaMemsetAsync(m->p, 0, bytes, stream), "zero activation buffer");
    plan.bufs.push_back(std::move(m));
    plan.buf_level.push_back(level);
    plan.buf_c.push_back(C);
    return int(plan.bufs.size()) - 1;
  }

  TensorView view(int buf, int c_off, int c) {
    TensorView v;
    v.buf = buf;
    v.level = buf >= 0 ? plan.buf_level[buf] : 3;
    v.c_stride = buf >= 0 ? plan.buf_c[buf] : net.fam.out_channels();
    v.c_off = c_off;
    v.c = c;
    return v;
  }

  void record_io(int layer, TensorView in, TensorView out) {
    plan.layer_in[layer] = in;
    plan.layer_out[layer] = out;
  }

  // conv1_1 fused with the input conversion (conv_first.cu): reads the fp32
  // frames, writes the 64-channel level-0 activation `out`
  void first(int layer, TensorView out) {
    const ConvLayerDev& L = net.layers[layer];
    if (L.def.cout > 64 || out.level != 0 || out.c_off % 8 != 0)
      fail(AVEC_ERR_UNSUPPORTED, "first layer must write <= 64 channels at level 0");
    PlanOp op;
    op.kind = PlanOp::kFirst;
    op.layers[0] = layer;
    ConvParams& p = op.cp;
    const Geometry& gi = plan.geo[0];
    p.k = 3;
    p.n_images = plan.n;
    p.H = gi.H;
    p.W = gi.W;
    p.Hp = gi.Hp();
    p.Wp = gi.Wp();
    p.P = gi.P;
    p.n_groups = 1;
    p.tiles_per_image = (p.H * p.Wp + 127) / 128;
    p.total_tiles = p.n_images * p.tiles_per_image;
    ConvGroupParams& gp = p.g[0];
    gp.bias = L.bias;
    gp.slope = L.slope;
    gp.act = L.def.act;
    gp.cout = L.def.cout;
    gp.out = plan.bufs[out.buf]->p;
    gp.out_c_off = out.c_off;
    gp.out_c_stride = out.c_stride;
    if (L.w_tf32) {  // "input tf32": kind::tf32 MMAs on fp32 taps and weights
      p.tf32 = 1;
      op.maps.wgt[0] = make_map_2d_f32(L.w_tf32, 32, L.cout_pad, 64);
    } else {
      op.maps.wgt[0] = make_map_2d(L.w, 64, L.cout_pad, 64);
    }
    op.maps.out[0] = make_map_3d_store(plan.bufs[out.buf]->p, plan.buf_c[out.buf], uint64_t(gi.Hp()) * gi.Wp(),
                                       plan.n);
    TensorView in;
    in.buf = -2;
    in.c = 3;
    record_io(layer, in, out);  // parity hook shows the layer its real 3-channel input
    plan.ops.push_back(op);
  }

  // conv1_1 + conv1_2 + pool1 as one kernel (conv12.cu) writing the pooled
  // level-1 buffer; false when the shapes do not allow it (AVEC_CONV12=0 disables)
  bool conv12(int l1, int l2, int pooled) {
    static const bool on = [] {
      const char* e = std::getenv("AVEC_CONV12");
      return !(e && e[0] == '0');
    }();
    const ConvLayerDev& A = net.layers[l1];
    const ConvLayerDev& B = net.layers[l2];
    const Geometry& g0 = plan.geo[0];
    // ("input tf32" nets take the conv_first path: conv12 is bf16-only)
    if (!on || net.fam.input_tf32 || A.def.cin != 3 || A.def.k != 3 || A.def.cout != 64 || A.def.act != kActRelu ||
        B.exec_k != 3 ||
        B.def.cin != 64 || B.def.cout != 64 || B.def.act != kActRelu || g0.H % 2 || g0.W % 4 ||
        plan.buf_c[pooled] != 64)
      return false;
    PlanOp op;
    op.kind = PlanOp::kConv12;
    op.layers[0] = l2;
    op.head_l6[0] = l1;
    ConvParams& p = op.cp;
    p.k = 3;
    p.n_images = plan.n;
    p.H = g0.H;
    p.W = g0.W;
    p.Hp = g0.Hp();
    p.Wp = g0.Wp();
    p.P = g0.P;
    p.n_groups = 1;
    p.pool = 1;
    p.pool_P = plan.geo[1].P;
    p.col_blocks = (p.W + conv12_tile_cols() - 1) / conv12_tile_cols();
    p.tiles_per_image = p.H / 2 * p.col_blocks;
    p.total_tiles = p.n_images * p.tiles_per_image;
    ConvGroupParams& g2 = p.g[0];
    g2.bias = B.bias;
    g2.slope = B.slope;
    g2.act = B.def.act;
    g2.cout = 64;
    g2.out = plan.bufs[pooled]->p;
    g2.out_c_off = 0;
    g2.out_c_stride = 64;
    ConvGroupParams& g1 = p.g[1];
    g1.bias = A.bias;
    g1.slope = A.slope;
    g1.act = A.def.act;
    g1.cout = 64;
    op.maps.act_big[0] = make_map_frames(plan.in.p, uint64_t(p.W), uint64_t(p.H), uint64_t(plan.n) * 3);
    op.maps.wgt[0] = make_map_2d(B.w, 9 * 64, B.cout_pad, 64, conv12_wgt_k());  // [64 cout][K chunk]
    op.maps.wgt[1] = make_map_2d(A.w, 64, A.cout_pad, 64, 32);  // [64 cout][32 K] SW64
    const Geometry& g1g = plan.geo[1];
    op.maps.out_pool[0] = make_map_4d_store(plan.bufs[pooled]->p, 64, g1g.Wp(), g1g.Hp(), plan.n, 16);
    op.maps.out_pool[1] = make_map_4d_store(plan.bufs[pooled]->p, 64, g1g.Wp(), g1g.Hp(), plan.n, 15);
    TensorView in;
    in.buf = -2;
    in.c = 3;
    record_io(l2, in, view(pooled, 0, 64));  // conv1_2's parity view: the frame in, pooled out
    plan.layer_fusion[l1] = 2;
    plan.layer_fusion[l2] = 3;
    plan.layer_in_from[l2] = l1;
    plan.ops.push_back(op);
    return true;
  }

  // A 3x3 ReLU conv writing all of a 64/128-channel buffer that only a 2x2
  // max-pool reads: run it with the pool fused into its epilogue (conv_pm.cu
  // POOL tiles) and skip the full-resolution tensor. AVEC_POOLFUSE=0 disables.
  bool pool_fusable(int layer, int level) const {
    static const bool on = [] {
      const char* e = std::getenv("AVEC_POOLFUSE");
      return !(e && e[0] == '0');
    }();
    const ConvLayerDev& L = net.layers[layer];
    if (!on || L.exec_k != 3 || L.def.act != kActRelu || (L.def.cout != 64 && L.def.cout != 128)) return false;
    const Geometry& g = plan.geo[level];
    const int ncta = pm_ncta(L.def.cout, L.exec_k, L.cin_pad / 64);
    return g.H % (2 * ncta) == 0 && g.W % 2 == 0;
  }

  // conv `layer` from `in`, then 2x2/2 max-pool into buffer `pooled` (level + 1)
  void conv_pool(int layer, TensorView in, int pooled) {
    const int level = in.level;
    const int cout = net.layers[layer].def.cout;
    if (pool_fusable(layer, level)) {
      conv({layer}, {in}, {view(pooled, 0, cout)}, true);
      plan.layer_fusion[layer] = 1;
    } else {
      const int full = buffer(level, cout);
      conv({layer}, {in}, {view(full, 0, cout)});
      pool(full, pooled);
    }
  }

  // Mconv6 -> Mconv7 of each branch as one fused launch (conv_head.cu) when the
  // shapes allow; otherwise two conv launches through the `mid` buffers.
  // outs2: optional fp32 NCHW second destinations (BODY_25's last PAF stage).
  // AVEC_HEADFUSE=0 disables.
  void head(std::vector<int> l6, std::vector<int> l7, std::vector<TensorView> in, std::vector<TensorView> mid,
            std::vector<TensorView> out, std::vector<TensorView> out2 = {}) {
    static const bool on = [] {
      const char* e = std::getenv("AVEC_HEADFUSE");
      return !(e && e[0] == '0');
    }();
    bool ok = on;
    for (size_t g = 0; g < l6.size(); ++g) {
      const ConvLayerDev& A = net.layers[l6[g]];
      const ConvLayerDev& B = net.layers[l7[g]];
      const int c6 = A.def.cout;
      ok = ok && A.exec_k == 1 && B.exec_k == 1 && (c6 == 128 || c6 == 256 || c6 == 512) && B.def.cout <= 64 &&
           B.def.cin == c6 && B.def.cin_map.empty() && B.cin_pad == c6 && B.def.act == kActNone &&
           in[g].level == 3;
      const TensorView& o = out[g];
      ok = ok && (o.buf == -1 || (o.c_off % 8 == 0 && o.c_off + round_up(B.def.cout, 8) <= o.c_stride &&
                                  o.level == in[g].level));
      if (!out2.empty()) ok = ok && out2[g].buf == -1 && o.buf != -1;
    }
    if (!ok) {
      std::vector<int> a(l6), b(l7);
      if (a.size() == 1) {
        conv({a[0]}, {in[0]}, {mid[0]});
        conv({b[0]}, {mid[0]}, {out[0]});
        if (!out2.empty()) conv({b[0]}, {mid[0]}, {out2[0]});
      } else {
        conv({a[0], a[1]}, {in[0], in[1]}, {mid[0], mid[1]});
        conv({b[0], b[1]}, {mid[0], mid[1]}, {out[0], out[1]});
      }
      return;
    }
    PlanOp op;
    op.kind = PlanOp::kHead;
    HeadParams& p = op.hp;
    const Geometry& gi = plan.geo[in[0].level];
    const ConvLayerDev& A0 = net.layers[l6[0]];
    p.n_images = plan.n;
    p.H = gi.H;
    p.W = gi.W;
    p.Hp = gi.Hp();
    p.Wp = gi.Wp();
    p.P = gi.P;
    p.in_c_off = in[0].c_off;
    p.cin_chunks = A0.cin_pad / 64;
    p.nb = 128;
    p.blocks = A0.def.cout / p.nb;
    p.tiles_per_image = (p.H * p.Wp + 127) / 128;
    p.n_groups = int(l6.size());
    // CTA pairs (conv_head2) where several c6 blocks would re-read the input
    // and the input tile fits in smem; AVEC_HEAD2=0 disables
    static const bool pair_on = [] {
      const char* e = std::getenv("AVEC_HEAD2");
      return !(e && e[0] == '0');
    }();
    p.ncta = pair_on && p.blocks >= 2 && p.cin_chunks <= conv_head_pair_max_chunks() ? 2 : 1;
    if (p.ncta == 2) p.tiles_per_image = (p.tiles_per_image + 1) / 2;  // pairs of 128-pixel tiles
    p.total_tiles = p.n_groups * p.n_images * p.tiles_per_image;
    const uint64_t rows = uint64_t(plan.n) * gi.Hp() * gi.Wp();
    for (size_t g = 0; g < l6.size(); ++g) {
      const ConvLayerDev& A = net.layers[l6[g]];
      const ConvLayerDev& B = net.layers[l7[g]];
      if (A.cin_pad != A0.cin_pad || A.def.cout != A0.def.cout || in[g].c_off != p.in_c_off)
        fail(AVEC_ERR_INVALID_MODEL, "grouped head layers differ in shape");
      HeadGroup& hg = p.g[g];
      hg.bias6 = A.bias;
      hg.slope6 = A.slope;
      hg.act6 = A.def.act;
      hg.bias7 = B.bias;
      hg.c7 = B.def.cout;
      const TensorView& o = out[g];
      hg.out = o.buf == -1 ? static_cast<void*>(plan.out.p) : plan.bufs[o.buf]->p;
      hg.out_mode = o.buf == -1 ? kOutNchwF32 : kOutTmaBf16;
      hg.out_c_off = o.c_off;
      hg.out_c_stride = o.c_stride;
      hg.out2 = out2.empty() ? nullptr : plan.out.as<float>();
      hg.out2_c_off = out2.empty() ? 0 : out2[g].c_off;
      hg.out2_c_stride = out2.empty() ? 0 : out2[g].c_stride;
      const int ib = in[g].buf;
      op.hm.x[g] = make_map_2d(plan.bufs[ib]->p, plan.buf_c[ib], rows, 128);
      // the pair kernel loads half a block per CTA: 64 of W6's 128 rows, 32 of W7's 64
      op.hm.w6[g] = make_map_2d(A.w, A.cin_pad, A.cout_pad, p.ncta == 2 ? 64 : 128);
      op.hm.w7[g] = make_map_2d(B.w, B.cin_pad, B.cout_pad, p.ncta == 2 ? 32 : 64);
      if (o.buf != -1) {
        op.hm.out32[g] = make_map_3d_store(plan.bufs[o.buf]->p, plan.buf_c[o.buf], uint64_t(gi.Hp()) * gi.Wp(), plan.n, 32);
        op.hm.out16[g] = make_map_3d_store(plan.bufs[o.buf]->p, plan.buf_c[o.buf], uint64_t(gi.Hp()) * gi.Wp(), plan.n, 16);
        op.hm.out8[g] = make_map_3d_store(plan.bufs[o.buf]->p, plan.buf_c[o.buf], uint64_t(gi.Hp()) * gi.Wp(), plan.n, 8);
      }
      op.layers[g] = l7[g];
      op.head_l6[g] = l6[g];
      // the parity hook shows the fp32 copy when there is one (as the unfused plan did)
      record_io(l7[g], in[g], out2.empty() ? out[g] : out2[g]);
      plan.layer_fusion[l6[g]] = 2;
      plan.layer_fusion[l7[g]] = 3;
      plan.layer_in_from[l7[g]] = l6[g];
    }
    plan.ops.push_back(op);
  }

  // one launch covering 1 or 2 conv layers (sibling branches) of equal shape;
  // `pool`: the single output view is the 2x2-pooled result (level + 1)
  // `spill`: the destination channels from the view's end up to the next
  // multiple of 128 may be overwritten (a dense block's next slice, written by
  // a later layer, or padding), which lets a 96-channel layer take the
  // swap-AB kernel's 128-channel tiles
  void conv(std::initializer_list<int> layers_il, std::initializer_list<TensorView> ins,
            std::initializer_list<TensorView> outs, bool pool = false, bool spill = false) {
    std::vector<int> layers(layers_il);
    std::vector<TensorView> in(ins), out(outs);
    PlanOp op;
    op.kind = PlanOp::kConv;
    ConvParams& p = op.cp;
    const ConvLayerDev& L0 = net.layers[layers[0]];
    const Geometry& gi = plan.geo[in[0].level];
    p.k = L0.exec_k;
    p.cin_chunks = L0.cin_pad / 64;
    // live input channels (highest nonzero weight column + 1) over the group:
    // the pixel-major kernel skips the zero tail of the last 64-channel chunk
    // (AVEC_K16TAIL=0 turns this off)
    static const bool k16_tail = [] {
      const char* e = std::getenv("AVEC_K16TAIL");
      return !(e && e[0] == '0');
    }();
    int live = k16_tail ? 0 : L0.cin_pad;
    for (int l : layers) {
      const ConvDef& d = net.layers[l].def;
      if (net.layers[l].exec_k != d.k) live = L0.cin_pad;  // conv1_1's packed taps
      else live = std::max(live, d.cin_map.empty() ? d.cin : *std::max_element(d.cin_map.begin(), d.cin_map.end()) + 1);
    }
    p.k16_last = std::min(4, std::max(1, (live - 64 * (p.cin_chunks - 1) + 15) / 16));
    p.in_c_off = in[0].c_off;
    p.n_images = plan.n;
    p.H = gi.H;
    p.W = gi.W;
    p.Hp = gi.Hp();
    p.Wp = gi.Wp();
    p.P = gi.P;
    const bool to_output = out[0].buf == -1;
    // Kernel choice (measured): swap-AB (M = 128 Cout,
    // N = 256-pixel MMAs, 96 B/clk of smem operand reads) for the 7x7 layers
    // and for 3x3 layers with exactly 128 output channels; pixel-major
    // (M = 128 pixels, N = Cout) elsewhere — with N = 256 it is as lean, with
    // N <= 128 it hits the 128 B/clk operand-read ceiling, but it is the only
    // sensible tile for 64-channel and thin-head outputs and its direct-store
    // epilogue suits the short-K, high-resolution layers.
    static const int tc3 = [] {
      const char* e = std::getenv("AVEC_TC3");
      return e ? std::atoi(e) : 0;
    }();
    // BODY_25's level-3 dense-block convs (3x3, 96/128 channels) on the
    // swap-AB kernel (128 x 256 MMAs instead of the pixel-major N = 96/128
    // ones). Measured at C5 and rejected, opt-in AVEC_TC_DENSE=1: 96-channel
    // layers 96-107 -> 124-133 us (a quarter of every tile is padding), 128-
    // channel layers 120 -> 125 us, the block's first convs 207/313 ->
    // 271/323 us; all 90 launches 14.8 -> 16.0 ms (2 subs: 20.5 ms)
    static const bool tc_dense = [] {
      const char* e = std::getenv("AVEC_TC_DENSE");
      return e && e[0] == '1';
    }();
    const bool dense_tc = tc_dense && spill && L0.exec_k == 3 && (L0.def.cout == 96 || L0.def.cout == 128) &&
                          layers.size() == 1 && !pool && out[0].c_off + 128 <= out[0].c_stride;
    const bool want_tc = L0.exec_k == 7 || dense_tc ||
                         (tc3 && L0.exec_k == 3 && L0.def.cout == 128 && L0.cin_pad >= 128);
    bool tc_ok = want_tc && !to_output && !pool;
    for (size_t g = 0; g < layers.size(); ++g)
      tc_ok = tc_ok && out[g].c_off % 8 == 0 && out[g].level == in[g].level;
    p.pixel_major = tc_ok ? 0 : 1;
    if (L0.exec_k == 7 && p.pixel_major) fail(AVEC_ERR_UNSUPPORTED, "7x7 layer needs the swap-AB kernel");
    // outputs at 8-aligned channel offsets take the TMA-store path: swap-AB
    // stores 64-channel boxes (cout % 64 == 0); pixel-major stores 64/32/16/8-
    // channel boxes covering round_up(cout, 8) channels, so the buffer layouts
    // keep the channels up to the next multiple of 8 free (netspec.hpp)
    bool slab = !to_output;
    for (size_t g = 0; g < layers.size(); ++g) {
      const int cout = net.layers[layers[g]].def.cout;
      const int span = !p.pixel_major && dense_tc ? 128 : round_up(cout, 8);
      slab = slab && (p.pixel_major || cout % 64 == 0 || dense_tc) && out[g].c_off % 8 == 0 &&
             out[g].c_off + span <= out[g].c_stride && out[g].level == in[g].level + (pool ? 1 : 0);
    }
    if (pool && (!slab || layers.size() != 1 || !p.pixel_major))
      fail(AVEC_ERR_UNSUPPORTED, "fused pooling needs one pixel-major slab output");
    p.out_mode = to_output ? kOutNchwF32 : slab ? kOutTmaBf16 : kOutDirectBf16;
    if (p.pixel_major) {
      p.pm_n = conv_pm_tile_n(L0.def.cout);
      p.subs = conv_pm_subs(p.pm_n);
      p.m_tiles = (L0.def.cout + p.pm_n - 1) / p.pm_n;
      p.ncta = pm_ncta(p.pm_n, L0.exec_k, p.cin_chunks);
      if (pool) {
        // [2 rows x 128 columns] per CTA; the pair stacks its two row pairs
        p.pool = 1;
        p.pool_P = plan.geo[in[0].level + 1].P;
        p.col_blocks = (p.W + 127) / 128;
        p.tiles_per_image = p.H / (2 * p.ncta) * p.col_blocks;
      } else {
        const int px = 128 * p.subs * p.ncta;
        p.tiles_per_image = (p.H * p.Wp + px - 1) / px;
      }
    } else {
      p.pm_n = 0;
      p.m_tiles = L0.cout_pad / 128;
      // 512-pixel tiles share each weight k-block across two MMAs; fall back to
      // 256-pixel tiles (double-buffered TMEM) when that leaves SMs idle
      const int per_img_units = int(layers.size()) * plan.n * p.m_tiles;  // tiles per pixel-tile index
      const int wide = per_img_units * ((p.H * p.Wp + 511) / 512);
      static const int dense_subs = [] {
        const char* e = std::getenv("AVEC_TC_DENSE_SUBS");
        return e ? std::atoi(e) : 1;
      }();
      p.subs = (L0.exec_k == 7 || tc3 == 3 || (tc3 == 1 && wide >= 2 * 148)) ? 2 : 1;
      if (dense_tc) p.subs = dense_subs == 2 ? 2 : 1;
      // launches that will run split-K (wide tiles fill less than half the
      // SMs) take 256-pixel tiles: twice the tiles, half the split count, half
      // the fp32 partial traffic per tile. AVEC_SPLITK_NARROW=0 keeps 512.
      static const bool narrow = [] {
        const char* e = std::getenv("AVEC_SPLITK_NARROW");
        return !(e && e[0] == '0');
      }();
      if (p.subs == 2 && narrow && conv_tc_splits(wide, p.cin_chunks * p.k, sm_count()) > 1) p.subs = 1;
      // Tile width: with 512-pixel tiles a C2 7x7 launch is 128 tiles on 148
      // SMs. Narrower tiles (the second MMA shrinks, N = T - 256) trade a
      // little per-tile weight streaming for filling the SMs: pick the width
      // maximising (useful positions / computed positions) x (busy SM-waves).
      // Opt-in (AVEC_TILE_FIT=1): measured -2.3% serial step time on C2 (480-px
      // tiles) but -3.7% throughput with the server's two slots in flight, where
      // the other stream already fills the idle SMs and only the extra per-tile
      // weight traffic remains.
      static const bool tile_fit = [] {
        const char* e = std::getenv("AVEC_TILE_FIT");
        return e && e[0] == '1';
      }();
      p.tile_px = 256 * p.subs;
      if (p.subs == 2 && tile_fit) {
        const int sms = sm_count();
        const int pos = p.H * p.Wp;
        double best = 0;
        for (int T = 512; T >= 288; T -= 32) {
          const int tpi = (pos + T - 1) / T;
          const int tiles = per_img_units * tpi;
          const int waves = (tiles + sms - 1) / sms;
          const double eff = double(pos) / (double(tpi) * T) * double(tiles) / (double(waves) * sms);
          if (eff > best * 1.01) {
            best = eff;
            p.tile_px = T;
          }
        }
      }
      p.tiles_per_image = (p.H * p.Wp + p.tile_px - 1) / p.tile_px;
    }
    p.n_groups = int(layers.size());
    p.total_tiles = p.n_groups * p.n_images * p.tiles_per_image * p.m_tiles;
    p.units_per_seg = (p.H * p.Wp + 31) / 32;
    // balanced persistent partition for the wide-tile swap-AB launches
    // Opt-in (AVEC_BALANCED=1): measured slower on C2 (95.6 vs 82.7 us per 7x7
    // pair) because the runs that span two segments re-stream the weights twice
    // and set the kernel's critical path; kept for shapes whose regular tile
    // count leaves many SMs idle.
    static const bool balanced_on = [] {
      const char* e = std::getenv("AVEC_BALANCED");
      return e && e[0] == '1';
    }();
    p.balanced_units = (balanced_on && !p.pixel_major && p.subs == 2 && p.m_tiles == 1)
                           ? p.n_groups * p.n_images * p.units_per_seg
                           : 0;
    // split-K for swap-AB launches too small to fill the SMs (C1's single
    // frame: 10 tiles of 7x7 work for 148 SMs; frame groups of 1-4 frames)
    p.splits = 1;
    if (!p.pixel_major && p.balanced_units == 0 && p.out_mode != kOutNchwF32) {
      p.splits = conv_tc_splits(p.total_tiles, p.cin_chunks * p.k, sm_count());
      if (p.splits > 1)
        plan.ws_bytes = std::max(plan.ws_bytes, size_t(p.total_tiles) * p.splits * p.tile_px * 128 * 4);
    }
    for (size_t g = 0; g < layers.size(); ++g) {
      const ConvLayerDev& L = net.layers[layers[g]];
      if (L.exec_k != p.k || L.cin_pad != L0.cin_pad || L.cout_pad != L0.cout_pad ||
          in[g].c_off != p.in_c_off || (out[g].buf == -1) != to_output)
        fail(AVEC_ERR_INVALID_MODEL, "grouped conv layers differ in shape");
      if (pool) {
        const int ob = out[g].buf;
        const Geometry& go = plan.geo[in[g].level + 1];
        op.maps.out_pool[g] = make_map_4d_store(plan.bufs[ob]->p, plan.buf_c[ob], go.Wp(), go.Hp(), plan.n);
      } else if (p.out_mode == kOutTmaBf16) {
        const int ob = out[g].buf;
        op.maps.out[g] = make_map_3d_store(plan.bufs[ob]->p, plan.buf_c[ob], uint64_t(gi.Hp()) * gi.Wp(),
                                           plan.n);
        if (p.pixel_major) {
          const uint64_t rows = uint64_t(gi.Hp()) * gi.Wp();
          op.maps.out32[g] = make_map_3d_store(plan.bufs[ob]->p, plan.buf_c[ob], rows, plan.n, 32);
          op.maps.out16[g] = make_map_3d_store(plan.bufs[ob]->p, plan.buf_c[ob], rows, plan.n, 16);
          op.maps.out8[g] = make_map_3d_store(plan.bufs[ob]->p, plan.buf_c[ob], rows, plan.n, 8);
        }
      }
      ConvGroupParams& gp = p.g[g];
      gp.bias = L.bias;
      gp.out = to_output ? plan.out.p : plan.bufs[out[g].buf]->p;
      gp.out_c_off = out[g].c_off;
      gp.out_c_stride = out[g].c_stride;
      gp.cout = L.def.cout;
      gp.act = L.def.act;
      gp.slope = L.slope;
      const int ib = in[g].buf;
      const uint64_t rows = uint64_t(plan.n) * gi.Hp() * gi.Wp();
      op.maps.act_big[g] = make_map_2d(plan.bufs[ib]->p, plan.buf_c[ib], rows, 256);
      op.maps.act_small[g] = make_map_2d(plan.bufs[ib]->p, plan.buf_c[ib], rows, 8);
      op.maps.act_mid[g] = make_map_2d(plan.bufs[ib]->p, plan.buf_c[ib], rows, 128);
      op.maps.wgt[g] = make_map_2d(L.w, uint64_t(L.exec_k) * L.exec_k * L.cin_pad, L.cout_pad,
                                   p.pixel_major ? uint32_t(p.pm_n / p.ncta) : 128u);
      op.layers[g] = layers[g];
      record_io(layers[g], in[g], out[g]);
    }
    plan.ops.push_back(op);
  }

  void pool(int src, int dst) {
    PlanOp op;
    op.kind = PlanOp::kPool;
    op.src = src;
    op.dst = dst;
    op.level = plan.buf_level[src];
    op.C = plan.buf_c[src];
    plan.ops.push_back(op);
  }
};

// VGG-19[:10] + CPM adapters (shared by both families); conv4_4_CPM writes the
// 128-channel trunk into `cat` at channel `trunk_off`. Returns the next layer.
int build_trunk(PlanBuilder& b, Plan& plan, int cat, int trunk_off) {
  int li = 0;
  // level 0
  const int p1 = b.buffer(1, 64), a1 = b.buffer(1, 128);
  if (b.conv12(0, 1, p1)) {  // conv1_1 + conv1_2 + pool1 in one kernel
    li = 2;
  } else {
    const int a0 = b.buffer(0, 64);
    b.first(li++, b.view(a0, 0, 64));          // conv1_1 fused with the frame conversion
    b.conv_pool(li++, b.view(a0, 0, 64), p1);  // conv1_2 + pool1
  }
  b.conv({li++}, {b.view(p1, 0, 64)}, {b.view(a1, 0, 128)});   // conv2_1
  const int p2 = b.buffer(2, 128), a2 = b.buffer(2, 256), b2 = b.buffer(2, 256);
  b.conv_pool(li++, b.view(a1, 0, 128), p2);  // conv2_2 + pool2
  b.conv({li++}, {b.view(p2, 0, 128)}, {b.view(a2, 0, 256)});  // conv3_1
  b.conv({li++}, {b.view(a2, 0, 256)}, {b.view(b2, 0, 256)});  // conv3_2
  b.conv({li++}, {b.view(b2, 0, 256)}, {b.view(a2, 0, 256)});  // conv3_3
  b.conv({li++}, {b.view(a2, 0, 256)}, {b.view(b2, 0, 256)});  // conv3_4
  const int p3 = b.buffer(3, 256), a3 = b.buffer(3, 512), b3 = b.buffer(3, 512),
            c3 = b.buffer(3, 256);
  b.pool(b2, p3);
  b.conv({li++}, {b.view(p3, 0, 256)}, {b.view(a3, 0, 512)});  // conv4_1
  b.conv({li++}, {b.view(a3, 0, 512)}, {b.view(b3, 0, 512)});  // conv4_2
  b.conv({li++}, {b.view(b3, 0, 512)}, {b.view(c3, 0, 256)});  // conv4_3_CPM
  b.conv({li++}, {b.view(c3, 0, 256)}, {b.view(cat, trunk_off, 128)});  // conv4_4_CPM -> trunk slot
  return li;
}

// COCO program (pose_deploy_linevec.prototxt) on padded-flat buffers
void build_coco_plan(Plan& plan, const PoseNet& net, int device, cudaStream_t stream) {
  const PoseFamily& f = net.fam;
  PlanBuilder b{plan, net, device, stream};
  const int nl = int(f.convs.size());
  plan.layer_in.assign(nl, TensorView{});
  plan.layer_out.assign(nl, TensorView{});
  plan.layer_fusion.assign(nl, 0);
  plan.layer_in_from.resize(nl);
  for (int i = 0; i < nl; ++i) plan.layer_in_from[i] = i;
  const int cat = b.buffer(3, kCocoCatChannels);  // [trunk | L1 at kCocoPaf | L2 at kCocoHeat]
  int li = build_trunk(b, plan, cat, 0);
  const int T = f.trunk_channels, C1 = f.paf_channels, C2 = f.heat_channels;  // T == kCocoPaf
  // branch buffers
  const int l1a = b.buffer(3, 128), l1b = b.buffer(3, 128), l2a = b.buffer(3, 128),
            l2b = b.buffer(3, 128), l1x = b.buffer(3, 512), l2x = b.buffer(3, 512);
  const int s1 = li;  // stage 1: L1 layers s1..s1+4, L2 layers s1+5..s1+9
  b.conv({s1 + 0, s1 + 5}, {b.view(cat, 0, T), b.view(cat, 0, T)}, {b.view(l1a, 0, 128), b.view(l2a, 0, 128)});
  b.conv({s1 + 1, s1 + 6}, {b.view(l1a, 0, 128), b.view(l2a, 0, 128)}, {b.view(l1b, 0, 128), b.view(l2b, 0, 128)});
  b.conv({s1 + 2, s1 + 7}, {b.view(l1b, 0, 128), b.view(l2b, 0, 128)}, {b.view(l1a, 0, 128), b.view(l2a, 0, 128)});
  b.head({s1 + 3, s1 + 8}, {s1 + 4, s1 + 9}, {b.view(l1a, 0, 128), b.view(l2a, 0, 128)},
         {b.view(l1x, 0, 512), b.view(l2x, 0, 512)}, {b.view(cat, kCocoPaf, C1), b.view(cat, kCocoHeat, C2)});
  li += 10;
  for (int t = 2; t <= f.stages; ++t) {
    const int s = li;  // L1: s..s+6, L2: s+7..s+13
    const int catc = T + C1 + C2;  // Caffe channels (cin_map places them)
    b.conv({s + 0, s + 7}, {b.view(cat, 0, catc), b.view(cat, 0, catc)},
           {b.view(l1a, 0, 128), b.view(l2a, 0, 128)});
    int x = l1a, y = l1b, u = l2a, v = l2b;
    for (int i = 1; i <= 4; ++i) {  // Mconv2..5 (7x7)
      b.conv({s + i, s + 7 + i}, {b.view(x, 0, 128), b.view(u, 0, 128)}, {b.view(y, 0, 128), b.view(v, 0, 128)});
      std::swap(x, y);
      std::swap(u, v);
    }
    // Mconv6 (1x1, ReLU) + Mconv7 (1x1) per branch, fused
    const std::vector<TensorView> outs =
        t == f.stages ? std::vector<TensorView>{b.view(-1, C2, C1), b.view(-1, 0, C2)}  // wire: [heat | paf] fp32
                      : std::vector<TensorView>{b.view(cat, kCocoPaf, C1), b.view(cat, kCocoHeat, C2)};
    b.head({s + 5, s + 12}, {s + 6, s + 13}, {b.view(x, 0, 128), b.view(u, 0, 128)},
           {b.view(y, 0, 128), b.view(v, 0, 128)}, outs);
    li += 14;
  }
  if (li != nl) fail(AVEC_ERR_INVALID_MODEL, "plan/layer table mismatch");
}

// BODY_25 program: 4 PAF stages then 2 heatmap stages, each 5 dense blocks of
// three 3x3 PReLU convs concatenated in place (ping-pong X/Y buffers) + Mconv6/7.
// Stage concat buffer: [heat 0..25 | PAF 32..83 | trunk 88..215] (netspec.hpp).
void build_body25_plan(Plan& plan, const PoseNet& net, int device, cudaStream_t stream) {
  const PoseFamily& f = net.fam;
  PlanBuilder b{plan, net, device, stream};
  const int nl = int(f.convs.size());
  plan.layer_in.assign(nl, TensorView{});
  plan.layer_out.assign(nl, TensorView{});
  plan.layer_fusion.assign(nl, 0);
  plan.layer_in_from.resize(nl);
  for (int i = 0; i < nl; ++i) plan.layer_in_from[i] = i;
  const int cat = b.buffer(3, kB25CatChannels);
  int li = build_trunk(b, plan, cat, kB25Trunk);
  const int X0 = b.buffer(3, 384), Y0 = b.buffer(3, 384), m6 = b.buffer(3, 512);
  const int P = f.paf_channels, Hc = f.heat_channels;
  auto stage = [&](TensorView in, int w, int c6, std::vector<TensorView> heads) {
    int X = X0, Y = Y0;
    for (int blk = 1; blk <= 5; ++blk) {
      // each layer may spill zeros past its slice: the next layer of the block
      // overwrites them, the last one's land in the 3w..round_up(3w + 32) pad
      b.conv({li++}, {blk == 1 ? in : b.view(X, 0, 3 * w)}, {b.view(Y, 0, w)}, false, true);
      b.conv({li++}, {b.view(Y, 0, w)}, {b.view(Y, w, w)}, false, true);
      b.conv({li++}, {b.view(Y, w, w)}, {b.view(Y, 2 * w, w)}, false, true);
      std::swap(X, Y);
    }
    const int l6 = li++, l7 = li++;  // Mconv6 (1x1, PReLU) + Mconv7 (1x1), fused
    std::vector<TensorView> out2;
    if (heads.size() > 1) out2.push_back(heads[1]);
    b.head({l6}, {l7}, {b.view(X, 0, 3 * w)}, {b.view(m6, 0, c6)}, {heads[0]}, out2);
  };
  // PAF stage 0 reads the trunk; stages 1..3 read [PAF | trunk] = window [32, 224)
  stage(b.view(cat, kB25Trunk, 128), 96, 256, {b.view(cat, kB25Paf, P)});
  for (int t = 1; t <= 3; ++t) {
    std::vector<TensorView> heads{b.view(cat, kB25Paf, P)};
    if (t == 3) heads.push_back(b.view(-1, Hc, P));  // final PAFs also go out on the wire (fp32)
    stage(b.view(cat, kB25Paf, 192), 128, 512, heads);
  }
  stage(b.view(cat, kB25Paf, 192), 96, 256, {b.view(cat, kB25Heat, Hc)});  // heat stage 0
  stage(b.view(cat, 0, 256), 128, 512, {b.view(-1, 0, Hc)});               // heat stage 1
  if (li != nl) fail(AVEC_ERR_INVALID_MODEL, "plan/layer table mismatch");
}

void run_ops(avec_ctx* ctx, const Plan& plan, const PoseNet& net, size_t first, size_t last,
             cudaStream_t st) {
  for (size_t i = first; i < last; ++i) {
    const PlanOp& op = plan.ops[i];
    switch (op.kind) {
      case PlanOp::kFirst:
        launch_conv_first(op.maps, op.cp, plan.in.as<float>(), ctx->sms, st);
        break;
      case PlanOp::kHead:
        launch_conv_head(op.hm, op.hp, ctx->sms, st);
        break;
      case PlanOp::kConv12:
        launch_conv12(op.maps, op.cp, ctx->sms, st);
        break;
      case PlanOp::kConv:
        if (op.cp.pixel_major)
          launch_conv_pm(op.maps, op.cp, ctx->sms, st);
        else
          launch_conv_tc(op.maps, op.cp, ctx->sms, st);
        break;
      case PlanOp::kPool: {
        const Geometry& g = plan.geo[op.level];
        launch_maxpool2(plan.bufs[op.src]->p, plan.n, g.H, g.W, g.P, op.C, plan.bufs[op.dst]->p,
                        plan.geo[op.level + 1].P, st);
        break;
      }
    }
  }
}

}  // namespace

Plan* get_plan(avec_ctx* ctx, Slot* slot, const Model& m, int n_img, int H, int W) {
  auto key = std::make_tuple(m.id, n_img, H, W);
  auto it = slot->plans.find(key);
  if (it != slot->plans.end()) {
    it->second->last_use = ++slot->use_clock;
    return it->second.get();
  }
  static const size_t max_plans = [] {
    const char* e = std::getenv("AVEC_PLANS_PER_SLOT");
    const int v = e ? std::atoi(e) : 4;
    return size_t(v > 0 ? v : 1);
  }();
  if (slot->plans.size() >= max_plans) {
    // the slot is leased to this caller, but its previous forward may still
    // run on the slot stream or on a caller stream (marked by `done`, whose
    // pending flag the lease may already have cleared)
    check_cuda(cudaStreamSynchronize(slot->stream), "plan eviction sync");
    check_cuda(cudaEventSynchronize(slot->done), "plan eviction sync");
    auto lru = slot->plans.begin();
    for (auto p = slot->plans.begin(); p != slot->plans.end(); ++p)
      if (p->second->last_use < lru->second->last_use) lru = p;
    slot->plans.erase(lru);
  }
  auto plan = std::make_unique<Plan>();
  plan->last_use = ++slot->use_clock;
  plan->n = n_img;
  plan->H = H;
  plan->W = W;
  for (int l = 0; l < 4; ++l) plan->geo[l] = Geometry{H >> l, W >> l, l == 3 ? 3 : 1};
  plan->in_elems = uint64_t(n_img) * 3 * H * W;
  plan->out_elems = uint64_t(n_img) * m.net->fam.out_channels() * (H / 8) * (W / 8);
  plan->in.ensure(plan->in_elems * 4, ctx->device);
  plan->out.ensure(plan->out_elems * 4, ctx->device);
  if (m.net->fam.body25())
    build_body25_plan(*plan, *m.net, ctx->device, slot->stream);
  else
    build_coco_plan(*plan, *m.net, ctx->device, slot->stream);
  // the zeroed buffers must be in place before a forward on any stream (a
  // caller's stream in forward_device) reads them
  check_cuda(cudaStreamSynchronize(slot->stream), "plan zero-fill");
  if (plan->ws_bytes) {  // split-K partials, shared by the plan's (stream-ordered) launches
    plan->ws.ensure(plan->ws_bytes, ctx->device);
    for (PlanOp& op : plan->ops)
      if (op.kind == PlanOp::kConv && op.cp.splits > 1) op.cp.ws = plan->ws.as<float>();
  }
  // capture the whole op sequence once; replays cost one launch
  cudaGraph_t g = nullptr;
  check_cuda(cudaStreamBeginCapture(slot->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
  try {
    run_ops(ctx, *plan, *m.net, 0, plan->ops.size(), slot->stream);
  } catch (...) {
    cudaStreamEndCapture(slot->stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  check_cuda(cudaStreamEndCapture(slot->stream, &g), "end capture");
  cudaError_t e = cudaGraphInstantiate(&plan->graph, g, 0);
  cudaGraphDestroy(g);
  check_cuda(e, "graph instantiate");
  Plan* raw = plan.get();
  slot->plans.emplace(key, std::move(plan));
  return raw;
}

void posenet_shape(const Model& m, uint32_t n, uint32_t c, uint32_t h, uint32_t w, int& n_img) {
  const uint64_t chans = uint64_t(n) * c;
  if (chans % 3 != 0)
    fail(AVEC_ERR_INVALID_ARGUMENT, "pose net needs 3 channels per frame, got " + std::to_string(chans));
  if (h % 8 || w % 8)
    fail(AVEC_ERR_INVALID_ARGUMENT, "pose net needs height and width divisible by 8");
  n_img = int(chans / 3);
  const uint64_t E = chans * h * w;
  const uint64_t K = uint64_t(n_img) * m.net->fam.out_channels() * (h / 8) * (w / 8);
  const uint64_t law = uint64_t(std::llround(double(E) / m.divisor));
  if (law != K)
    fail(AVEC_ERR_INVALID_ARGUMENT, "output divisor " + std::to_string(m.divisor) +
                                        " gives " + std::to_string(law) + " outputs, the net yields " +
                                        std::to_string(K));
}

// ------------------------------------------------------------------ context
void ctx_init(avec_ctx* ctx, int device, int slots) {
  int count = 0;
  check_cuda(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
  if (device < 0 || device >= count)
    fail(AVEC_ERR_INVALID_ARGUMENT, "no CUDA device " + std::to_string(device));
  check_cuda(cudaSetDevice(device), "cudaSetDevice");
  cudaDeviceProp prop;
  check_cuda(cudaGetDeviceProperties(&prop, device), "device properties");
  if (prop.major != 10)
    fail(AVEC_ERR_UNSUPPORTED, std::string("needs an sm_100 (B200) device, found ") + prop.name);
  ctx->device = device;
  ctx->sms = prop.multiProcessorCount;
  ctx->label = "b200:" + std::to_string(device);
  conv_configure();
  conv_pm_configure();
  conv_first_configure();
  conv_head_configure();
  conv12_configure();
  if (slots <= 0) slots = 2;
  for (int i = 0; i < slots; ++i) {
    auto s = std::make_unique<Slot>();
    s->index = i;
    check_cuda(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking), "stream");
    check_cuda(cudaStreamCreateWithFlags(&s->copy_in, cudaStreamNonBlocking), "stream");
    check_cuda(cudaStreamCreateWithFlags(&s->copy_out, cudaStreamNonBlocking), "stream");
    check_cuda(cudaEventCreate(&s->ev0), "event");
    check_cuda(cudaEventCreate(&s->ev1), "event");
    check_cuda(cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming), "event");
    for (int b = 0; b < 2; ++b) {
      check_cuda(cudaEventCreateWithFlags(&s->stage_ev[b], cudaEventDisableTiming), "event");
      s->stage[b].ensure(kStageChunk);
    }
    ctx->slots.push_back(std::move(s));
    ctx->slot_busy.push_back(false);
  }
}

void ctx_shutdown(avec_ctx* ctx) {
  cudaSetDevice(ctx->device);
  for (auto& s : ctx->slots) {
    if (s->stream) cudaStreamSynchronize(s->stream);
    s->plans.clear();
    if (s->stream) cudaStreamDestroy(s->stream);
    for (cudaStream_t st : {s->copy_in, s->copy_out})
      if (st) cudaStreamDestroy(st);
    for (cudaEvent_t e : s->chunk_ev) cudaEventDestroy(e);
    cudaEventDestroy(s->ev0);
    cudaEventDestroy(s->ev1);
    cudaEventDestroy(s->done);
    cudaEventDestroy(s->stage_ev[0]);
    cudaEventDestroy(s->stage_ev[1]);
  }
  ctx->slots.clear();
  ctx->models.clear();
}

uint64_t model_register(avec_ctx* ctx, const uint8_t* digest, const std::string& name,
                        const uint8_t* structure, size_t structure_len, const uint8_t* weights,
                        uint64_t weights_len, double divisor) {
  // backend.cpp:70-73: divisor positive and finite, structure non-empty
  if (!(divisor > 0.0) || !std::isfinite(divisor))
    fail(AVEC_ERR_INVALID_MODEL, "output divisor must be positive and finite");
  if (structure_len == 0 || !structure) fail(AVEC_ERR_INVALID_MODEL, "model structure is empty");
  std::array<uint8_t, 32> key;
  std::memcpy(key.data(), digest, 32);
  {
    std::lock_guard<std::mutex> lk(ctx->model_m);
    auto it = ctx->id_by_digest.find(key);
    if (it != ctx->id_by_digest.end()) return it->second;  // idempotent per digest
  }
  Model m;
  m.divisor = divisor;
  m.name = name;
  if (is_avecnet(structure, structure_len)) {
    PoseFamily fam = parse_avecnet(structure, structure_len);
    const uint64_t nf = fam.weight_floats();
    std::vector<float> synth;
    const float* w = nullptr;
    if (weights_len == 0) {
      synth.resize(nf);
      synth_weights(fam, synth.data());
      w = synth.data();
    } else if (weights_len == nf * 4) {
      w = reinterpret_cast<const float*>(weights);
    } else {
      fail(AVEC_ERR_INVALID_MODEL, "pose-net weights must be " + std::to_string(nf * 4) +
                                       " bytes (Caffe-order fp32), got " + std::to_string(weights_len));
    }
    m.kind = AVEC_MODEL_POSENET;
    m.net = upload_posenet(ctx->device, std::move(fam), w);
  }
  std::lock_guard<std::mutex> lk(ctx->model_m);
  auto it = ctx->id_by_digest.find(key);
  if (it != ctx->id_by_digest.end()) return it->second;
  m.id = ctx->next_id++;
  ctx->id_by_digest.emplace(key, m.id);
  ctx->models.emplace(m.id, m);
  return m.id;
}

Model model_lookup(avec_ctx* ctx, uint64_t handle) {
  std::lock_guard<std::mutex> lk(ctx->model_m);
  auto it = ctx->models.find(handle);
  if (it == ctx->models.end())
    fail(AVEC_ERR_UNKNOWN_MODEL, "handle was never issued by this backend");
  return it->second;
}

uint64_t output_elems_for(const Model& m, uint32_t n, uint32_t c, uint32_t h, uint32_t w) {
  const uint64_t E = uint64_t(n) * c * h * w;
  if (E == 0) fail(AVEC_ERR_INVALID_ARGUMENT, "empty input");
  if (m.kind == AVEC_MODEL_POSENET) {
    int n_img = 0;
    posenet_shape(m, n, c, h, w, n_img);
    return uint64_t(n_img) * m.net->fam.out_channels() * (h / 8) * (w / 8);
  }
  // backend.cpp:42-47
  const uint64_t K = uint64_t(std::llround(double(E) / m.divisor));
  if (K < 1) fail(AVEC_ERR_DEGENERATE_OUTPUT, "model yields zero output elements");
  if (K > E) fail(AVEC_ERR_DEGENERATE_OUTPUT, "model yields more output elements than inputs");
  return K;
}

namespace {

// Large segment-mean cycles from pinned memory (C3's forwarded-memcpy sweep:
// with c = 1 the reply is as large as the frame): the frame is cut at segment
// boundaries into ~8 MB chunks; chunk c's H2D (copy_in stream), its segments
// (slot stream) and its output's D2H (copy_out stream) chain by events, so
// H2D of later chunks, the kernels and D2H of earlier chunks overlap and both
// PCIe directions stream at once instead of H2D then D2H.
constexpr uint64_t kOverlapMin = uint64_t(16) << 20;

void overlapped_segment_means(Slot* s, const float* in, float* out, uint64_t E, uint64_t K) {
  const uint64_t chunks = std::max<uint64_t>(2, std::min<uint64_t>(64, E * 4 / (uint64_t(8) << 20)));
  while (s->chunk_ev.size() < 2 * chunks) {
    cudaEvent_t e = nullptr;
    check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    s->chunk_ev.push_back(e);
  }
  check_cuda(cudaStreamSynchronize(s->stream), "slot idle");  // any earlier use of d_in/d_out is done
  check_cuda(cudaEventRecord(s->ev0, s->copy_in), "ev0");
  for (uint64_t c = 0; c < chunks; ++c) {
    const uint64_t j0 = c * K / chunks, j1 = (c + 1) * K / chunks;
    const uint64_t a = segment_bound(j0, E, K), b = segment_bound(j1, E, K);
    if (b > a)
      check_cuda(cudaMemcpyAsync(s->d_in.as<float>() + a, in + a, (b - a) * 4, cudaMemcpyHostToDevice, s->copy_in),
                 "H2D chunk");
    check_cuda(cudaEventRecord(s->chunk_ev[2 * c], s->copy_in), "chunk event");
    check_cuda(cudaStreamWaitEvent(s->stream, s->chunk_ev[2 * c], 0), "wait H2D");
    launch_segment_means(s->d_in.as<float>(), s->d_out.as<float>(), E, K, s->stream, j0, j1);
    check_cuda(cudaEventRecord(s->chunk_ev[2 * c + 1], s->stream), "chunk event");
    check_cuda(cudaStreamWaitEvent(s->copy_out, s->chunk_ev[2 * c + 1], 0), "wait kernel");
    if (j1 > j0)
      check_cuda(cudaMemcpyAsync(out + j0, s->d_out.as<float>() + j0, (j1 - j0) * 4, cudaMemcpyDeviceToHost,
                                 s->copy_out),
                 "D2H chunk");
  }
  check_cuda(cudaEventRecord(s->ev1, s->copy_out), "ev1");
  check_cuda(cudaEventSynchronize(s->ev1), "overlapped sync");
}

// A pose-net cycle between pinned host buffers as two frame groups (frames
// are independent; batch folded into channels, server.cpp:297-301): group
// g's H2D (copy_in), its graph (slot stream, behind its H2D's event) and its
// output's D2H (copy_out, behind the graph) chain by events, so group 1's
// input crosses PCIe while group 0 computes and group 0's output returns
// while group 1 computes: one synchronous cycle no longer pays its copies
// in series. The group plan's buffers are shared by the groups, so each group
// enters and leaves them by a device copy from/to the slot's staging (in
// stream order on the slot stream). Only for large cycles (>= 64 MB of
// frames): halving the batch costs the group plans' efficiency, which C5's
// copies repay and C2's do not (bench.py, same box: C5 32x1312x736 e2e
// 994 -> 1032 frames/s, one thread 854 -> 921; C2 8x656x368 e2e 2808 ->
// 2643). AVEC_FWD_PIPE=0 turns it off (A/B).
constexpr uint64_t kPipeMin = uint64_t(64) << 20;

bool pipelined_forward_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("AVEC_FWD_PIPE");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool pipelined_posenet(avec_ctx* ctx, Slot* s, const Model& m, int n_img, int h, int w, const float* in, float* out,
                       uint64_t E, uint64_t K) {
  const int gf = (n_img + 1) / 2;  // frames of group 0; group 1 takes the rest
  s->d_in.ensure(E * 4, ctx->device);
  s->d_out.ensure(K * 4, ctx->device);
  while (s->chunk_ev.size() < 4) {
    cudaEvent_t e = nullptr;
    check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    s->chunk_ev.push_back(e);
  }
  const uint64_t fin = E / n_img, fout = K / n_img;  // elements per frame in / out
  Plan* plans[2] = {get_plan(ctx, s, m, gf, h, w), nullptr};  // built (captured) before anything is queued
  plans[1] = n_img - gf == gf ? plans[0] : get_plan(ctx, s, m, n_img - gf, h, w);
  // both group plans must be resident at once (a one-plan cache, AVEC_PLANS_PER_SLOT=1, evicts the first)
  if (!s->plans.count(std::make_tuple(m.id, gf, h, w))) return false;
  check_cuda(cudaStreamSynchronize(s->stream), "slot idle");  // earlier users of the staging are done
  check_cuda(cudaEventRecord(s->ev0, s->copy_in), "ev0");
  for (int g = 0; g < 2; ++g) {
    const int f0 = g ? gf : 0, nf = g ? n_img - gf : gf;
    Plan* plan = plans[g];
    float* din = s->d_in.as<float>() + uint64_t(f0) * fin;
    float* dout = s->d_out.as<float>() + uint64_t(f0) * fout;
    check_cuda(cudaMemcpyAsync(din, in + uint64_t(f0) * fin, uint64_t(nf) * fin * 4, cudaMemcpyHostToDevice,
                               s->copy_in),
               "group H2D");
    check_cuda(cudaEventRecord(s->chunk_ev[2 * g], s->copy_in), "group event");
    check_cuda(cudaStreamWaitEvent(s->stream, s->chunk_ev[2 * g], 0), "wait group H2D");
    check_cuda(cudaMemcpyAsync(plan->in.p, din, uint64_t(nf) * fin * 4, cudaMemcpyDeviceToDevice, s->stream),
               "group in");
    check_cuda(cudaGraphLaunch(plan->graph, s->stream), "group graph");
    check_cuda(cudaMemcpyAsync(dout, plan->out.p, uint64_t(nf) * fout * 4, cudaMemcpyDeviceToDevice, s->stream),
               "group out");
    check_cuda(cudaEventRecord(s->chunk_ev[2 * g + 1], s->stream), "group event");
    check_cuda(cudaStreamWaitEvent(s->copy_out, s->chunk_ev[2 * g + 1], 0), "wait group graph");
    check_cuda(cudaMemcpyAsync(out + uint64_t(f0) * fout, dout, uint64_t(nf) * fout * 4, cudaMemcpyDeviceToHost,
                               s->copy_out),
               "group D2H");
  }
  check_cuda(cudaEventRecord(s->ev1, s->copy_out), "ev1");
  check_cuda(cudaEventSynchronize(s->ev1), "pipelined forward sync");
  return true;
}

}  // namespace

double forward_host(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                    const float* in, uint64_t in_elems, float* out, uint64_t out_elems) {
  const Model m = model_lookup(ctx, handle);
  const uint64_t E = uint64_t(n) * c * h * w;
  if (in_elems != E) fail(AVEC_ERR_INVALID_ARGUMENT, "frame data size disagrees with dims");
  const uint64_t K = output_elems_for(m, n, c, h, w);
  if (out_elems != K)
    fail(AVEC_ERR_INVALID_ARGUMENT, "output buffer holds " + std::to_string(out_elems) +
                                        " elements, forward yields " + std::to_string(K));
  check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
  SlotLease lease(ctx);
  Slot* s = lease.slot();
  lease.after_pending(s->stream);
  if (m.kind == AVEC_MODEL_POSENET) {
    int n_img = 0;
    posenet_shape(m, n, c, h, w, n_img);
    if (!(n_img >= 2 && E * 4 >= kPipeMin && is_pinned(in) && is_pinned(out) && pipelined_forward_enabled() &&
          pipelined_posenet(ctx, s, m, n_img, int(h), int(w), in, out, E, K))) {
      Plan* plan = get_plan(ctx, s, m, n_img, int(h), int(w));
      check_cuda(cudaEventRecord(s->ev0, s->stream), "ev0");
      stage_h2d(s, plan->in.p, in, E * 4);
      check_cuda(cudaGraphLaunch(plan->graph, s->stream), "graph launch");
      stage_d2h(s, out, plan->out.p, K * 4);
    }
  } else if (E * 4 >= kOverlapMin && is_pinned(in) && is_pinned(out)) {
    s->d_in.ensure(E * 4, ctx->device);
    s->d_out.ensure(K * 4, ctx->device);
    overlapped_segment_means(s, in, out, E, K);
  } else {
    s->d_in.ensure(E * 4, ctx->device);
    s->d_out.ensure(K * 4, ctx->device);
    check_cuda(cudaEventRecord(s->ev0, s->stream), "ev0");
    stage_h2d(s, s->d_in.p, in, E * 4);
    launch_segment_means(s->d_in.as<float>(), s->d_out.as<float>(), E, K, s->stream);
    check_cuda(cudaGetLastError(), "segment-mean launch");
    stage_d2h(s, out, s->d_out.p, K * 4);
  }
  float ms = 0.f;
  check_cuda(cudaEventElapsedTime(&ms, s->ev0, s->ev1), "event time");
  return double(ms) * 1e-3;
}

void forward_device(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                    const float* d_in, float* d_out, cudaStream_t stream) {
  const Model m = model_lookup(ctx, handle);
  const uint64_t E = uint64_t(n) * c * h * w;
  const uint64_t K = output_elems_for(m, n, c, h, w);
  check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
  SlotLease lease(ctx);
  Slot* s = lease.slot();
  cudaStream_t st = stream ? stream : s->stream;
  lease.after_pending(st);
  if (m.kind == AVEC_MODEL_POSENET) {
    int n_img = 0;
    posenet_shape(m, n, c, h, w, n_img);
    Plan* plan = get_plan(ctx, s, m, n_img, int(h), int(w));
    // the captured graph reads/writes the plan's own buffers
    check_cuda(cudaMemcpyAsync(plan->in.p, d_in, E * 4, cudaMemcpyDeviceToDevice, st), "D2D in");
    check_cuda(cudaGraphLaunch(plan->graph, st), "graph launch");
    check_cuda(cudaMemcpyAsync(d_out, plan->out.p, K * 4, cudaMemcpyDeviceToDevice, st), "D2D out");
  } else {
    launch_segment_means(d_in, d_out, E, K, st);
  }
  if (stream) {
    // asynchronous: the slot's plan buffers stay busy until `done` fires
    check_cuda(cudaEventRecord(s->done, st), "done event");
    s->pending = true;
  } else {
    check_cuda(cudaStreamSynchronize(st), "forward sync");
  }
}

std::vector<OpProfile> posenet_profile(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c,
                                       uint32_t h, uint32_t w, const float* d_in, int reps) {
  const Model m = model_lookup(ctx, handle);
  if (m.kind != AVEC_MODEL_POSENET) fail(AVEC_ERR_INVALID_ARGUMENT, "not a pose net");
  int n_img = 0;
  posenet_shape(m, n, c, h, w, n_img);
  check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
  SlotLease lease(ctx);
  Slot* s = lease.slot();
  lease.after_pending(s->stream);
  Plan* plan = get_plan(ctx, s, m, n_img, int(h), int(w));
  const uint64_t E = uint64_t(n) * c * h * w;
  check_cuda(cudaMemcpyAsync(plan->in.p, d_in, E * 4, cudaMemcpyDeviceToDevice, s->stream), "D2D");
  check_cuda(cudaGraphLaunch(plan->graph, s->stream), "warm graph");
  const size_t nops = plan->ops.size();
  std::vector<cudaEvent_t> ev(nops + 1);
  for (auto& e : ev) check_cuda(cudaEventCreate(&e), "event");
  std::vector<OpProfile> prof(nops);
#ifdef AVEC_TRACE
  const int trace_op = std::getenv("AVEC_TRACE_OP") ? std::atoi(std::getenv("AVEC_TRACE_OP")) : -1;
#endif
  for (int r = 0; r < reps; ++r) {
    for (size_t i = 0; i < nops; ++i) {
      check_cuda(cudaEventRecord(ev[i], s->stream), "event");
#ifdef AVEC_TRACE
      if (r == reps - 1 && int(i) == trace_op) conv_pm_trace(1, s->stream), conv_tc_trace(1, s->stream);
      run_ops(ctx, *plan, *m.net, i, i + 1, s->stream);
      if (r == reps - 1 && int(i) == trace_op) conv_pm_trace(0, s->stream), conv_tc_trace(0, s->stream);
#else
      run_ops(ctx, *plan, *m.net, i, i + 1, s->stream);
#endif
    }
    check_cuda(cudaEventRecord(ev[nops], s->stream), "event");
    check_cuda(cudaEventSynchronize(ev[nops]), "event sync");
    for (size_t i = 0; i < nops; ++i) {
      float ms = 0;
      check_cuda(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]), "elapsed");
      prof[i].ms += ms / float(reps);
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  const PoseFamily& f = m.net->fam;
  for (size_t i = 0; i < nops; ++i) {
    const PlanOp& op = plan->ops[i];
    OpProfile& p = prof[i];
    p.layers[0] = op.layers[0];
    p.layers[1] = op.layers[1];
    p.flops = 0;
    p.bytes = 0;
    if (op.kind == PlanOp::kPool) {
      const Geometry& g = plan->geo[op.level];
      p.kind = 2;
      p.bytes = double(n_img) * g.H * g.W * op.C * 2 * 1.25;  // read 4, write 1 bf16 per window
      continue;
    }
    if (op.kind == PlanOp::kConv12) {  // conv1_1 + conv1_2 + pool1: frame in, pooled 64 channels out
      p.kind = 5;
      const double px = double(n_img) * h * w;
      p.flops = 2.0 * px * (27.0 * 64 + 576.0 * 64);
      p.bytes = px * (12.0 + 64 * 2 / 4.0);
      continue;
    }
    if (op.kind == PlanOp::kHead) {  // Mconv6 + Mconv7: both layers' FLOPs, input + head output bytes
      p.kind = 4;
      for (int g = 0; g < 2; ++g) {
        if (op.layers[g] < 0) continue;
        const ConvDef& d6 = f.convs[op.head_l6[g]];
        const ConvDef& d7 = f.convs[op.layers[g]];
        const double px = double(n_img) * (h >> d6.level) * (w >> d6.level);
        p.flops += 2.0 * px * (double(d6.cin) * d6.cout + double(d7.cin) * d7.cout);
        const bool final_out = plan->layer_out[op.layers[g]].buf == -1;
        p.bytes += px * (d6.cin * 2.0 + d7.cout * (final_out ? 4.0 : 2.0));
      }
      continue;
    }
    p.kind = op.kind == PlanOp::kFirst ? 0 : op.cp.pixel_major ? 1 : 3;
    for (int g = 0; g < 2; ++g) {
      if (op.layers[g] < 0) continue;
      const ConvDef& d = f.convs[op.layers[g]];
      const double px = double(n_img) * (h >> d.level) * (w >> d.level);
      p.flops += 2.0 * px * d.cin * d.cout * d.k * d.k;
      const double in_b = op.kind == PlanOp::kFirst ? 4.0 : 2.0;  // fp32 frame or bf16 act
      const TensorView& ov = plan->layer_out[op.layers[g]];
      const bool final_out = ov.buf == -1;
      const double out_px = ov.level > d.level ? px / 4 : px;  // fused 2x2 pool
      p.bytes += px * d.cin * in_b + out_px * d.cout * (final_out ? 4.0 : 2.0);
    }
  }
  return prof;
}

void posenet_layer_fusion(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                          int layer, int* kind, int* in_layer) {
  const Model m = model_lookup(ctx, handle);
  if (m.kind != AVEC_MODEL_POSENET) fail(AVEC_ERR_INVALID_ARGUMENT, "not a pose net");
  int n_img = 0;
  posenet_shape(m, n, c, h, w, n_img);
  if (layer < 0 || layer >= int(m.net->fam.convs.size())) fail(AVEC_ERR_INVALID_ARGUMENT, "layer index");
  check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
  SlotLease lease(ctx);
  Plan* plan = get_plan(ctx, lease.slot(), m, n_img, int(h), int(w));
  *kind = plan->layer_fusion[layer];
  *in_layer = plan->layer_in_from[layer];
}

int posenet_layer_out_level(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                            int layer) {
  const Model m = model_lookup(ctx, handle);
  if (m.kind != AVEC_MODEL_POSENET) fail(AVEC_ERR_INVALID_ARGUMENT, "not a pose net");
  int n_img = 0;
  posenet_shape(m, n, c, h, w, n_img);
  const PoseFamily& f = m.net->fam;
  if (layer < 0 || layer >= int(f.convs.size())) fail(AVEC_ERR_INVALID_ARGUMENT, "layer index");
  check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
  SlotLease lease(ctx);
  Plan* plan = get_plan(ctx, lease.slot(), m, n_img, int(h), int(w));
  const TensorView& v = plan->layer_out[layer];
  return v.buf >= 0 ? v.level : f.convs[layer].level;
}

namespace {

// Parity hooks: run the plan of this shape from the host frames `in` through
// the op that produces `layer`, on the leased slot's stream (ordered after the
// slot's previous asynchronous forward, which may still read plan->in).
Plan* run_to_layer(avec_ctx* ctx, SlotLease& lease, const Model& m, uint32_t n, uint32_t c, uint32_t h,
                   uint32_t w, const float* in, int layer, int& n_img) {
  if (m.kind != AVEC_MODEL_POSENET) fail(AVEC_ERR_INVALID_ARGUMENT, "not a pose net");
  posenet_shape(m, n, c, h, w, n_img);
  const PoseFamily& f = m.net->fam;
  if (layer < 0 || layer >= int(f.convs.size())) fail(AVEC_ERR_INVALID_ARGUMENT, "layer index");
  Slot* s = lease.slot();
  lease.after_pending(s->stream);
  Plan* plan = get_plan(ctx, s, m, n_img, int(h), int(w));
  if (plan->layer_fusion[layer] == 2)
    fail(AVEC_ERR_UNSUPPORTED, f.convs[layer].name + " is fused into the next layer: its output never leaves the SM");
  const uint64_t E = uint64_t(n) * c * h * w;
  check_cuda(cudaMemcpyAsync(plan->in.p, in, E * 4, cudaMemcpyHostToDevice, s->stream), "H2D");
  size_t last = 0;
  for (size_t i = 0; i < plan->ops.size(); ++i)
    if (plan->ops[i].layers[0] == layer || plan->ops[i].layers[1] == layer) last = i + 1;
  run_ops(ctx, *plan, *m.net, 0, last, s->stream);
  check_cuda(cudaStreamSynchronize(s->stream), "layer io sync");
  return plan;
}

float bf16_to_float(uint16_t b) {
  const uint32_t u = uint32_t(b) << 16;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

}  // namespace

void posenet_layer_rows(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                        const float* in, int layer, int n_in, const int32_t* in_rows, float* layer_in, int n_out,
                        const int32_t* out_rows, float* layer_out) {
  const Model m = model_lookup(ctx, handle);
  check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
  if (n_in < 0 || n_out < 0 || (n_in && (!in_rows || !layer_in)) || (n_out && (!out_rows || !layer_out)))
    fail(AVEC_ERR_INVALID_ARGUMENT, "row selections");
  SlotLease lease(ctx);
  Slot* s = lease.slot();
  int n_img = 0;
  Plan* plan = run_to_layer(ctx, lease, m, n, c, h, w, in, layer, n_img);
  const PoseFamily& f = m.net->fam;
  const ConvDef& d = f.convs[layer];
  const ConvDef& din = f.convs[plan->layer_in_from[layer]];
  std::vector<float> out_all;  // fp32 NCHW plan output, fetched once if a view needs it
  // rows (image, y) of view `v` at level `lv` as unpadded fp32 [W][cdim];
  // rows outside the image are zeros (the next layer's zero padding)
  auto rows = [&](const TensorView& v, int lv, int cdim, const std::vector<int>& map, int count,
                  const int32_t* sel, float* dst) {
    const Geometry& g = plan->geo[lv];
    const int Hl = int(h) >> lv, Wl = int(w) >> lv;
    std::vector<uint16_t> raw;
    for (int r = 0; r < count; ++r) {
      const int b = sel[2 * r], y = sel[2 * r + 1];
      float* o = dst + size_t(r) * Wl * cdim;
      if (b < 0 || b >= n_img) fail(AVEC_ERR_INVALID_ARGUMENT, "row selection: image index");
      if (y < 0 || y >= Hl) {
        std::fill(o, o + size_t(Wl) * cdim, 0.f);
        continue;
      }
      if (v.buf == -2) {  // the frames as the first layer sees them: bf16 (or tf32) of x - 0.5
        for (int x = 0; x < Wl; ++x)
          for (int ch = 0; ch < 3; ++ch) {
            const float xv = in[((size_t(b) * 3 + ch) * Hl + y) * Wl + x] - 0.5f;
            o[x * 3 + ch] = f.input_tf32 ? tf32_value(xv) : bf16_value(xv);
          }
      } else if (v.buf == -1) {
        if (out_all.empty()) {
          out_all.resize(plan->out_elems);
          check_cuda(cudaMemcpy(out_all.data(), plan->out.p, out_all.size() * 4, cudaMemcpyDeviceToHost), "D2H");
        }
        const int C = f.out_channels();
        for (int ch = 0; ch < cdim; ++ch)
          for (int x = 0; x < Wl; ++x)
            o[size_t(x) * cdim + ch] = out_all[((size_t(b) * C + v.c_off + ch) * Hl + y) * Wl + x];
      } else {
        const int C = v.c_stride;
        raw.resize(size_t(Wl) * C);
        const size_t off = ((size_t(b) * g.Hp() + y + g.P) * g.Wp() + g.P) * C;
        check_cuda(cudaMemcpy(raw.data(), plan->bufs[v.buf]->as<uint16_t>() + off, raw.size() * 2,
                              cudaMemcpyDeviceToHost),
                   "D2H row");
        for (int x = 0; x < Wl; ++x)
          for (int ch = 0; ch < cdim; ++ch)
            o[size_t(x) * cdim + ch] = bf16_to_float(raw[size_t(x) * C + v.c_off + (map.empty() ? ch : map[ch])]);
      }
    }
  };
  const TensorView& vin = plan->layer_in[layer];
  const TensorView& vout = plan->layer_out[layer];
  const int in_level = vin.buf >= 0 ? vin.level : d.level;
  const int out_level = vout.buf >= 0 ? vout.level : d.level;
  // stage inputs: Caffe channel ci lives at window channel cin_map[ci] of the concat buffer
  std::vector<int> map;
  if (layer != 0 && !din.cin_map.empty() && vin.buf >= 0) map = din.cin_map;
  rows(vin, in_level, din.cin, map, n_in, in_rows, layer_in);
  rows(vout, out_level, d.cout, {}, n_out, out_rows, layer_out);
  (void)s;
}

void posenet_layer_io(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h,
                      uint32_t w, const float* in, int layer, float* layer_in,
                      uint64_t layer_in_elems, float* layer_out, uint64_t layer_out_elems) {
  const Model m = model_lookup(ctx, handle);
  const PoseFamily& f = m.net->fam;
  check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
  SlotLease lease(ctx);
  Slot* s = lease.slot();
  int n_img = 0;
  Plan* plan = run_to_layer(ctx, lease, m, n, c, h, w, in, layer, n_img);
  const ConvDef& d = f.convs[layer];
  // a fused head's second layer sees the head's input (the first layer's input)
  const ConvDef& din = f.convs[plan->layer_in_from[layer]];
  // the output view is one level down when the layer's 2x2 pool is fused
  const int out_level = plan->layer_out[layer].buf >= 0 ? plan->layer_out[layer].level : d.level;
  const uint64_t need_in = uint64_t(n_img) * (int(h) >> d.level) * (int(w) >> d.level) * din.cin;
  const uint64_t need_out = uint64_t(n_img) * (int(h) >> out_level) * (int(w) >> out_level) * d.cout;
  if (layer_in_elems != need_in || layer_out_elems != need_out)
    fail(AVEC_ERR_INVALID_ARGUMENT, "layer buffers have the wrong size");
  // `map`: Caffe channel -> channel inside the view's window (stage inputs)
  auto fetch = [&](const TensorView& v, int cdim, float* dst, const std::vector<int>& map) {
    const int lv = v.buf >= 0 ? v.level : d.level;
    const Geometry& g = plan->geo[lv];
    const int Hl = int(h) >> lv, Wl = int(w) >> lv;
    if (v.buf == -2) {  // network input as the first layer sees it: bf16 (or tf32) of x - 0.5, NHWC
      for (int b = 0; b < n_img; ++b)
        for (int y = 0; y < Hl; ++y)
          for (int x = 0; x < Wl; ++x)
            for (int ch = 0; ch < 3; ++ch) {
              const float xv = in[((size_t(b) * 3 + ch) * Hl + y) * Wl + x] - 0.5f;
              dst[((size_t(b) * Hl + y) * Wl + x) * 3 + ch] = f.input_tf32 ? tf32_value(xv) : bf16_value(xv);
            }
      return;
    }
    if (v.buf == -1) {  // fp32 NCHW plan output -> NHWC channel range
      std::vector<float> all(plan->out_elems);
      check_cuda(cudaMemcpy(all.data(), plan->out.p, all.size() * 4, cudaMemcpyDeviceToHost), "D2H");
      const int C = f.out_channels();
      for (int b = 0; b < n_img; ++b)
        for (int ch = 0; ch < cdim; ++ch)
          for (int y = 0; y < Hl; ++y)
            for (int x = 0; x < Wl; ++x)
              dst[((size_t(b) * Hl + y) * Wl + x) * cdim + ch] =
                  all[((size_t(b) * C + v.c_off + ch) * Hl + y) * Wl + x];
      return;
    }
    const int off = v.c_off;
    const int grab = map.empty() ? v.c : v.c_stride - v.c_off;
    DevMem tmp;
    tmp.ensure(size_t(n_img) * Hl * Wl * grab * 4, ctx->device);
    launch_unpad_to_f32(plan->bufs[v.buf]->p, n_img, Hl, Wl, g.P, v.c_stride, off, grab,
                        tmp.as<float>(), s->stream);
    std::vector<float> hostv(size_t(n_img) * Hl * Wl * grab);
    check_cuda(cudaMemcpyAsync(hostv.data(), tmp.p, hostv.size() * 4, cudaMemcpyDeviceToHost, s->stream), "D2H");
    check_cuda(cudaStreamSynchronize(s->stream), "sync");
    for (size_t p = 0; p < size_t(n_img) * Hl * Wl; ++p)
      for (int ch = 0; ch < cdim; ++ch) {
        const int src_ch = map.empty() ? ch : map[ch];
        dst[p * cdim + ch] = hostv[p * grab + src_ch];
      }
  };
  fetch(plan->layer_in[layer], din.cin, layer_in, layer == 0 ? std::vector<int>{} : din.cin_map);
  fetch(plan->layer_out[layer], d.cout, layer_out, {});
}

}  // namespace avec

#ifdef AVEC_TRACE
// trace builds only: the stamps of the launch traced by avec_posenet_profile
extern "C" int avec_trace_dump(unsigned long long* host, int n) { return avec::conv_pm_trace_dump(host, n); }
extern "C" int avec_trace_dump_tc(unsigned long long* host, int n) { return avec::conv_tc_trace_dump(host, n); }
#endif
