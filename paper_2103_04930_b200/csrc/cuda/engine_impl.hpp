// Engine state behind avec_ctx: device handle table, execution slots,
// pinned staging, pose-net plans. Internal to libavec_cuda.so.
#pragma once

#include <array>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "conv_tc.cuh"
#include "engine.hpp"
#include "netspec.hpp"

namespace avec {

// owning device allocation (freed on the device it came from)
struct DevMem {
  void* p = nullptr;
  size_t bytes = 0;
  int device = -1;
  DevMem() = default;
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  ~DevMem();
  void reset();
  // grow-only; contents are not preserved
  void ensure(size_t n, int dev);
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

struct PinnedMem {
  void* p = nullptr;
  size_t bytes = 0;
  PinnedMem() = default;
  PinnedMem(const PinnedMem&) = delete;
  PinnedMem& operator=(const PinnedMem&) = delete;
  ~PinnedMem();
  void ensure(size_t n);
};

// one conv layer resident on the device (bf16 packed for the TMA/UMMA path)
struct ConvLayerDev {
  ConvDef def;
  int exec_k = 0;  // filter size as executed (the first layer: 1, K = its 27 taps, conv_first.cu)
  int cin_pad = 0, cout_pad = 0;
  void* w = nullptr;       // bf16 [cout_pad][k*k][cin_pad]
  float* w_tf32 = nullptr; // the first layer of an "input tf32" net: [cout_pad][32] tf32 (27 taps, zeros)
  float* bias = nullptr;   // [cout_pad]
  float* slope = nullptr;  // [cout_pad] PReLU slopes (zeros unless act == prelu)
};

struct PoseNet {
  PoseFamily fam;
  std::vector<ConvLayerDev> layers;
  DevMem mem;  // all weights of this device
};

struct Geometry {
  int H = 0, W = 0, P = 0;
  int Hp() const { return H + 2 * P; }
  int Wp() const { return W + 2 * P; }
};

// a channel range of a plan buffer (or the fp32 NCHW output when buf < 0)
struct TensorView {
  int buf = -1;  // index into Plan::bufs; -1 = plan output (fp32 NCHW), -2 = plan input
  int level = 0;
  int c_stride = 0, c_off = 0, c = 0;
};

struct PlanOp {
  enum Kind { kFirst, kConv, kPool, kHead, kConv12 } kind = kConv;
  ConvParams cp{};
  ConvMaps maps{};
  HeadParams hp{};  // kHead: fused Mconv6 + Mconv7 (layers[] = the Mconv7 layers)
  HeadMaps hm{};
  int head_l6[2] = {-1, -1};  // kHead: the Mconv6 layers; kConv12: conv1_1 in [0]
  int layers[2] = {-1, -1};
  int src = -1, dst = -1, level = 0, C = 0;  // pool: src/dst buffers
};

struct Plan {
  int n = 0, H = 0, W = 0;
  Geometry geo[4];
  std::vector<std::unique_ptr<DevMem>> bufs;
  std::vector<int> buf_level, buf_c;
  std::vector<PlanOp> ops;
  std::vector<TensorView> layer_in, layer_out;
  // parity-hook view of each layer: 0 plain, 1 output 2x2-pooled (level + 1),
  // 2 fused into the next layer (no output of its own), 3 second layer of a
  // fused head (its input view is the head's input, described by layer_in_from)
  std::vector<int> layer_fusion, layer_in_from;
  DevMem in, out;  // fp32 NCHW frames in, fp32 NCHW net output
  DevMem ws;       // split-K partial sums (conv_tc), ws_bytes
  size_t ws_bytes = 0;
  uint64_t in_elems = 0, out_elems = 0;
  cudaGraphExec_t graph = nullptr;
  uint64_t last_use = 0;  // slot-local LRU clock
  ~Plan();
};

struct Slot {
  int index = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t done = nullptr;  // last enqueued async work on a caller stream
  bool pending = false;
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  PinnedMem stage[2];
  // side streams of the chunked segment-mean cycle (H2D, D2H) and its events
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  DevMem d_in, d_out;  // segment-mean path
  // cached plans (activation buffers + CUDA graph) per (model, frames, H, W),
  // least recently used evicted beyond AVEC_PLANS_PER_SLOT (default 4): a
  // long-lived server seeing many resolutions must not grow without bound
  std::map<std::tuple<uint64_t, int, int, int>, std::unique_ptr<Plan>> plans;
  uint64_t use_clock = 0;
};

struct Model {
  uint64_t id = 0;
  int kind = AVEC_MODEL_MOCKPOSE;
  double divisor = 1.0;
  std::string name;
  std::shared_ptr<PoseNet> net;
};

}  // namespace avec

struct avec_ctx {
  int device = 0;
  int sms = 148;
  std::string label;
  std::vector<std::unique_ptr<avec::Slot>> slots;
  std::vector<bool> slot_busy;
  size_t next_slot = 0;  // round-robin cursor (guarded by slot_m)
  std::mutex slot_m;
  std::condition_variable slot_cv;
  std::mutex model_m;
  std::map<std::array<uint8_t, 32>, uint64_t> id_by_digest;
  std::map<uint64_t, avec::Model> models;
  uint64_t next_id = 1;
  avec::DevMem scratch;  // post-processing scratch (guarded by post_m)
  std::mutex post_m;
};

namespace avec {

// engine entry points used by capi.cpp
void ctx_init(avec_ctx* ctx, int device, int slots);
void ctx_shutdown(avec_ctx* ctx);
uint64_t model_register(avec_ctx* ctx, const uint8_t* digest, const std::string& name,
                        const uint8_t* structure, size_t structure_len, const uint8_t* weights,
                        uint64_t weights_len, double divisor);
Model model_lookup(avec_ctx* ctx, uint64_t handle);
uint64_t output_elems_for(const Model& m, uint32_t n, uint32_t c, uint32_t h, uint32_t w);
// frames per pose-net forward of these dims (validates the shape and size law)
void posenet_shape(const Model& m, uint32_t n, uint32_t c, uint32_t h, uint32_t w, int& n_img);
// the slot's cached plan (activation buffers + CUDA graph) for this shape,
// built and captured on the slot's stream on first use
Plan* get_plan(avec_ctx* ctx, Slot* slot, const Model& m, int n_img, int H, int W);
double forward_host(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                    const float* in, uint64_t in_elems, float* out, uint64_t out_elems);
void forward_device(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                    const float* d_in, float* d_out, cudaStream_t stream);
struct OpProfile {
  int kind;        // 0 first conv (CUDA cores), 1 tcgen05 conv, 2 max-pool
  double flops;    // algorithmic 2*MACs of the launch
  double bytes;    // algorithmic bytes (inputs read once + outputs written once)
  float ms;        // CUDA-event duration on the launching stream
  int layers[2];
};
std::vector<OpProfile> posenet_profile(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c,
                                       uint32_t h, uint32_t w, const float* d_in, int reps);
// pyramid level of a layer's output view: its own level, or one more when
// the plan fuses the following 2x2 max-pool into it
// parity-hook view of a layer in the plan of this shape: kind 0 plain,
// 1 pooled output, 2 fused into the next layer, 3 second layer of a fused
// head whose input is `in_layer`'s input
void posenet_layer_fusion(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                          int layer, int* kind, int* in_layer);
int posenet_layer_out_level(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                            int layer);
// pipelined cycles (pipeline.cu, avec_stream_* in include/avec_cuda.h)
avec_stream* stream_create(avec_ctx* ctx);
void stream_destroy(avec_stream* s);
void stream_prepare(avec_stream* s, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w);
void stream_begin(avec_stream* s, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w, const float* in,
                  float* out, uint64_t out_elems);
void stream_feed(avec_stream* s, uint64_t landed_bytes);
double stream_finish(avec_stream* s);
void stream_abort(avec_stream* s);
// selected rows (image, y) of a layer's input and output views, full-size parity
void posenet_layer_rows(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                        const float* in, int layer, int n_in, const int32_t* in_rows, float* layer_in, int n_out,
                        const int32_t* out_rows, float* layer_out);
void posenet_layer_io(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h,
                      uint32_t w, const float* in, int layer, float* layer_in,
                      uint64_t layer_in_elems, float* layer_out, uint64_t layer_out_elems);

}  // namespace avec
