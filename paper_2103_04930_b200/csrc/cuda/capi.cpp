// extern "C" boundary of libavec_cuda.so (include/avec_cuda.h). No exception
// crosses it: every entry point converts avec::Error / std::exception into an
// AVEC_* code plus a thread-local message.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <unordered_map>
#include <vector>

#include "engine_impl.hpp"

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return AVEC_OK;
  } catch (const avec::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host out of memory";
    return AVEC_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return AVEC_ERR_CUDA;
  }
}

void need(const void* p, const char* what) {
  if (!p) avec::fail(AVEC_ERR_INVALID_ARGUMENT, std::string(what) + " is NULL");
}

// Pinned host memory is pooled. cudaFreeHost synchronises the device, so a
// session closing mid-run used to stall every other session's cycle (measured
// 400-520 ms communication spikes through avec-server with 4 clients);
// cudaHostAlloc of a frame-sized buffer costs milliseconds of page locking.
// Freed blocks (2 MiB granules) are kept for reuse up to kCacheBytes and
// handed out best-fit.
class HostPool {
 public:
  static constexpr uint64_t kGranule = 2ull << 20;
  static constexpr uint64_t kCacheBytes = 8ull << 30;

  void* take(uint64_t bytes) {
    const uint64_t sz = (std::max<uint64_t>(bytes, 1) + kGranule - 1) / kGranule * kGranule;
    {
      std::lock_guard<std::mutex> lk(m_);
      auto it = free_.lower_bound(sz);
      if (it != free_.end() && it->first <= 2 * sz) {  // best fit, at most 2x the request
        void* p = it->second;
        cached_ -= it->first;
        live_[p] = it->first;
        free_.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    if (cudaHostAlloc(&p, sz, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    std::lock_guard<std::mutex> lk(m_);
    live_[p] = sz;
    return p;
  }

  void give(void* p) {
    if (!p) return;
    std::unique_lock<std::mutex> lk(m_);
    auto it = live_.find(p);
    if (it == live_.end()) {  // not ours: plain pinned free
      lk.unlock();
      cudaFreeHost(p);
      return;
    }
    const uint64_t sz = it->second;
    live_.erase(it);
    if (cached_ + sz <= kCacheBytes) {
      free_.emplace(sz, p);
      cached_ += sz;
      return;
    }
    lk.unlock();
    cudaFreeHost(p);
  }

 private:
  std::mutex m_;
  std::multimap<uint64_t, void*> free_;
  std::unordered_map<void*, uint64_t> live_;
  uint64_t cached_ = 0;
};

HostPool& host_pool() {
  static HostPool* pool = new HostPool;  // never destroyed: blocks outlive static teardown order
  return *pool;
}

}  // namespace

extern "C" {

const char* avec_last_error(void) { return g_last_error.c_str(); }

const char* avec_version(void) { return "avec-b200 0.1 (sm_100a)"; }

int avec_device_count(int* count) {
  return guarded([&] {
    need(count, "count");
    avec::check_cuda(cudaGetDeviceCount(count), "cudaGetDeviceCount");
  });
}

int avec_ctx_create(int device, int slots, avec_ctx** out) {
  return guarded([&] {
    need(out, "out");
    *out = nullptr;
    auto* ctx = new avec_ctx();
    try {
      avec::ctx_init(ctx, device, slots);
    } catch (...) {
      delete ctx;
      throw;
    }
    *out = ctx;
  });
}

void avec_ctx_destroy(avec_ctx* ctx) {
  if (!ctx) return;
  try {
    avec::ctx_shutdown(ctx);
  } catch (...) {
  }
  delete ctx;
}

const char* avec_ctx_label(const avec_ctx* ctx) { return ctx ? ctx->label.c_str() : ""; }

int avec_model_register(avec_ctx* ctx, const uint8_t* digest32, const char* name, size_t name_len,
                        const uint8_t* structure, size_t structure_len, const uint8_t* weights,
                        uint64_t weights_len, double output_divisor, uint64_t* handle_out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(digest32, "digest");
    need(handle_out, "handle_out");
    if (weights_len && !weights) avec::fail(AVEC_ERR_INVALID_ARGUMENT, "weights is NULL");
    *handle_out = avec::model_register(ctx, digest32, std::string(name ? name : "", name ? name_len : 0),
                                       structure, structure_len, weights, weights_len,
                                       output_divisor);
  });
}

int avec_model_kind(avec_ctx* ctx, uint64_t handle, int* kind_out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(kind_out, "kind_out");
    *kind_out = avec::model_lookup(ctx, handle).kind;
  });
}

int avec_output_elems(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h,
                      uint32_t w, uint64_t* out_elems) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out_elems, "out_elems");
    *out_elems = avec::output_elems_for(avec::model_lookup(ctx, handle), n, c, h, w);
  });
}

int avec_forward(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                 const float* in, uint64_t in_elems, float* out, uint64_t out_elems,
                 double* compute_s) {
  return guarded([&] {
    need(ctx, "ctx");
    need(in, "in");
    need(out, "out");
    const double s = avec::forward_host(ctx, handle, n, c, h, w, in, in_elems, out, out_elems);
    if (compute_s) *compute_s = s;
  });
}

int avec_forward_device(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h,
                        uint32_t w, const float* d_in, float* d_out, void* cuda_stream) {
  return guarded([&] {
    need(ctx, "ctx");
    need(d_in, "d_in");
    need(d_out, "d_out");
    avec::forward_device(ctx, handle, n, c, h, w, d_in, d_out,
                         static_cast<cudaStream_t>(cuda_stream));
  });
}

int avec_upsample_device(avec_ctx* ctx, const float* d_in, int planes, int h, int w, int scale,
                         float* d_out, void* cuda_stream) {
  return guarded([&] {
    need(ctx, "ctx");
    need(d_in, "d_in");
    need(d_out, "d_out");
    if (planes < 1 || h < 1 || w < 1 || scale < 1) avec::fail(AVEC_ERR_INVALID_ARGUMENT, "bad upsample shape");
    avec::check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    avec::launch_upsample(d_in, planes, h, w, scale, d_out, st);
    if (!st) avec::check_cuda(cudaStreamSynchronize(st), "upsample sync");
  });
}

int avec_nms_device(avec_ctx* ctx, const float* d_in, int planes, int h, int w, float threshold,
                    int max_peaks, int* d_counts, float* d_peaks, void* cuda_stream) {
  return guarded([&] {
    need(ctx, "ctx");
    need(d_in, "d_in");
    need(d_counts, "d_counts");
    need(d_peaks, "d_peaks");
    if (planes < 1 || h < 1 || w < 1 || max_peaks < 1) avec::fail(AVEC_ERR_INVALID_ARGUMENT, "bad nms shape");
    avec::check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
    std::lock_guard<std::mutex> lk(ctx->post_m);
    const size_t need_bytes = avec::nms_scratch_bytes(planes, h, w, max_peaks);
    ctx->scratch.ensure(need_bytes, ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    avec::launch_nms(d_in, planes, h, w, threshold, max_peaks, d_counts, d_peaks, ctx->scratch.p,
                     ctx->scratch.bytes, st);
    // scratch is shared per context: drain before releasing it
    avec::check_cuda(cudaStreamSynchronize(st), "nms sync");
  });
}

int avec_upsample_nms_device(avec_ctx* ctx, const float* d_in, int planes, int h, int w, int scale, float threshold,
                             int max_peaks, float* d_out, int* d_counts, float* d_peaks, void* cuda_stream) {
  return guarded([&] {
    need(ctx, "ctx");
    need(d_in, "d_in");
    need(d_out, "d_out");
    need(d_counts, "d_counts");
    need(d_peaks, "d_peaks");
    if (planes < 1 || h < 1 || w < 1 || max_peaks < 1) avec::fail(AVEC_ERR_INVALID_ARGUMENT, "bad upsample+nms shape");
    if (scale != 8) avec::fail(AVEC_ERR_UNSUPPORTED, "the fused upsample+nms is x8 (the pose net's stride)");
    avec::check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
    std::lock_guard<std::mutex> lk(ctx->post_m);
    ctx->scratch.ensure(avec::nms_scratch_bytes(planes, 8 * h, 8 * w, max_peaks), ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    avec::launch_upsample_nms(d_in, planes, h, w, threshold, max_peaks, d_out, d_counts, d_peaks, ctx->scratch.p,
                              ctx->scratch.bytes, st);
    avec::check_cuda(cudaStreamSynchronize(st), "upsample+nms sync");  // scratch is shared per context
  });
}

int avec_paf_candidates_device(avec_ctx* ctx, const float* d_paf, int H, int W, const int* d_counts,
                               const float* d_peaks, int max_peaks, const int* limb_parts, const int* limb_paf,
                               int n_limbs, float paf_threshold, float* d_cand, void* cuda_stream) {
  return guarded([&] {
    need(ctx, "ctx");
    need(d_paf, "d_paf");
    need(d_counts, "d_counts");
    need(d_peaks, "d_peaks");
    need(limb_parts, "limb_parts");
    need(limb_paf, "limb_paf");
    need(d_cand, "d_cand");
    avec::check_cuda(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    avec::launch_paf_candidates(d_paf, H, W, d_counts, d_peaks, max_peaks, limb_parts, limb_paf, n_limbs,
                                paf_threshold, d_cand, st);
    avec::check_cuda(cudaStreamSynchronize(st), "paf candidates sync");
  });
}

int avec_assemble_people(const int* counts, const float* peaks, int n_parts, int max_peaks, const float* cand,
                         const int* limb_parts, int n_limbs, int new_row_limbs, int max_people, int* people,
                         float* people_score, int* n_people) {
  return guarded([&] {
    need(counts, "counts");
    need(peaks, "peaks");
    need(cand, "cand");
    need(limb_parts, "limb_parts");
    need(people, "people");
    need(people_score, "people_score");
    need(n_people, "n_people");
    *n_people = avec::assemble_people(counts, peaks, n_parts, max_peaks, cand, limb_parts, n_limbs, new_row_limbs,
                                      max_people, people, people_score);
  });
}

int avec_coco_limbs(int* limb_parts, int* limb_paf, int* n_limbs, int* new_row_limbs) {
  return guarded([&] {
    need(n_limbs, "n_limbs");
    // OpenPose COCO limb sequence (1-based parts) and the PAF channel pairs of
    // its 57-channel output, re-based to parts 0..17 and the 38 PAF planes
    static const int seq[19][2] = {{2, 3},   {2, 6},   {3, 4},  {4, 5},   {6, 7},   {7, 8},  {2, 9},
                                   {9, 10},  {10, 11}, {2, 12}, {12, 13}, {13, 14}, {2, 1},  {1, 15},
                                   {15, 17}, {1, 16},  {16, 18}, {3, 17}, {6, 18}};
    static const int map[19][2] = {{31, 32}, {39, 40}, {33, 34}, {35, 36}, {41, 42}, {43, 44}, {19, 20},
                                   {21, 22}, {23, 24}, {25, 26}, {27, 28}, {29, 30}, {47, 48}, {49, 50},
                                   {53, 54}, {51, 52}, {55, 56}, {37, 38}, {45, 46}};
    *n_limbs = 19;
    if (new_row_limbs) *new_row_limbs = 17;
    for (int l = 0; l < 19; ++l)
      for (int k = 0; k < 2; ++k) {
        if (limb_parts) limb_parts[2 * l + k] = seq[l][k] - 1;
        if (limb_paf) limb_paf[2 * l + k] = map[l][k] - 19;
      }
  });
}

int avec_posenet_layer_fusion(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                              int layer, int* kind, int* in_layer) {
  return guarded([&] {
    need(ctx, "ctx");
    need(kind, "kind");
    need(in_layer, "in_layer");
    avec::posenet_layer_fusion(ctx, handle, n, c, h, w, layer, kind, in_layer);
  });
}

int avec_posenet_layer_out_level(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h,
                                 uint32_t w, int layer, int* level) {
  return guarded([&] {
    need(ctx, "ctx");
    need(level, "level");
    *level = avec::posenet_layer_out_level(ctx, handle, n, c, h, w, layer);
  });
}

int avec_posenet_layer_io(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h,
                          uint32_t w, const float* in, int layer, float* layer_in,
                          uint64_t layer_in_elems, float* layer_out, uint64_t layer_out_elems) {
  return guarded([&] {
    need(ctx, "ctx");
    need(in, "in");
    need(layer_in, "layer_in");
    need(layer_out, "layer_out");
    avec::posenet_layer_io(ctx, handle, n, c, h, w, in, layer, layer_in, layer_in_elems, layer_out,
                           layer_out_elems);
  });
}

int avec_stream_create(avec_ctx* ctx, avec_stream** out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out, "out");
    *out = avec::stream_create(ctx);
  });
}

void avec_stream_destroy(avec_stream* s) {
  try {
    avec::stream_destroy(s);
  } catch (...) {
  }
}

int avec_stream_prepare(avec_stream* s, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w) {
  return guarded([&] {
    need(s, "stream");
    avec::stream_prepare(s, handle, n, c, h, w);
  });
}

int avec_stream_begin(avec_stream* s, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                      const float* in, float* out, uint64_t out_elems) {
  return guarded([&] {
    need(s, "stream");
    need(in, "in");
    need(out, "out");
    avec::stream_begin(s, handle, n, c, h, w, in, out, out_elems);
  });
}

int avec_stream_feed(avec_stream* s, uint64_t landed_bytes) {
  return guarded([&] {
    need(s, "stream");
    avec::stream_feed(s, landed_bytes);
  });
}

int avec_stream_finish(avec_stream* s, double* compute_s) {
  return guarded([&] {
    need(s, "stream");
    const double t = avec::stream_finish(s);
    if (compute_s) *compute_s = t;
  });
}

int avec_stream_abort(avec_stream* s) {
  return guarded([&] {
    need(s, "stream");
    avec::stream_abort(s);
  });
}

int avec_posenet_layer_rows(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h, uint32_t w,
                            const float* in, int layer, int n_in, const int32_t* in_rows, float* layer_in,
                            int n_out, const int32_t* out_rows, float* layer_out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(in, "in");
    avec::posenet_layer_rows(ctx, handle, n, c, h, w, in, layer, n_in, in_rows, layer_in, n_out, out_rows,
                             layer_out);
  });
}

int avec_posenet_profile(avec_ctx* ctx, uint64_t handle, uint32_t n, uint32_t c, uint32_t h,
                         uint32_t w, const float* d_in, int reps, int max_ops, int* n_ops,
                         int* op_kind, double* op_flops, double* op_bytes, float* op_ms) {
  return guarded([&] {
    need(ctx, "ctx");
    need(d_in, "d_in");
    need(n_ops, "n_ops");
    auto prof = avec::posenet_profile(ctx, handle, n, c, h, w, d_in, reps < 1 ? 1 : reps);
    *n_ops = int(prof.size());
    for (int i = 0; i < int(prof.size()) && i < max_ops; ++i) {
      if (op_kind) op_kind[i] = prof[i].kind;
      if (op_flops) op_flops[i] = prof[i].flops;
      if (op_bytes) op_bytes[i] = prof[i].bytes;
      if (op_ms) op_ms[i] = prof[i].ms;
    }
  });
}

int avec_posenet_num_layers(avec_ctx* ctx, uint64_t handle, int* n_layers) {
  return guarded([&] {
    need(ctx, "ctx");
    need(n_layers, "n_layers");
    auto m = avec::model_lookup(ctx, handle);
    if (m.kind != AVEC_MODEL_POSENET) avec::fail(AVEC_ERR_INVALID_ARGUMENT, "not a pose net");
    *n_layers = int(m.net->fam.convs.size());
  });
}

int avec_posenet_layer_info(avec_ctx* ctx, uint64_t handle, int layer, int* cin, int* cout, int* k,
                            int* level, int* relu) {
  return guarded([&] {
    need(ctx, "ctx");
    auto m = avec::model_lookup(ctx, handle);
    if (m.kind != AVEC_MODEL_POSENET) avec::fail(AVEC_ERR_INVALID_ARGUMENT, "not a pose net");
    if (layer < 0 || layer >= int(m.net->fam.convs.size()))
      avec::fail(AVEC_ERR_INVALID_ARGUMENT, "layer index");
    const auto& d = m.net->fam.convs[layer];
    if (cin) *cin = d.cin;
    if (cout) *cout = d.cout;
    if (k) *k = d.k;
    if (level) *level = d.level;
    if (relu) *relu = d.act;
  });
}

int avec_posenet_synth_weights(const uint8_t* structure, size_t structure_len, float* out,
                               uint64_t* out_floats) {
  return guarded([&] {
    need(structure, "structure");
    need(out_floats, "out_floats");
    auto fam = avec::parse_avecnet(structure, structure_len);
    const uint64_t n = fam.weight_floats();
    if (out) {
      if (*out_floats < n) avec::fail(AVEC_ERR_INVALID_ARGUMENT, "output too small");
      avec::synth_weights(fam, out);
    }
    *out_floats = n;
  });
}

void* avec_host_alloc(uint64_t bytes) {
  void* p = host_pool().take(bytes);
  if (!p) g_last_error = "cudaHostAlloc failed";
  return p;
}

void avec_host_free(void* p) { host_pool().give(p); }

}  // extern "C"
