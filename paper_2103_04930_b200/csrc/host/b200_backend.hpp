// The B200 compute plugin: accelfwd-style Backend over the C-ABI of
// libavec_cuda.so (include/avec_cuda.h), one avec_ctx per GPU.
//
// Multi-GPU: frames are independent, so there is no
// collective. Two placement policies:
//  * affinity (default): each forward runs whole on the least-loaded GPU;
//    sessions spread across GPUs (C4: 8 clients, one per B200);
//  * session: session k always runs on GPU (k - 1) mod G (C4: 8 clients, one
//    session per B200 of the box);
//  * split: a batched pose-net forward (channels = 3N) is cut into contiguous
//    frame groups, one per GPU, run concurrently; each GPU writes its slice of
//    the NCHW output, which is batch-major, so slices are contiguous (C5).
#pragma once

#include <atomic>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "backend.hpp"

struct avec_ctx;

// exported by libavec_host.so for the Python mirror (sharding.py): the split
// policy's partition of `frames` into `groups` (first[g], count[g])
extern "C" int avec_frame_groups(std::uint64_t frames, int groups, std::uint64_t* first, std::uint64_t* count);

namespace avec::backend {

// Frame-group partition of the split policy (and of bench.py's ranks, through
// avec_frame_groups): contiguous groups whose sizes differ by at most one,
// earlier groups take the remainder.
struct FrameGroup {
  std::uint64_t first = 0, count = 0;
};
std::vector<FrameGroup> frame_groups(std::uint64_t frames, int groups);

class B200Backend final : public Backend {
 public:
  enum class Policy { affinity, split, session };
  // devices empty = all visible GPUs
  explicit B200Backend(std::vector<int> devices = {}, int slots_per_device = 2,
                       Policy policy = Policy::affinity);
  ~B200Backend() override;

  ModelHandle register_model(const wire::ModelDescriptor& model) override;
  Heatmap forward(ModelHandle model, const Frame& frame) override;
  std::string_view label() const override { return label_; }

  bool zero_copy() const override { return true; }
  std::uint64_t output_elems(ModelHandle model, const wire::Dims& dims) override;
  double forward_into(ModelHandle model, const wire::Dims& dims, const float* in, std::uint64_t n_in,
                      float* out, std::uint64_t n_out) override;
  double forward_session(std::uint64_t session, ModelHandle model, const wire::Dims& dims, const float* in,
                         std::uint64_t n_in, float* out, std::uint64_t n_out) override;
  int concurrency() const override;
  std::unique_ptr<Pipeline> open_pipeline(std::uint64_t session) override;
  void* alloc_host(std::size_t bytes) override;
  void free_host(void* p) override;

  int device_count() const { return int(ctx_.size()); }
  struct PipePool;  // per-GPU avec_streams of pipelined cycles (b200_backend.cpp)
  int devices() const override { return int(ctx_.size()); }

 private:
  struct Entry {
    int kind = 0;
    std::vector<std::uint64_t> per_device;  // handle on each context
  };
  Entry lookup(ModelHandle h);
  int pick_device();
  double run_on(int dev, const Entry& e, const wire::Dims& d, const float* in, std::uint64_t n_in,
                float* out, std::uint64_t n_out);

  std::vector<avec_ctx*> ctx_;
  std::vector<int> devices_;
  int slots_;
  Policy policy_;
  std::string label_;
  std::unique_ptr<std::atomic<int>[]> inflight_;
  std::unique_ptr<std::atomic<int>[]> pipelines_;  // open pipelines per device (placement)
  std::unique_ptr<std::atomic<int>[]> streaming_;  // pipelined cycles running per device
  std::vector<std::unique_ptr<PipePool>> pools_;
  bool pipelining_ = true;                          // AVEC_PIPELINE=0 disables
  std::mutex m_;
  std::map<wire::Digest, std::uint64_t> id_by_digest_;
  std::map<std::uint64_t, Entry> models_;
  std::uint64_t next_id_ = 1;
};

}  // namespace avec::backend
