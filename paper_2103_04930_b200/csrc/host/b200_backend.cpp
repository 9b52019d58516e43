#include "b200_backend.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <set>
#include <tuple>
#include <stdexcept>
#include <thread>

#include "avec_cuda.h"

namespace avec::backend {

namespace {

[[noreturn]] void rethrow(int rc) {
  const std::string msg = avec_last_error();
  switch (rc) {
    case AVEC_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case AVEC_ERR_UNKNOWN_MODEL: throw Error(ErrorCode::unknown_model, msg);
    case AVEC_ERR_INVALID_MODEL: throw Error(ErrorCode::invalid_model, msg);
    case AVEC_ERR_DEGENERATE_OUTPUT: throw Error(ErrorCode::degenerate_output, msg);
    default: throw Error(ErrorCode::internal, msg);
  }
}

void check(int rc) {
  if (rc != AVEC_OK) rethrow(rc);
}

}  // namespace

// Pipelined cycles on one GPU run on a small pool of avec_streams shared by
// all of the device's sessions (AVEC_PIPE_BUSY, default 2): group plans and
// staging are built once per device and shape, not per session (a plan
// build allocates hundreds of MB, and the driver serialises allocations
// against every other session's work).
//
// A cycle is pipelined only while its GPU has at most one other cycle to do
// (and the server at most 2 sessions per GPU): frame groups trade some
// efficiency (smaller launches) for overlapping the receive, which pays while
// the GPU would otherwise wait for the network, not when other sessions'
// whole batches keep it busy (measured C2, 4 sessions on 1 GPU: 2567 -> 2067
// frames/s when every cycle was pipelined).
struct B200Backend::PipePool {
  using Key = std::tuple<std::uint64_t, std::uint32_t, std::uint32_t, std::uint32_t, std::uint32_t>;
  avec_ctx* ctx = nullptr;
  int cap = 1;
  std::mutex m;
  std::vector<avec_stream*> streams;
  std::vector<char> held;            // a cycle or a preparation owns the stream
  std::vector<std::set<Key>> ready;  // shapes each stream is prepared for
  ~PipePool() {
    for (auto* s : streams) avec_stream_destroy(s);
  }
  // a free stream (creating one below the cap); -1 if none. With `key`, only
  // a stream already prepared for it.
  int acquire(const Key* key) {
    std::lock_guard<std::mutex> lk(m);
    for (size_t i = 0; i < streams.size(); ++i)
      if (!held[i] && (!key || ready[i].count(*key))) {
        held[i] = 1;
        return int(i);
      }
    if (key || int(streams.size()) >= cap) return -1;
    avec_stream* s = nullptr;
    if (avec_stream_create(ctx, &s) != AVEC_OK) return -1;
    streams.push_back(s);
    held.push_back(1);
    ready.emplace_back();
    return int(streams.size()) - 1;
  }
  void release(int i) {
    std::lock_guard<std::mutex> lk(m);
    held[i] = 0;
  }
};


std::vector<FrameGroup> frame_groups(std::uint64_t frames, int groups) {
  std::vector<FrameGroup> out;
  if (groups < 1) return out;
  std::uint64_t first = 0;
  for (int g = 0; g < groups; ++g) {
    const std::uint64_t n = frames / groups + (std::uint64_t(g) < frames % groups ? 1 : 0);
    out.push_back({first, n});
    first += n;
  }
  return out;
}

B200Backend::B200Backend(std::vector<int> devices, int slots_per_device, Policy policy)
    : slots_(slots_per_device < 1 ? 2 : slots_per_device), policy_(policy) {
  if (devices.empty()) {
    int n = 0;
    check(avec_device_count(&n));
    for (int i = 0; i < n; ++i) devices.push_back(i);
  }
  if (devices.empty()) throw Error(ErrorCode::internal, "no CUDA device visible");
  try {
    for (int d : devices) {
      avec_ctx* c = nullptr;
      check(avec_ctx_create(d, slots_, &c));
      ctx_.push_back(c);
    }
  } catch (...) {
    for (auto* c : ctx_) avec_ctx_destroy(c);
    throw;
  }
  devices_ = devices;
  inflight_.reset(new std::atomic<int>[ctx_.size()]);
  pipelines_.reset(new std::atomic<int>[ctx_.size()]);
  streaming_.reset(new std::atomic<int>[ctx_.size()]);
  for (size_t i = 0; i < ctx_.size(); ++i) inflight_[i] = pipelines_[i] = streaming_[i] = 0;
  static const int cap = [] {
    const char* e = std::getenv("AVEC_PIPE_BUSY");
    return e ? std::max(1, std::atoi(e)) : 2;
  }();
  for (auto* c : ctx_) {
    pools_.push_back(std::make_unique<PipePool>());
    pools_.back()->ctx = c;
    pools_.back()->cap = cap;
  }
  if (const char* e = std::getenv("AVEC_PIPELINE")) pipelining_ = e[0] != '0';
  label_ = ctx_.size() == 1 ? std::string(avec_ctx_label(ctx_[0]))
                            : "b200x" + std::to_string(ctx_.size()) +
                                  (policy_ == Policy::split     ? ":split"
                                   : policy_ == Policy::session ? ":session"
                                                                : ":affinity");
}

B200Backend::~B200Backend() {
  pools_.clear();  // streams before their contexts
  for (auto* c : ctx_) avec_ctx_destroy(c);
}

ModelHandle B200Backend::register_model(const wire::ModelDescriptor& m) {
  // reference backend.cpp:70-73 validation happens in the engine, per device
  std::lock_guard<std::mutex> lk(m_);
  auto it = id_by_digest_.find(m.digest);
  if (it != id_by_digest_.end()) return {it->second};
  Entry e;
  for (auto* c : ctx_) {
    std::uint64_t h = 0;
    const int rc = avec_model_register(c, m.digest.data(), m.name.data(), m.name.size(),
                                       m.structure.data(), m.structure.size(), m.weights.data(),
                                       m.weights.size(), m.output_divisor, &h);
    if (rc != AVEC_OK) rethrow(rc);
    e.per_device.push_back(h);
  }
  check(avec_model_kind(ctx_[0], e.per_device[0], &e.kind));
  const std::uint64_t id = next_id_++;
  id_by_digest_.emplace(m.digest, id);
  models_.emplace(id, std::move(e));
  return {id};
}

B200Backend::Entry B200Backend::lookup(ModelHandle h) {
  std::lock_guard<std::mutex> lk(m_);
  auto it = models_.find(h.id);
  if (it == models_.end()) throw Error(ErrorCode::unknown_model, "handle was never issued by this backend");
  return it->second;
}

std::uint64_t B200Backend::output_elems(ModelHandle model, const wire::Dims& d) {
  const Entry e = lookup(model);
  std::uint64_t k = 0;
  check(avec_output_elems(ctx_[0], e.per_device[0], d.batch, d.channels, d.height, d.width, &k));
  return k;
}

int B200Backend::concurrency() const {
  return policy_ == Policy::split ? slots_ : int(ctx_.size()) * slots_;
}

int B200Backend::pick_device() {
  int best = 0;
  for (size_t i = 1; i < ctx_.size(); ++i)
    if (inflight_[i].load() < inflight_[best].load()) best = int(i);
  return best;
}

double B200Backend::run_on(int dev, const Entry& e, const wire::Dims& d, const float* in,
                           std::uint64_t n_in, float* out, std::uint64_t n_out) {
  inflight_[dev]++;
  double s = 0;
  const int rc = avec_forward(ctx_[dev], e.per_device[dev], d.batch, d.channels, d.height, d.width, in,
                              n_in, out, n_out, &s);
  inflight_[dev]--;
  if (rc != AVEC_OK) rethrow(rc);
  return s;
}

double B200Backend::forward_into(ModelHandle model, const wire::Dims& d, const float* in,
                                 std::uint64_t n_in, float* out, std::uint64_t n_out) {
  const Entry e = lookup(model);
  const std::uint64_t frames = std::uint64_t(d.batch) * d.channels / 3;
  const int G = int(ctx_.size());
  if (policy_ == Policy::affinity || G == 1 || e.kind != AVEC_MODEL_POSENET || frames < 2 ||
      std::uint64_t(d.batch) * d.channels % 3 != 0)
    return run_on(pick_device(), e, d, in, n_in, out, n_out);
  // split: contiguous frame groups, one per GPU, concurrently
  const std::uint64_t per_frame_in = 3ull * d.height * d.width;
  const std::uint64_t per_frame_out = n_out / frames;
  const auto part = frame_groups(frames, int(std::min<std::uint64_t>(frames, G)));
  const int groups = int(part.size());
  std::vector<double> secs(groups, 0.0);
  std::vector<std::exception_ptr> errs(groups);
  std::vector<std::thread> th;
  for (int g = 0; g < groups; ++g) {
    const std::uint64_t f0 = part[g].first, nf = part[g].count;
    const wire::Dims sub{1, std::uint32_t(3 * nf), d.height, d.width};
    th.emplace_back([&, g, f0, nf, sub] {
      try {
        secs[g] = run_on(g, e, sub, in + f0 * per_frame_in, nf * per_frame_in, out + f0 * per_frame_out,
                         nf * per_frame_out);
      } catch (...) {
        errs[g] = std::current_exception();
      }
    });
  }
  for (auto& t : th) t.join();
  for (auto& ep : errs)
    if (ep) std::rethrow_exception(ep);
  return *std::max_element(secs.begin(), secs.end());
}

double B200Backend::forward_session(std::uint64_t session, ModelHandle model, const wire::Dims& d, const float* in,
                                    std::uint64_t n_in, float* out, std::uint64_t n_out) {
  if (policy_ != Policy::session) return forward_into(model, d, in, n_in, out, n_out);
  const Entry e = lookup(model);
  const int dev = int((session == 0 ? 0 : session - 1) % ctx_.size());
  return run_on(dev, e, d, in, n_in, out, n_out);
}

namespace {

class B200Pipeline final : public Pipeline {
 public:
  B200Pipeline(B200Backend::PipePool* pool, std::function<std::uint64_t(ModelHandle)> handle_of,
               std::atomic<int>* open, std::atomic<int>* active, std::atomic<int>* inflight)
      : pool_(pool), handle_of_(std::move(handle_of)), open_(open), active_(active), inflight_(inflight) {
    ++*open_;
  }
  ~B200Pipeline() override {
    if (held_ >= 0) {
      avec_stream_abort(pool_->streams[held_]);
      release();
    }
    --*open_;
  }
  bool begin(ModelHandle model, const wire::Dims& d, const float* in, float* out, std::uint64_t n_out) override {
    // at most `cap` cycles (dispatched or pipelined) on this GPU
    if (inflight_->load() >= pool_->cap) return false;
    if (active_->fetch_add(1) + inflight_->load() >= pool_->cap) {
      --*active_;
      return false;
    }
    const auto key = key_of(model, d);
    held_ = pool_->acquire(&key);
    if (held_ < 0) {
      --*active_;
      return false;
    }
    const int rc =
        avec_stream_begin(pool_->streams[held_], handle_of_(model), d.batch, d.channels, d.height, d.width, in, out, n_out);
    if (rc != AVEC_OK) {
      release();
      rethrow(rc);
    }
    return true;
  }
  void prepare(ModelHandle model, const wire::Dims& d) override {
    const auto key = key_of(model, d);
    for (int tries = 0; tries < pool_->cap; ++tries) {
      const int i = pool_->acquire(nullptr);
      if (i < 0) return;  // all streams busy: prepared next time
      const bool have = pool_->ready[i].count(key) > 0;
      int rc = AVEC_OK;
      if (!have)
        rc = avec_stream_prepare(pool_->streams[i], handle_of_(model), d.batch, d.channels, d.height, d.width);
      if (rc == AVEC_OK && !have) {
        std::lock_guard<std::mutex> lk(pool_->m);
        pool_->ready[i].insert(key);
      }
      pool_->release(i);
      check(rc);
      if (have) return;
    }
  }
  void feed(std::uint64_t landed) override { check(avec_stream_feed(pool_->streams[held_], landed)); }
  double finish() override {
    double secs = 0;
    const int rc = avec_stream_finish(pool_->streams[held_], &secs);
    release();
    check(rc);
    return secs;
  }
  void abort() override {
    const int rc = held_ >= 0 ? avec_stream_abort(pool_->streams[held_]) : AVEC_OK;
    release();
    check(rc);
  }

 private:
  B200Backend::PipePool::Key key_of(ModelHandle m, const wire::Dims& d) const {
    return {handle_of_(m), d.batch, d.channels, d.height, d.width};
  }
  void release() {
    if (held_ >= 0) {
      pool_->release(held_);
      --*active_;
    }
    held_ = -1;
  }
  B200Backend::PipePool* pool_;
  std::function<std::uint64_t(ModelHandle)> handle_of_;
  std::atomic<int>*open_, *active_, *inflight_;
  int held_ = -1;
};

}  // namespace

std::unique_ptr<Pipeline> B200Backend::open_pipeline(std::uint64_t session) {
  // split cycles span every GPU; a pipeline lives on one
  if (!pipelining_ || (policy_ == Policy::split && ctx_.size() > 1)) return nullptr;
  int dev = 0;
  if (policy_ == Policy::session) {
    dev = int((session == 0 ? 0 : session - 1) % ctx_.size());
  } else {  // affinity: the GPU with the fewest open pipelines
    for (size_t i = 1; i < ctx_.size(); ++i)
      if (pipelines_[i].load() < pipelines_[dev].load()) dev = int(i);
  }
  return std::make_unique<B200Pipeline>(
      pools_[dev].get(), [this, dev](ModelHandle h) { return lookup(h).per_device[dev]; }, &pipelines_[dev],
      &streaming_[dev], &inflight_[dev]);
}

Heatmap B200Backend::forward(ModelHandle model, const Frame& frame) {
  if (frame.data.size() != frame.dims.elem_count())
    throw std::invalid_argument("frame data size disagrees with dims");
  Heatmap h;
  h.data.resize(output_elems(model, frame.dims));
  forward_into(model, frame.dims, frame.data.data(), frame.data.size(), h.data.data(), h.data.size());
  return h;
}

void* B200Backend::alloc_host(std::size_t bytes) {
  void* p = avec_host_alloc(bytes);
  if (!p) throw std::bad_alloc();
  return p;
}

void B200Backend::free_host(void* p) { avec_host_free(p); }

}  // namespace avec::backend

extern "C" int avec_frame_groups(std::uint64_t frames, int groups, std::uint64_t* first, std::uint64_t* count) {
  if (groups < 1 || !first || !count) return AVEC_ERR_INVALID_ARGUMENT;
  const auto part = avec::backend::frame_groups(frames, groups);
  for (int g = 0; g < groups; ++g) {
    first[g] = part[g].first;
    count[g] = part[g].count;
  }
  return AVEC_OK;
}
