#include "backend.hpp"

#include <chrono>
#include <cstdlib>
#include <thread>

namespace avec::backend {

FifoGate::Pass FifoGate::enter() {
  std::unique_lock<std::mutex> lk(m_);
  const std::uint64_t ticket = next_++;
  cv_.wait(lk, [&] { return serving_ == ticket; });
  return Pass(this);
}

void FifoGate::leave() {
  {
    std::lock_guard<std::mutex> lk(m_);
    ++serving_;
  }
  cv_.notify_all();
}

void* Backend::alloc_host(std::size_t bytes) {
  void* p = std::aligned_alloc(4096, (bytes + 4095) / 4096 * 4096);
  if (!p) throw std::bad_alloc();
  return p;
}

void Backend::free_host(void* p) { std::free(p); }

BackendProfile preset_profile(std::string_view name, std::string_view kind, double scale) {
  struct Row {
    std::string_view name;
    double images, video, load;
  };
  // per-frame seconds {images, video} and model load seconds (reference presets)
  static constexpr Row rows[] = {{"device", 2.0, 2.5, 6.43},
                                 {"edge", 0.91, 1.43, 5.937},
                                 {"cloud", 0.095, 0.111, 1.757},
                                 {"none", 0.0, 0.0, 0.0}};
  if (kind != "images" && kind != "video")
    throw Error(ErrorCode::bad_config, "unknown workload kind: " + std::string(kind));
  if (!(scale > 0.0)) throw Error(ErrorCode::bad_config, "scale factor must be > 0");
  for (const Row& r : rows)
    if (r.name == name) {
      BackendProfile p;
      p.per_frame_compute_s = (kind == "images" ? r.images : r.video) * scale;
      p.model_load_s = r.load * scale;
      p.label = std::string(name);
      return p;
    }
  throw Error(ErrorCode::bad_config, "unknown backend preset: " + std::string(name));
}

namespace {

class DelayBackend final : public Backend {
 public:
  DelayBackend(std::shared_ptr<Backend> inner, BackendProfile profile)
      : inner_(std::move(inner)), profile_(std::move(profile)) {}

  ModelHandle register_model(const wire::ModelDescriptor& m) override {
    auto pass = gate_.enter();
    if (profile_.model_load_s > 0 && !loaded_.count(m.digest)) sleep_for(profile_.model_load_s);
    loaded_.insert(m.digest);
    return inner_->register_model(m);
  }

  Heatmap forward(ModelHandle h, const Frame& f) override {
    auto pass = gate_.enter();
    const auto deadline = deadline_from_now();
    Heatmap out = inner_->forward(h, f);
    std::this_thread::sleep_until(deadline);
    return out;
  }

  std::string_view label() const override { return profile_.label; }
  bool zero_copy() const override { return inner_->zero_copy(); }
  std::uint64_t output_elems(ModelHandle h, const wire::Dims& d) override {
    return inner_->output_elems(h, d);
  }
  double forward_into(ModelHandle h, const wire::Dims& d, const float* in, std::uint64_t n, float* out,
                      std::uint64_t k) override {
    auto pass = gate_.enter();
    const auto t0 = std::chrono::steady_clock::now();
    const auto deadline = deadline_from_now();
    inner_->forward_into(h, d, in, n, out, k);
    std::this_thread::sleep_until(deadline);
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  void* alloc_host(std::size_t b) override { return inner_->alloc_host(b); }
  void free_host(void* p) override { inner_->free_host(p); }

 private:
  std::chrono::steady_clock::time_point deadline_from_now() const {
    return std::chrono::steady_clock::now() +
           std::chrono::duration_cast<std::chrono::steady_clock::duration>(
               std::chrono::duration<double>(profile_.per_frame_compute_s));
  }
  static void sleep_for(double s) { std::this_thread::sleep_for(std::chrono::duration<double>(s)); }

  std::shared_ptr<Backend> inner_;
  BackendProfile profile_;
  FifoGate gate_;
  std::set<wire::Digest> loaded_;  // guarded by gate_
};

}  // namespace

std::shared_ptr<Backend> wrap_delay(std::shared_ptr<Backend> inner, BackendProfile profile) {
  return std::make_shared<DelayBackend>(std::move(inner), std::move(profile));
}

}  // namespace avec::backend
