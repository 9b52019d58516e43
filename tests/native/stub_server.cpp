// TEST-ONLY: the product server (avec::server::Server) over a CPU stub backend,
// so protocol/state-machine tests run on machines without a GPU. The stub
// computes the reference's segment means (proj/src/backend.cpp:39-67) with a
// plain loop; it is a test double, never linked into avec-server.
// --concurrency N makes it report N parallel workers (like GPUs x slots) and
// --jitter-ms M sleeps a pseudo-random 0..M ms per forward so completions
// interleave out of arrival order; --print-forward-log dumps
// Server::forward_log() on shutdown for the FIFO check (harness.cpp:676-681).
#include <atomic>
#include <memory>
#include <stdexcept>
#include <chrono>
#include <cmath>
#include <csignal>
#include <thread>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>

#include "backend.hpp"
#include "server.hpp"

namespace {

std::atomic<int> g_begins{0}, g_feeds{0}, g_finishes{0}, g_aborts{0};

// segment means (proj/src/backend.cpp:39-67), shared by forward and the pipeline
void segmeans(const float* x, std::uint64_t e, double c, float* out, std::uint64_t k) {
  const double width = double(e) / double(k);
  std::uint64_t lo = 0;
  for (std::uint64_t j = 0; j < k; ++j) {
    const std::uint64_t hi = (j + 1 == k) ? e : std::uint64_t(double(j + 1) * width);
    double s = 0;
    for (std::uint64_t i = lo; i < hi; ++i) s += double(x[i]);
    out[j] = float(s / double(hi - lo));
    lo = hi;
  }
  (void)c;
}

class StubBackend;

// --pipeline: a CPU stand-in for the GPU pipeline, exercising the server's
// cycle speculation (begin at the FrameData header with the previous cycle's
// model and dims, feed while bytes land, finish by the dispatcher, abort when
// Resolution disagrees). finish() computes with the GUESSED model, so a
// guess the server failed to drop shows up as a wrong result.
class StubPipeline final : public avec::backend::Pipeline {
 public:
  explicit StubPipeline(StubBackend* be) : be_(be) {}
  bool begin(avec::backend::ModelHandle m, const avec::wire::Dims& d, const float* in, float* out,
             std::uint64_t n_out) override;
  void feed(std::uint64_t landed) override {
    if (landed < landed_) throw std::runtime_error("feed went backwards");
    landed_ = landed;
    ++g_feeds;
  }
  double finish() override;
  void abort() override { ++g_aborts; }

 private:
  StubBackend* be_;
  avec::backend::ModelHandle model_;
  avec::wire::Dims dims_;
  const float* in_ = nullptr;
  float* out_ = nullptr;
  std::uint64_t n_out_ = 0, landed_ = 0;
};

class StubBackend final : public avec::backend::Backend {
 public:
  StubBackend(int concurrency, int jitter_ms, bool pipeline)
      : concurrency_(concurrency), jitter_ms_(jitter_ms), pipeline_(pipeline) {}
  int concurrency() const override { return concurrency_; }
  bool zero_copy() const override { return pipeline_; }
  std::uint64_t output_elems(avec::backend::ModelHandle h, const avec::wire::Dims& d) override {
    return std::uint64_t(std::llround(double(d.elem_count()) / divisor(h)));
  }
  double forward_into(avec::backend::ModelHandle h, const avec::wire::Dims& d, const float* in, std::uint64_t n,
                      float* out, std::uint64_t k) override {
    (void)d;
    segmeans(in, n, divisor(h), out, k);
    return 0.0;
  }
  std::unique_ptr<avec::backend::Pipeline> open_pipeline(std::uint64_t) override {
    if (!pipeline_) return nullptr;
    return std::make_unique<StubPipeline>(this);
  }
  double divisor(avec::backend::ModelHandle h) {
    std::lock_guard<std::mutex> lk(m_);
    auto it = div_.find(h.id);
    if (it == div_.end()) throw avec::backend::Error(avec::backend::ErrorCode::unknown_model, "unknown model");
    return it->second;
  }
  avec::backend::ModelHandle register_model(const avec::wire::ModelDescriptor& m) override {
    using avec::backend::Error;
    using avec::backend::ErrorCode;
    if (!(m.output_divisor > 0.0) || !std::isfinite(m.output_divisor))
      throw Error(ErrorCode::invalid_model, "output divisor must be positive and finite");
    if (m.structure.empty()) throw Error(ErrorCode::invalid_model, "model structure is empty");
    std::lock_guard<std::mutex> lk(m_);
    auto it = ids_.find(m.digest);
    if (it != ids_.end()) return {it->second};
    const std::uint64_t id = next_++;
    ids_[m.digest] = id;
    div_[id] = m.output_divisor;
    return {id};
  }
  avec::backend::Heatmap forward(avec::backend::ModelHandle h, const avec::backend::Frame& f) override {
    using avec::backend::Error;
    using avec::backend::ErrorCode;
    double c;
    {
      std::lock_guard<std::mutex> lk(m_);
      auto it = div_.find(h.id);
      if (it == div_.end()) throw Error(ErrorCode::unknown_model, "handle was never issued by this backend");
      c = it->second;
    }
    if (jitter_ms_ > 0) {
      const std::uint64_t r = (calls_.fetch_add(1) * 0x9E3779B97F4A7C15ull) >> 40;
      std::this_thread::sleep_for(std::chrono::microseconds(r % (1000 * std::uint64_t(jitter_ms_))));
    }
    const std::uint64_t e = f.data.size();
    const std::uint64_t k = std::uint64_t(std::llround(double(e) / c));
    if (k < 1 || k > e) throw Error(ErrorCode::degenerate_output, "degenerate output size");
    const double width = double(e) / double(k);
    avec::backend::Heatmap out;
    out.data.resize(k);
    std::uint64_t lo = 0;
    for (std::uint64_t j = 0; j < k; ++j) {
      const std::uint64_t hi = (j + 1 == k) ? e : std::uint64_t(double(j + 1) * width);
      double s = 0;
      for (std::uint64_t i = lo; i < hi; ++i) s += double(f.data[i]);
      out.data[j] = float(s / double(hi - lo));
      lo = hi;
    }
    return out;
  }
  std::string_view label() const override { return "stub"; }

 private:
  int concurrency_ = 1, jitter_ms_ = 0;
  bool pipeline_ = false;
  std::atomic<std::uint64_t> calls_{0};
  std::mutex m_;
  std::map<avec::wire::Digest, std::uint64_t> ids_;
  std::map<std::uint64_t, double> div_;
  std::uint64_t next_ = 1;
};

bool StubPipeline::begin(avec::backend::ModelHandle m, const avec::wire::Dims& d, const float* in, float* out,
                         std::uint64_t n_out) {
  model_ = m, dims_ = d, in_ = in, out_ = out, n_out_ = n_out, landed_ = 0;
  ++g_begins;
  return true;
}

double StubPipeline::finish() {
  if (landed_ != dims_.elem_count() * 4) throw std::runtime_error("finish before the frame landed");
  segmeans(in_, dims_.elem_count(), be_->divisor(model_), out_, n_out_);
  ++g_finishes;
  return 0.0;
}

}  // namespace

int main(int argc, char** argv) {
  std::string log;
  unsigned max_sessions = 16;
  unsigned long long max_model = 1ull << 30;
  int concurrency = 1, jitter_ms = 0;
  unsigned long long log_cap = 1ull << 20;
  bool print_log = false, pipeline = false;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "--print-forward-log") {
      print_log = true;
      continue;
    }
    if (a == "--pipeline") {
      pipeline = true;
      continue;
    }
    if (i + 1 >= argc) break;
    if (a == "--concurrency") concurrency = std::stoi(argv[i + 1]);
    else if (a == "--jitter-ms") jitter_ms = std::stoi(argv[i + 1]);
    else if (a == "--forward-log-cap") log_cap = std::stoull(argv[i + 1]);
    else if (a == "--log") log = argv[i + 1];
    else if (a == "--max-sessions") max_sessions = std::stoul(argv[i + 1]);
    else if (a == "--max-model-bytes") max_model = std::stoull(argv[i + 1]);
    ++i;
  }
  sigset_t set;
  sigemptyset(&set);
  sigaddset(&set, SIGINT);
  sigaddset(&set, SIGTERM);
  pthread_sigmask(SIG_BLOCK, &set, nullptr);
  avec::server::ServerConfig cfg;
  cfg.log_path = log;
  cfg.limits.max_sessions = max_sessions;
  cfg.limits.max_model_bytes = max_model;
  cfg.forward_log_cap = log_cap;
  auto be = std::make_shared<StubBackend>(concurrency, jitter_ms, pipeline);
  avec::server::Server srv(be, cfg);
  const auto port = srv.listen("127.0.0.1", 0);
  std::printf("listening on 127.0.0.1:%u (backend %s)\n", port, std::string(be->label()).c_str());
  std::fflush(stdout);
  int sig = 0;
  sigwait(&set, &sig);
  std::printf("shutting down (signal %d)\n", sig);
  const std::size_t live_threads = srv.session_threads();  // before the drain joins them
  srv.shutdown();
  if (print_log) {
    std::printf("forward_log [");
    const auto log_entries = srv.forward_log();
    for (std::size_t i = 0; i < log_entries.size(); ++i)
      std::printf("%s[%llu, %llu]", i ? ", " : "", (unsigned long long)log_entries[i].arrival_seq,
                  (unsigned long long)log_entries[i].session_id);
    std::printf("]\nsession_threads %zu\n", live_threads);
    std::printf("pipeline begins %d feeds %d finishes %d aborts %d\n", g_begins.load(), g_feeds.load(),
                g_finishes.load(), g_aborts.load());
  }
  std::fflush(stdout);
  return 0;
}
