// TEST-ONLY: the product server (avec::server::Server) over a CPU stub backend,
// so protocol/state-machine tests run on machines without a GPU. The stub
// computes the reference's segment means (proj/src/backend.cpp:39-67) with a
// plain loop; it is a test double (like the reference tests' MockPose /
// wrap_delay), never linked into avec-server.
#include <cmath>
#include <csignal>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>

#include "backend.hpp"
#include "server.hpp"

namespace {

class StubBackend final : public avec::backend::Backend {
 public:
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
    auto pass = gate_.enter();
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
  std::mutex m_;
  avec::backend::FifoGate gate_;
  std::map<avec::wire::Digest, std::uint64_t> ids_;
  std::map<std::uint64_t, double> div_;
  std::uint64_t next_ = 1;
};

}  // namespace

int main(int argc, char** argv) {
  std::string log;
  unsigned max_sessions = 16;
  unsigned long long max_model = 1ull << 30;
  for (int i = 1; i + 1 < argc; i += 2) {
    std::string a = argv[i];
    if (a == "--log") log = argv[i + 1];
    else if (a == "--max-sessions") max_sessions = std::stoul(argv[i + 1]);
    else if (a == "--max-model-bytes") max_model = std::stoull(argv[i + 1]);
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
  auto be = std::make_shared<StubBackend>();
  avec::server::Server srv(be, cfg);
  const auto port = srv.listen("127.0.0.1", 0);
  std::printf("listening on 127.0.0.1:%u (backend %s)\n", port, std::string(be->label()).c_str());
  std::fflush(stdout);
  int sig = 0;
  sigwait(&set, &sig);
  srv.shutdown();
  return 0;
}
