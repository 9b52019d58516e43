// The reference destination server (accelfwd::server::Server + MockPoseBackend)
// with the flags of tools/server_main.cpp:25-43 that matter here, parsed without
// CLI11 (absent from the mount). Same banner (server_main.cpp:71) and SIGTERM
// drain (server_main.cpp:48-80). Test infrastructure / CPU baseline only.
#include <csignal>

#include "accelfwd/server.hpp"
#include "ref_common.hpp"

using namespace accelfwd;

int main(int argc, char** argv) {
  auto a = refdrv::parse_args(argc, argv);
  std::string bind = refdrv::get(a, "bind", "127.0.0.1");
  std::uint16_t port = std::uint16_t(std::stoul(refdrv::get(a, "port", "0")));
  sigset_t set;
  sigemptyset(&set);
  sigaddset(&set, SIGINT);
  sigaddset(&set, SIGTERM);
  pthread_sigmask(SIG_BLOCK, &set, nullptr);
  try {
    server::ServerConfig cfg;
    cfg.limits.max_sessions = std::stoul(refdrv::get(a, "max-sessions", "16"));
    cfg.limits.max_model_bytes =
        std::stoull(refdrv::get(a, "max-model-bytes", std::to_string(1ull << 30)));
    cfg.log_path = refdrv::get(a, "log", "");
    std::shared_ptr<backend::Backend> be = std::make_shared<backend::MockPoseBackend>();
    server::Server srv(be, cfg);
    std::uint16_t bound = srv.listen(bind, port);
    std::printf("listening on %s:%u (backend %s)\n", bind.c_str(), bound,
                std::string(be->label()).c_str());
    std::fflush(stdout);
    int sig = 0;
    sigwait(&set, &sig);
    std::printf("shutting down (signal %d)\n", sig);
    std::fflush(stdout);
    srv.shutdown();
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
