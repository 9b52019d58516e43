// The reference's OWN destination server (accelfwd::server::Server, proj/src/
// server.cpp) with the B200 engine plugged in through the C-ABI shim
// (b200_shim.hpp) instead of MockPoseBackend — the plugin-level drop-in.
// Same banner and signal handling as the reference CLI (server_main.cpp).
#include <csignal>

#include "accelfwd/server.hpp"
#include "b200_shim.hpp"
#include "ref_common.hpp"

using namespace accelfwd;

int main(int argc, char** argv) {
  auto a = refdrv::parse_args(argc, argv);
  sigset_t set;
  sigemptyset(&set);
  sigaddset(&set, SIGINT);
  sigaddset(&set, SIGTERM);
  pthread_sigmask(SIG_BLOCK, &set, nullptr);
  try {
    std::shared_ptr<backend::Backend> be =
        std::make_shared<backend::B200Backend>(std::stoi(refdrv::get(a, "device", "0")));
    server::Server srv(be);
    const auto port = srv.listen("127.0.0.1", std::uint16_t(std::stoul(refdrv::get(a, "port", "0"))));
    std::printf("listening on 127.0.0.1:%u (backend %s)\n", port, std::string(be->label()).c_str());
    std::fflush(stdout);
    int sig = 0;
    sigwait(&set, &sig);
    srv.shutdown();
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
