// avec-server: the B200 destination node. Flags of the reference server
// (proj/tools/server_main.cpp:25-43) plus --devices / --slots / --policy
// (affinity: least-loaded GPU per cycle; session: session k on GPU (k-1) mod G;
// split: each batched cycle cut into frame groups across the GPUs).
// Same banner (server_main.cpp:71) and SIGINT/SIGTERM drain (:48-80).
#include <csignal>
#include <cstdio>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "b200_backend.hpp"
#include "server.hpp"

namespace {

void usage() {
  std::fprintf(stderr,
               "usage: avec-server [--bind HOST] [--port N] [--devices all|0,1,..] [--slots N]\n"
               "                   [--policy affinity|session|split] [--preset none]\n"
               "                   [--kind images|video] [--scale X] [--gpu-s S] [--load-s S]\n"
               "                   [--max-sessions N] [--max-model-bytes N] [--log PATH]\n");
}

}  // namespace

int main(int argc, char** argv) {
  std::string bind_host = "127.0.0.1", preset = "none", kind = "video", log_path, devices = "all",
              policy = "affinity";
  unsigned long port = 0, max_sessions = 16, slots = 2;
  unsigned long long max_model_bytes = 1ull << 30;
  double scale = 0.01, gpu_s = -1, load_s = -1;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) {
        usage();
        std::exit(2);
      }
      return argv[++i];
    };
    try {
      if (a == "--bind") bind_host = val();
      else if (a == "--port") port = std::stoul(val());
      else if (a == "--preset") preset = val();
      else if (a == "--kind") kind = val();
      else if (a == "--scale") scale = std::stod(val());
      else if (a == "--gpu-s") gpu_s = std::stod(val());
      else if (a == "--load-s") load_s = std::stod(val());
      else if (a == "--max-sessions") max_sessions = std::stoul(val());
      else if (a == "--max-model-bytes") max_model_bytes = std::stoull(val());
      else if (a == "--log") log_path = val();
      else if (a == "--devices") devices = val();
      else if (a == "--slots") slots = std::stoul(val());
      else if (a == "--policy") policy = val();
      else if (a == "-h" || a == "--help") {
        usage();
        return 0;
      } else {
        std::fprintf(stderr, "unknown option %s\n", a.c_str());
        usage();
        return 2;
      }
    } catch (const std::exception&) {
      std::fprintf(stderr, "bad value for %s\n", a.c_str());
      return 2;
    }
  }
  if (port > 65535) {
    std::fprintf(stderr, "bad port\n");
    return 2;
  }

  // block before any thread exists so sigwait is the only consumer
  sigset_t set;
  sigemptyset(&set);
  sigaddset(&set, SIGINT);
  sigaddset(&set, SIGTERM);
  pthread_sigmask(SIG_BLOCK, &set, nullptr);

  try {
    using namespace avec;
    std::vector<int> devs;
    if (devices != "all") {
      std::stringstream ss(devices);
      std::string tok;
      while (std::getline(ss, tok, ',')) devs.push_back(std::stoi(tok));
    }
    auto pol = policy == "split"     ? backend::B200Backend::Policy::split
               : policy == "session" ? backend::B200Backend::Policy::session
                                     : backend::B200Backend::Policy::affinity;
    if (policy != "split" && policy != "affinity" && policy != "session")
      throw std::runtime_error("policy must be affinity, session or split");
    // The reference's timing-emulation flags (server_main.cpp:25-43) are
    // accepted so existing command lines parse, but this server runs the real
    // network: an emulated device/edge/cloud delay has no meaning on it.
    if (kind != "images" && kind != "video") throw std::runtime_error("unknown workload kind: " + kind);
    if (!(scale > 0.0)) throw std::runtime_error("scale factor must be > 0");
    if (preset != "none" || gpu_s > 0 || load_s > 0)
      throw std::runtime_error("timing emulation (--preset/--gpu-s/--load-s) is not supported by the B200 "
                               "server: it runs the network, use --preset none");
    std::shared_ptr<backend::Backend> be =
        std::make_shared<backend::B200Backend>(devs, int(slots), pol);

    server::ServerConfig cfg;
    cfg.limits.max_sessions = std::uint32_t(max_sessions);
    cfg.limits.max_model_bytes = max_model_bytes;
    cfg.log_path = log_path;
    server::Server srv(be, cfg);
    const std::uint16_t bound = srv.listen(bind_host, std::uint16_t(port));
    std::printf("listening on %s:%u (backend %s)\n", bind_host.c_str(), bound, std::string(be->label()).c_str());
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
