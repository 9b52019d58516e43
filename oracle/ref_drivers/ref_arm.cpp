// Reference arm of bench.py: the reference's own server-side path, unmodified
// (Server + MockPoseBackend, server.cpp:84-338, backend.cpp:39-96) driven by
// the reference's own client Session over TCP loopback (client.cpp:144-197).
// Each step is one forward cycle of `batch` frames folded into channels.
// --clients N runs N concurrent sessions (C4 shape); the reference backend
// serves them FIFO on one dispatch thread by design (server.cpp:84-111).
// --endpoint HOST:PORT points the same reference clients, model and frames at
// another server instead (bench.py: the B200 avec-server, like for like).
#include <atomic>
#include <memory>
#include <thread>

#include "accelfwd/client.hpp"
#include "accelfwd/clock.hpp"
#include "accelfwd/server.hpp"
#include "ref_common.hpp"

using namespace accelfwd;

int main(int argc, char** argv) {
  try {
    auto a = refdrv::parse_args(argc, argv);
    std::uint32_t w = std::stoul(refdrv::get(a, "width", "656"));
    std::uint32_t h = std::stoul(refdrv::get(a, "height", "368"));
    std::uint32_t batch = std::stoul(refdrv::get(a, "batch", "8"));
    std::uint32_t steps = std::stoul(refdrv::get(a, "steps", "5"));
    std::uint32_t warmup = std::stoul(refdrv::get(a, "warmup", "3"));
    std::uint32_t clients = std::stoul(refdrv::get(a, "clients", "1"));
    double divisor = std::stod(refdrv::get(a, "divisor", std::to_string(192.0 / 57.0)));

    std::string ep = refdrv::get(a, "endpoint", "");
    std::unique_ptr<server::Server> srv;
    if (ep.empty()) {
      srv = std::make_unique<server::Server>(std::make_shared<backend::MockPoseBackend>());
      std::uint16_t port = srv->listen("127.0.0.1", 0);
      ep = "127.0.0.1:" + std::to_string(port);
    }

    harness::ModelSpec ms;
    ms.output_divisor = divisor;
    auto model = harness::synth_model(ms);

    // frames generated before timing: the client-side generator is not the path
    auto frame = refdrv::batched_frame(w, h, batch, 7, 0);

    std::vector<double> per_client_s(clients, 0), compute_s(clients, 0);
    std::atomic<int> ready{0};
    std::atomic<bool> go{false};
    std::vector<std::thread> th;
    std::vector<std::string> errs(clients);
    for (std::uint32_t c = 0; c < clients; ++c) {
      th.emplace_back([&, c] {
        try {
          auto s = client::Session::connect(ep);
          s.ensure_model(model);
          for (std::uint32_t i = 0; i < warmup; ++i) s.forward(frame);
          ready++;
          while (!go) std::this_thread::yield();
          Stopwatch sw;
          for (std::uint32_t i = 0; i < steps; ++i) {
            auto r = s.forward(frame);
            compute_s[c] += r.second.gpu_s;
          }
          per_client_s[c] = sw.elapsed_s();
          s.close();
        } catch (const std::exception& e) {
          errs[c] = e.what();
          ready++;
        }
      });
    }
    while (ready < int(clients)) std::this_thread::yield();
    Stopwatch wall;
    go = true;
    for (auto& t : th) t.join();
    double wall_s = wall.elapsed_s();
    if (srv) srv->shutdown();
    for (auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
    double frames = double(steps) * batch * clients;
    double cs = 0;
    for (double v : compute_s) cs += v;
    std::printf("{\"ok\": true, \"frames\": %.0f, \"wall_s\": %.6f, \"fps\": %.4f, "
                "\"ms_per_cycle\": %.4f, \"backend_ms_per_cycle\": %.4f, \"clients\": %u, "
                "\"batch\": %u, \"width\": %u, \"height\": %u, \"backend\": \"mockpose\", \"server\": \"%s\"}\n",
                frames, wall_s, frames / wall_s, 1e3 * wall_s / steps,
                1e3 * cs / (double(steps) * clients), clients, batch, w, h,
                srv ? "reference accelfwd::server::Server" : ep.c_str());
    return 0;
  } catch (const std::exception& e) {
    std::printf("{\"ok\": false, \"error\": \"%s\"}\n", e.what());
    return 1;
  }
}
