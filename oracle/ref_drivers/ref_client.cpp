// The UNMODIFIED reference client (accelfwd::client::Session) driven from the
// command line. Used by the tests as the "existing client shim": it connects to
// a server (ours, or the reference's), negotiates a model, forwards seeded
// harness frames and reports what came back. With --check-mockpose every
// result is memcmp'd against the reference's own local mockpose_forward
// (harness.cpp:657-663 style).
#include <algorithm>
#include <cinttypes>

#include "accelfwd/client.hpp"
#include "accelfwd/clock.hpp"
#include "accelfwd/error.hpp"
#include "ref_common.hpp"

using namespace accelfwd;

int main(int argc, char** argv) {
  try {
    auto a = refdrv::parse_args(argc, argv);
    std::string endpoint = refdrv::get(a, "endpoint", "127.0.0.1:7000");
    std::uint32_t w = std::stoul(refdrv::get(a, "width", "64"));
    std::uint32_t h = std::stoul(refdrv::get(a, "height", "64"));
    std::uint32_t batch = std::stoul(refdrv::get(a, "batch", "1"));
    std::uint32_t frames = std::stoul(refdrv::get(a, "frames", "4"));
    std::uint32_t warmup = std::stoul(refdrv::get(a, "warmup", "0"));
    std::uint64_t seed = std::stoull(refdrv::get(a, "seed", "7"));
    double divisor = std::stod(refdrv::get(a, "divisor", "3.368421"));
    bool check = a.count("check-mockpose") > 0;
    std::string dump = refdrv::get(a, "dump", "");
    double cycle_timeout = std::stod(refdrv::get(a, "cycle-timeout", "120"));

    wire::ModelDescriptor model;
    if (a.count("structure")) {
      auto s = refdrv::read_file(a["structure"]);
      std::vector<std::uint8_t> wts;
      if (a.count("weights")) wts = refdrv::read_file(a["weights"]);
      model = wire::make_model(refdrv::get(a, "name", "openpose"), std::move(s),
                               std::move(wts), divisor);
    } else {
      harness::ModelSpec ms;
      ms.output_divisor = divisor;
      ms.seed = std::stoull(refdrv::get(a, "model-seed", "1"));
      ms.structure_bytes = std::stoul(refdrv::get(a, "structure-bytes", "4096"));
      ms.weights_bytes = std::stoul(refdrv::get(a, "weights-bytes", "1048576"));
      ms.name = refdrv::get(a, "name", "pose-est");
      model = harness::synth_model(ms);
    }

    client::SessionConfig cfg;
    cfg.cycle_timeout_s = cycle_timeout;
    auto session = client::Session::connect(endpoint, cfg);
    Stopwatch setup;
    auto ens = session.ensure_model(model);
    double setup_s = setup.elapsed_s();

    std::FILE* dump_f = dump.empty() ? nullptr : std::fopen(dump.c_str(), "wb");
    wire::Sha256 all;
    std::uint64_t mismatches = 0, bytes_bad = 0;
    double gpu = 0, comm = 0, timed = 0;
    std::vector<double> lat;  // per-cycle wall seconds of the timed cycles
    wire::Dims dims{1, 3 * batch, h, w};
    const std::uint64_t expect_bytes =
        wire::transfer_size(dims, divisor) + wire::kCycleOverheadBytes;
    for (std::uint32_t i = 0; i < warmup + frames; ++i) {
      auto f = refdrv::batched_frame(w, h, batch, seed, i * batch);
      Stopwatch sw;
      auto [heat, t] = session.forward(f);
      double el = sw.elapsed_s();
      if (t.bytes_sent + t.bytes_received != expect_bytes) ++bytes_bad;
      if (i < warmup) continue;
      timed += el;
      lat.push_back(el);
      gpu += t.gpu_s;
      comm += t.communication_s;
      all.update({reinterpret_cast<const std::uint8_t*>(heat.data.data()),
                  heat.data.size() * 4});
      if (dump_f) std::fwrite(heat.data.data(), 4, heat.data.size(), dump_f);
      if (check) {
        auto expect = backend::mockpose_forward(f, divisor);
        if (expect.data.size() != heat.data.size() ||
            std::memcmp(expect.data.data(), heat.data.data(), heat.data.size() * 4))
          ++mismatches;
      }
    }
    if (dump_f) std::fclose(dump_f);
    session.close();
    std::sort(lat.begin(), lat.end());
    auto pct = [&](double q) { return lat.empty() ? 0.0 : 1e3 * lat[std::size_t(q * double(lat.size() - 1) + 0.5)]; };
    std::printf(
        "{\"ok\": true, \"cache_hit\": %s, \"setup_s\": %.6f, \"cycles\": %u, "
        "\"frames\": %u, \"timed_s\": %.6f, \"fps\": %.3f, \"gpu_s_mean\": %.6f, "
        "\"comm_s_mean\": %.6f, \"lat_ms_p50\": %.4f, \"lat_ms_p90\": %.4f, \"lat_ms_max\": %.4f, "
        "\"mismatches\": %" PRIu64 ", \"byte_account_bad\": %" PRIu64
        ", \"expect_cycle_bytes\": %" PRIu64 ", \"digest\": \"%s\", \"model_digest\": \"%s\"}\n",
        ens.cache_hit ? "true" : "false", setup_s, frames, frames * batch, timed,
        timed > 0 ? frames * batch / timed : 0.0, frames ? gpu / frames : 0.0,
        frames ? comm / frames : 0.0, pct(0.5), pct(0.9), pct(1.0), mismatches, bytes_bad, expect_bytes,
        wire::hex(all.finish()).c_str(), wire::hex(model.digest).c_str());
    return mismatches == 0 && bytes_bad == 0 ? 0 : 3;
  } catch (const std::exception& e) {
    std::printf("{\"ok\": false, \"error\": \"%s\"}\n", e.what());
    return 1;
  }
}
