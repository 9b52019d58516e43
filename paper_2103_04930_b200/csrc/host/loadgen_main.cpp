// avec-loadgen: N concurrent sessions driving an AVEC destination over TCP and
// reporting through-the-wire frames/s (BASELINE configs C2/C4). Frames follow
// the reference harness generator (proj/src/harness.cpp:29-42: seed_seq{lo32,
// hi32, index} -> mt19937_64, top 24 bits / 2^24), batch folded into channels.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "client.hpp"
#include "record.hpp"

namespace {

std::vector<float> gen_batch(std::uint64_t seed, std::uint32_t first, std::uint32_t batch, std::uint32_t w,
                             std::uint32_t h) {
  std::vector<float> out;
  out.reserve(std::size_t(batch) * 3 * w * h);
  for (std::uint32_t b = 0; b < batch; ++b) {
    std::seed_seq seq{std::uint32_t(seed), std::uint32_t(seed >> 32), first + b};
    std::mt19937_64 rng(seq);
    for (std::size_t i = 0; i < std::size_t(3) * w * h; ++i)
      out.push_back(float(double(rng() >> 40) * (1.0 / 16777216.0)));
  }
  return out;
}

}  // namespace

int main(int argc, char** argv) {
  std::string endpoint = "127.0.0.1:7000", model = "posenet";
  std::string input_dtype = "bf16";  // pose nets: "tf32" = the tf32 first layer (netspec "input tf32")
  unsigned clients = 1, steps = 20, warmup = 3, batch = 8, width = 656, height = 368;
  unsigned long elems_override = 0;  // raw FrameData size (memcpy sweep), Resolution = width x (E/width)
  // client 0's timed cycles as a reference-format run record (record.hpp)
  std::string record_csv, record_md, label = "b200", host = "loadgen";
  for (int i = 1; i + 1 < argc; i += 2) {
    std::string a = argv[i], v = argv[i + 1];
    if (a == "--endpoint") endpoint = v;
    else if (a == "--clients") clients = std::stoul(v);
    else if (a == "--steps") steps = std::stoul(v);
    else if (a == "--warmup") warmup = std::stoul(v);
    else if (a == "--batch") batch = std::stoul(v);
    else if (a == "--width") width = std::stoul(v);
    else if (a == "--height") height = std::stoul(v);
    else if (a == "--model") model = v;
    else if (a == "--input") input_dtype = v;
    else if (a == "--elems") elems_override = std::stoul(v);
    else if (a == "--record-csv") record_csv = v;
    else if (a == "--record-md") record_md = v;
    else if (a == "--label") label = v;
    else if (a == "--host") host = v;
    else {
      std::fprintf(stderr, "unknown option %s\n", a.c_str());
      return 2;
    }
  }
  using namespace avec;
  wire::ModelDescriptor md;
  if (input_dtype != "bf16" && input_dtype != "tf32") {
    std::fprintf(stderr, "--input must be bf16 or tf32\n");
    return 2;
  }
  const std::string input_line = input_dtype == "tf32" ? "input tf32\n" : "";
  if (model == "posenet") {
    std::string s = "avecnet 1\nfamily openpose_coco\n" + input_line + "init he_uniform 1\n";
    md = wire::make_model("openpose_coco", {s.begin(), s.end()}, {}, 192.0 / 57.0);
  } else if (model == "posenet-body25") {
    std::string s = "avecnet 1\nfamily openpose_body25\n" + input_line + "init he_uniform 1\n";
    md = wire::make_model("openpose_body25", {s.begin(), s.end()}, {}, 192.0 / 78.0);
  } else {
    // the reference's model: opaque structure -> segment means; "mockpose-c1"
    // (divisor 1) returns as many floats as it receives (memcpy sweep, C3)
    std::vector<std::uint8_t> s(4096, 7);
    md = wire::make_model("mockpose", s, {}, model == "mockpose-c1" ? 1.0 : 192.0 / 57.0);
  }
  std::vector<std::vector<float>> frames;
  if (elems_override) {
    height = std::uint32_t(elems_override / width);
    if (std::uint64_t(width) * height != elems_override) {
      std::printf("{\"ok\": false, \"error\": \"--elems must be a multiple of --width\"}\n");
      return 2;
    }
    batch = 1;
    for (unsigned c = 0; c < clients; ++c) {
      std::vector<float> f(elems_override);
      for (std::size_t i = 0; i < f.size(); ++i) f[i] = float(i % 1021) * 0.5f;
      frames.push_back(std::move(f));
    }
  } else {
    for (unsigned c = 0; c < clients; ++c) frames.push_back(gen_batch(7, c * batch, batch, width, height));
  }
  const std::uint32_t elems = std::uint32_t(frames[0].size());

  record::RunMeta meta;
  meta.label = label;
  meta.mode = "offload";
  meta.host = host;
  meta.destination = endpoint;
  meta.workload = "video:" + std::to_string(steps) + ":" + std::to_string(width) + "x" + std::to_string(height) +
                  ":batch" + std::to_string(batch);
  meta.model = md.name;
  meta.output_divisor = md.output_divisor;
  record::RunRecord rec(meta);
  double rec_setup_s = 0, rec_loop_s = 0;

  std::atomic<int> ready{0};
  std::atomic<bool> go{false};
  std::vector<double> busy(clients, 0.0), compute(clients, 0.0);
  // per-cycle wall / communication / gpu seconds of every client (tail diagnostics)
  std::vector<std::vector<double>> cyc(clients), comm(clients), gpu(clients);
  std::vector<std::string> errs(clients);
  std::vector<std::thread> th;
  for (unsigned c = 0; c < clients; ++c) {
    th.emplace_back([&, c] {
      try {
        const auto ts = std::chrono::steady_clock::now();
        auto s = client::Session::connect(endpoint, 10.0);
        s.ensure_model(md);
        if (c == 0) rec_setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - ts).count();
        std::vector<float> out;
        for (unsigned i = 0; i < warmup; ++i) s.forward(frames[c].data(), elems, width, height, out);
        ready++;
        while (!go) std::this_thread::yield();
        const auto t0 = std::chrono::steady_clock::now();
        for (unsigned i = 0; i < steps; ++i) {
          const record::CycleTiming t = s.forward_timed(frames[c].data(), elems, width, height, out);
          compute[c] += t.compute_s;
          cyc[c].push_back(t.communication_s + t.gpu_s + t.other_s);
          comm[c].push_back(t.communication_s);
          gpu[c].push_back(t.gpu_s);
          if (c == 0) rec.record(t);
        }
        busy[c] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (c == 0) rec_loop_s = busy[c];
        s.close();
      } catch (const std::exception& e) {
        errs[c] = e.what();
        ready++;
      }
    });
  }
  while (ready < int(clients)) std::this_thread::yield();
  const auto t0 = std::chrono::steady_clock::now();
  go = true;
  for (auto& t : th) t.join();
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (auto& e : errs)
    if (!e.empty()) {
      std::printf("{\"ok\": false, \"error\": \"%s\"}\n", e.c_str());
      return 1;
    }
  if (!record_csv.empty() || !record_md.empty()) {
    // warm-up cycles are in neither the rows nor the wall time, so
    // gpu + communication + other + setup == total_wall (profiler.cpp decomposition)
    rec.finalize(rec_setup_s, rec_setup_s + rec_loop_s);
    if (!record_csv.empty()) {
      std::ofstream f(record_csv);
      record::write_cycle_csv(rec, f);
    }
    if (!record_md.empty()) {
      std::ofstream f(record_md);
      record::write_summary_markdown(rec, f);
    }
  }
  double cs = 0;
  for (double v : compute) cs += v;
  std::vector<double> all, allc, allg;
  for (unsigned c = 0; c < clients; ++c) {
    all.insert(all.end(), cyc[c].begin(), cyc[c].end());
    allc.insert(allc.end(), comm[c].begin(), comm[c].end());
    allg.insert(allg.end(), gpu[c].begin(), gpu[c].end());
  }
  auto pct = [](std::vector<double> v, double q) {
    if (v.empty()) return 0.0;
    std::sort(v.begin(), v.end());
    return v[std::min(v.size() - 1, std::size_t(q * double(v.size())))];
  };
  const double frames_total = double(steps) * batch * clients;
  std::printf("{\"ok\": true, \"clients\": %u, \"steps\": %u, \"batch\": %u, \"frames\": %.0f, \"wall_s\": %.6f, "
              "\"fps\": %.3f, \"ms_per_cycle\": %.4f, \"server_compute_ms\": %.4f, \"model\": \"%s\", "
              "\"cycle_ms\": {\"p50\": %.3f, \"p90\": %.3f, \"max\": %.3f}, "
              "\"comm_ms\": {\"p50\": %.3f, \"p90\": %.3f, \"max\": %.3f}, "
              "\"gpu_ms\": {\"p50\": %.3f, \"p90\": %.3f, \"max\": %.3f}}\n",
              clients, steps, batch, frames_total, wall, frames_total / wall, 1e3 * wall / steps,
              1e3 * cs / (double(steps) * clients), model.c_str(), 1e3 * pct(all, 0.5), 1e3 * pct(all, 0.9),
              1e3 * pct(all, 1.0), 1e3 * pct(allc, 0.5), 1e3 * pct(allc, 0.9), 1e3 * pct(allc, 1.0),
              1e3 * pct(allg, 0.5), 1e3 * pct(allg, 0.9), 1e3 * pct(allg, 1.0));
  return 0;
}
