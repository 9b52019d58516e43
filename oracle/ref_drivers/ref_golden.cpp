// Emits golden vectors computed by the REFERENCE library itself, as JSON on
// stdout. tests/golden/make_golden.py runs this and commits the result so the
// GPU box (which has no /root/reference) can still check against it.
//
// Covers: output_elems / transfer_size (wire.cpp:18-27), gen_frame
// (harness.cpp:29-42), synth_model (harness.cpp:355-370), segment_means /
// mockpose_forward (backend.cpp:39-67), model_digest (wire.cpp:70-79) and the
// acceptance-9 brute-force instances (acceptance.cpp:386-421).
#include <cinttypes>
#include <random>

#include "accelfwd/error.hpp"

#include "ref_common.hpp"

using namespace accelfwd;

static void print_floats_hex(const std::vector<float>& v) {
  std::printf("[");
  for (std::size_t i = 0; i < v.size(); ++i) {
    std::uint32_t b;
    std::memcpy(&b, &v[i], 4);
    std::printf("%s%u", i ? "," : "", b);
  }
  std::printf("]");
}

static void print_doubles_bits(const std::vector<double>& v) {
  std::printf("[");
  for (std::size_t i = 0; i < v.size(); ++i) {
    std::uint64_t b;
    std::memcpy(&b, &v[i], 8);
    std::printf("%s\"%016" PRIx64 "\"", i ? "," : "", b);
  }
  std::printf("]");
}

int main() {
  std::printf("{\n");

  // ---- sizing law ----
  struct OE { std::uint64_t e; double c; };
  const OE oes[] = {{5, 2.0}, {3, 2.0}, {10, 3.0}, {1, 3.0}, {724224, 3.368421},
                    {406272, 3.368421}, {5793792, 192.0 / 57.0},
                    {92700672, 192.0 / 78.0}, {7, 0.5}, {1000001, 1.7}};
  std::printf("\"output_elems\": [");
  for (std::size_t i = 0; i < sizeof(oes) / sizeof(oes[0]); ++i) {
    std::uint64_t cbits;
    std::memcpy(&cbits, &oes[i].c, 8);
    std::printf("%s[%" PRIu64 ", \"%016" PRIx64 "\", %" PRIu64 "]", i ? ", " : "",
                oes[i].e, cbits, wire::output_elems(oes[i].e, oes[i].c));
  }
  std::printf("],\n");

  struct TS { wire::Dims d; double c; };
  const TS tss[] = {{{1, 3, 368, 656}, 3.368421}, {{1, 1, 1, 1}, 1.0},
                    {{1, 3, 100, 100}, 3.368421}, {{1, 24, 368, 656}, 192.0 / 57.0},
                    {{1, 96, 736, 1312}, 192.0 / 78.0}, {{1, 3, 368, 368}, 3.368421}};
  std::printf("\"transfer_size\": [");
  for (std::size_t i = 0; i < sizeof(tss) / sizeof(tss[0]); ++i) {
    std::uint64_t cbits;
    std::memcpy(&cbits, &tss[i].c, 8);
    std::printf("%s[%u, %u, %u, %u, \"%016" PRIx64 "\", %" PRIu64 "]", i ? ", " : "",
                tss[i].d.batch, tss[i].d.channels, tss[i].d.height, tss[i].d.width,
                cbits, wire::transfer_size(tss[i].d, tss[i].c));
  }
  std::printf("],\n");

  // ---- frame generator: small frame in full, big frames by digest ----
  {
    harness::Workload w;
    w.width = 8;
    w.height = 4;
    w.seed = 7;
    auto f = harness::gen_frame(w, 3);
    std::printf("\"gen_frame_small\": {\"w\": 8, \"h\": 4, \"seed\": 7, \"index\": 3, \"bits\": ");
    print_floats_hex(f.data);
    std::printf("},\n");
  }
  struct GF { std::uint32_t w, h; std::uint64_t seed; std::uint32_t index; double c; };
  const GF gfs[] = {{368, 368, 7, 0, 3.368421}, {656, 368, 7, 0, 3.368421},
                    {1312, 736, 7, 0, 3.368421}, {656, 368, 7, 5, 192.0 / 57.0},
                    {64, 64, 100, 3, 2.0}, {100, 100, 0x123456789abcdefULL, 1, 3.368421},
                    {37, 11, 42, 9, 1.5}};
  std::printf("\"gen_frame\": [");
  for (std::size_t i = 0; i < sizeof(gfs) / sizeof(gfs[0]); ++i) {
    harness::Workload w;
    w.width = gfs[i].w;
    w.height = gfs[i].h;
    w.seed = gfs[i].seed;
    auto f = harness::gen_frame(w, gfs[i].index);
    auto heat = backend::mockpose_forward(f, gfs[i].c);
    std::uint64_t cbits;
    std::memcpy(&cbits, &gfs[i].c, 8);
    std::printf("%s{\"w\": %u, \"h\": %u, \"seed\": %" PRIu64 ", \"index\": %u, "
                "\"frame_sha256\": \"%s\", \"divisor_bits\": \"%016" PRIx64 "\", "
                "\"k\": %zu, \"heat_sha256\": \"%s\", \"heat_first\": ",
                i ? ", " : "", gfs[i].w, gfs[i].h, gfs[i].seed, gfs[i].index,
                refdrv::digest_floats(f.data).c_str(), cbits, heat.data.size(),
                refdrv::digest_floats(heat.data).c_str());
    std::vector<float> first(heat.data.begin(), heat.data.begin() + 3);
    print_floats_hex(first);
    std::printf("}");
  }
  std::printf("],\n");

  // ---- batched frame (C2 shape) ----
  {
    auto f = refdrv::batched_frame(656, 368, 8, 7, 0);
    auto heat = backend::mockpose_forward(f, 192.0 / 57.0);
    std::printf("\"batched_c2\": {\"w\": 656, \"h\": 368, \"batch\": 8, \"seed\": 7, "
                "\"frame_sha256\": \"%s\", \"k\": %zu, \"heat_sha256\": \"%s\"},\n",
                refdrv::digest_floats(f.data).c_str(), heat.data.size(),
                refdrv::digest_floats(heat.data).c_str());
  }

  // ---- synthetic models ----
  std::printf("\"synth_model\": [");
  {
    harness::ModelSpec specs[3];
    specs[1].name = "stress-2";
    specs[1].output_divisor = 2.5;
    specs[1].weights_bytes = 32 * 1024;
    specs[1].seed = 7002;
    specs[2].structure_bytes = 13;
    specs[2].weights_bytes = 29;
    specs[2].seed = 99;
    for (int i = 0; i < 3; ++i) {
      auto m = harness::synth_model(specs[i]);
      std::uint64_t cbits;
      std::memcpy(&cbits, &specs[i].output_divisor, 8);
      std::printf("%s{\"name\": \"%s\", \"structure_bytes\": %u, \"weights_bytes\": %u, "
                  "\"divisor_bits\": \"%016" PRIx64 "\", \"seed\": %" PRIu64 ", "
                  "\"structure_sha256\": \"%s\", \"weights_sha256\": \"%s\", "
                  "\"digest\": \"%s\"}",
                  i ? ", " : "", specs[i].name.c_str(), specs[i].structure_bytes,
                  specs[i].weights_bytes, cbits, specs[i].seed,
                  wire::hex(wire::sha256(m.structure)).c_str(),
                  wire::hex(wire::sha256(m.weights)).c_str(),
                  wire::hex(m.digest).c_str());
    }
  }
  std::printf("],\n");

  // ---- brute-force segment-mean instances (acceptance.cpp:386-421 recipe) ----
  std::printf("\"segment_means\": [");
  {
    std::mt19937_64 rng(0x0bace1e5);
    int emitted = 0;
    for (int i = 0; i < 60; ++i) {
      std::uint64_t e = std::uniform_int_distribution<std::uint64_t>(1, 300)(rng);
      double c = e == 1 ? 1.0
                        : std::uniform_real_distribution<double>(1.0, double(e))(rng);
      std::vector<float> data(e);
      std::uniform_real_distribution<float> df(-8.0f, 8.0f);
      for (auto& x : data) x = df(rng);
      std::uint64_t k = wire::output_elems(e, c);
      if (k < 1 || k > e) continue;
      auto means = backend::segment_means(data, c);
      std::uint64_t cbits;
      std::memcpy(&cbits, &c, 8);
      std::printf("%s{\"divisor_bits\": \"%016" PRIx64 "\", \"data\": ", emitted ? ", " : "",
                  cbits);
      print_floats_hex(data);
      std::printf(", \"means\": ");
      print_doubles_bits(means);
      std::printf("}");
      ++emitted;
    }
  }
  std::printf("],\n");

  // ---- degenerate cases (test_backend.cpp:104-120) ----
  std::printf("\"degenerate\": [");
  {
    struct D { std::vector<float> data; double c; };
    D ds[] = {{{1.0f}, 3.0}, {{1, 2, 3, 4}, 0.3}};
    for (int i = 0; i < 2; ++i) {
      std::string what = "ok";
      try {
        backend::segment_means(ds[i].data, ds[i].c);
      } catch (const Error& e) {
        what = to_string(e.code());
      }
      std::printf("%s{\"n\": %zu, \"c\": %.17g, \"error\": \"%s\"}", i ? ", " : "",
                  ds[i].data.size(), ds[i].c, what.c_str());
    }
  }
  std::printf("]\n}\n");
  return 0;
}
