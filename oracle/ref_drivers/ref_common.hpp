// Shared helpers for the drivers that link the reference library (accelfwd).
// TEST INFRASTRUCTURE ONLY: these programs are checkers and the CPU baseline,
// never part of the product path.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "accelfwd/backend.hpp"
#include "accelfwd/harness.hpp"
#include "accelfwd/wire.hpp"

namespace refdrv {

// --key value argument map; flags without value get "1"
inline std::map<std::string, std::string> parse_args(int argc, char** argv) {
  std::map<std::string, std::string> a;
  for (int i = 1; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) throw std::invalid_argument("bad arg " + k);
    k = k.substr(2);
    if (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0)
      a[k] = argv[++i];
    else
      a[k] = "1";
  }
  return a;
}

inline std::string get(const std::map<std::string, std::string>& a,
                       const std::string& k, const std::string& dflt) {
  auto it = a.find(k);
  return it == a.end() ? dflt : it->second;
}

inline std::vector<std::uint8_t> read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  return std::vector<std::uint8_t>((std::istreambuf_iterator<char>(in)),
                                   std::istreambuf_iterator<char>());
}

// batch of `batch` consecutive harness frames folded into channels (3*batch),
// exactly as the wire carries a batched FrameData (server.cpp:297-301)
inline accelfwd::backend::Frame batched_frame(std::uint32_t w, std::uint32_t h,
                                             std::uint32_t batch,
                                             std::uint64_t seed,
                                             std::uint32_t first_index) {
  accelfwd::harness::Workload wl;
  wl.kind = accelfwd::backend::WorkloadKind::video;
  wl.width = w;
  wl.height = h;
  wl.seed = seed;
  accelfwd::backend::Frame f;
  f.dims = {1, 3 * batch, h, w};
  f.data.reserve(f.dims.elem_count());
  for (std::uint32_t b = 0; b < batch; ++b) {
    auto one = accelfwd::harness::gen_frame(wl, first_index + b);
    f.data.insert(f.data.end(), one.data.begin(), one.data.end());
  }
  return f;
}

inline std::string digest_floats(const std::vector<float>& v) {
  return accelfwd::wire::hex(accelfwd::wire::sha256(
      {reinterpret_cast<const std::uint8_t*>(v.data()), v.size() * 4}));
}

}  // namespace refdrv
