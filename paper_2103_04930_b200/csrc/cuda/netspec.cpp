// Pose-network family tables (OpenPose pose_deploy_linevec.prototxt, COCO).
#include "netspec.hpp"

#include <cmath>
#include <cstring>
#include <sstream>

#include "engine.hpp"

namespace avec {

uint64_t PoseFamily::weight_floats() const {
  uint64_t n = 0;
  for (const auto& c : convs) n += uint64_t(c.cout) * c.cin * c.k * c.k + c.cout;
  return n;
}

bool is_avecnet(const uint8_t* s, size_t n) {
  static const char kMagic[] = "avecnet 1";
  return n >= sizeof(kMagic) - 1 && std::memcmp(s, kMagic, sizeof(kMagic) - 1) == 0 &&
         (n == sizeof(kMagic) - 1 || s[sizeof(kMagic) - 1] == '\n' ||
          s[sizeof(kMagic) - 1] == '\r' || s[sizeof(kMagic) - 1] == ' ');
}

namespace {

void add(PoseFamily& f, const std::string& name, int cin, int cout, int k, int relu, int level) {
  f.convs.push_back({name, cin, cout, k, relu, level});
}

// VGG-19 first ten convolutions + the two CPM adapters, then the two-branch
// stages: stage 1 (3x3 convs) and stages 2..S (7x7 convs) whose input is the
// concat of the previous stage's two outputs and the 128-channel trunk.
void build_coco(PoseFamily& f) {
  add(f, "conv1_1", 3, 64, 3, 1, 0);
  add(f, "conv1_2", 64, 64, 3, 1, 0);
  add(f, "conv2_1", 64, 128, 3, 1, 1);
  add(f, "conv2_2", 128, 128, 3, 1, 1);
  add(f, "conv3_1", 128, 256, 3, 1, 2);
  add(f, "conv3_2", 256, 256, 3, 1, 2);
  add(f, "conv3_3", 256, 256, 3, 1, 2);
  add(f, "conv3_4", 256, 256, 3, 1, 2);
  add(f, "conv4_1", 256, 512, 3, 1, 3);
  add(f, "conv4_2", 512, 512, 3, 1, 3);
  add(f, "conv4_3_CPM", 512, 256, 3, 1, 3);
  add(f, "conv4_4_CPM", 256, 128, 3, 1, 3);
  const int outs[2] = {f.paf_channels, f.heat_channels};
  for (int b = 0; b < 2; ++b) {
    const std::string L = b == 0 ? "_L1" : "_L2";
    add(f, "conv5_1_CPM" + L, 128, 128, 3, 1, 3);
    add(f, "conv5_2_CPM" + L, 128, 128, 3, 1, 3);
    add(f, "conv5_3_CPM" + L, 128, 128, 3, 1, 3);
    add(f, "conv5_4_CPM" + L, 128, 512, 1, 1, 3);
    add(f, "conv5_5_CPM" + L, 512, outs[b], 1, 0, 3);
  }
  const int cat = f.paf_channels + f.heat_channels + f.trunk_channels;  // 185
  for (int t = 2; t <= f.stages; ++t) {
    for (int b = 0; b < 2; ++b) {
      const std::string sfx = "_stage" + std::to_string(t) + (b == 0 ? "_L1" : "_L2");
      add(f, "Mconv1" + sfx, cat, 128, 7, 1, 3);
      for (int i = 2; i <= 5; ++i) add(f, "Mconv" + std::to_string(i) + sfx, 128, 128, 7, 1, 3);
      add(f, "Mconv6" + sfx, 128, 128, 1, 1, 3);
      add(f, "Mconv7" + sfx, 128, outs[b], 1, 0, 3);
    }
  }
}

}  // namespace

PoseFamily parse_avecnet(const uint8_t* s, size_t n) {
  if (!is_avecnet(s, n)) fail(AVEC_ERR_INVALID_MODEL, "structure is not an avecnet spec");
  std::istringstream in(std::string(reinterpret_cast<const char*>(s), n));
  std::string line;
  PoseFamily f;
  bool have_family = false;
  std::getline(in, line);  // magic
  while (std::getline(in, line)) {
    auto hash = line.find('#');
    if (hash != std::string::npos) line = line.substr(0, hash);
    std::istringstream ls(line);
    std::string key;
    if (!(ls >> key)) continue;
    if (key == "family") {
      ls >> f.family;
      have_family = true;
    } else if (key == "stages") {
      ls >> f.stages;
      if (f.stages < 2 || f.stages > 6) fail(AVEC_ERR_INVALID_MODEL, "stages must be 2..6");
    } else if (key == "init") {
      std::string kind;
      ls >> kind >> f.init_seed;
      if (kind != "he_uniform") fail(AVEC_ERR_INVALID_MODEL, "unknown init " + kind);
    } else {
      fail(AVEC_ERR_INVALID_MODEL, "unknown avecnet key: " + key);
    }
  }
  if (!have_family) fail(AVEC_ERR_INVALID_MODEL, "avecnet spec without family");
  if (f.family == "openpose_coco") {
    build_coco(f);
  } else {
    fail(AVEC_ERR_INVALID_MODEL, "unknown pose-net family: " + f.family);
  }
  return f;
}

// splitmix64 stream per layer; u in [0,1) with 24 bits; w = (2u-1)*sqrt(6/fan_in)
void synth_weights(const PoseFamily& f, float* out) {
  uint64_t off = 0;
  for (size_t li = 0; li < f.convs.size(); ++li) {
    const ConvDef& c = f.convs[li];
    uint64_t state = f.init_seed ^ (0x9E3779B97F4A7C15ULL * (li + 1));
    auto next = [&state]() {
      state += 0x9E3779B97F4A7C15ULL;
      uint64_t z = state;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
      return z ^ (z >> 31);
    };
    const double fan_in = double(c.cin) * c.k * c.k;
    const double a = std::sqrt(6.0 / fan_in);
    const uint64_t nw = uint64_t(c.cout) * c.cin * c.k * c.k;
    for (uint64_t i = 0; i < nw; ++i) {
      double u = double(next() >> 40) * (1.0 / 16777216.0);
      out[off++] = float((2.0 * u - 1.0) * a);
    }
    for (int i = 0; i < c.cout; ++i) {
      double u = double(next() >> 40) * (1.0 / 16777216.0);
      out[off++] = float((2.0 * u - 1.0) * 0.05);
    }
  }
}

}  // namespace avec
