// Pose-network family tables.
//  * openpose_coco: OpenPose pose_deploy_linevec.prototxt (COCO, 18 parts).
//  * openpose_body25: OpenPose body_25/pose_deploy.prototxt, restated from
//    the public prototxt's structure (PReLU, dense 3-conv blocks, 4 PAF + 2
//    heatmap stages). Its MAC count reproduces SURVEY.md §8(d): 301,248 (VGG +
//    CPM) + 293,722 (stages) = 594,970 MAC per input pixel.
#include "netspec.hpp"

#include <cmath>
#include <cstring>
#include <sstream>

#include "engine.hpp"

namespace avec {

uint64_t PoseFamily::weight_floats() const {
  uint64_t n = 0;
  for (const auto& c : convs)
    n += uint64_t(c.cout) * c.cin * c.k * c.k + c.cout + (c.act == kActPrelu ? c.cout : 0);
  return n;
}

bool is_avecnet(const uint8_t* s, size_t n) {
  static const char kMagic[] = "avecnet 1";
  return n >= sizeof(kMagic) - 1 && std::memcmp(s, kMagic, sizeof(kMagic) - 1) == 0 &&
         (n == sizeof(kMagic) - 1 || s[sizeof(kMagic) - 1] == '\n' ||
          s[sizeof(kMagic) - 1] == '\r' || s[sizeof(kMagic) - 1] == ' ');
}

namespace {

ConvDef& add(PoseFamily& f, const std::string& name, int cin, int cout, int k, int act, int level) {
  ConvDef d;
  d.name = name;
  d.cin = cin;
  d.cout = cout;
  d.k = k;
  d.act = act;
  d.level = level;
  f.convs.push_back(d);
  return f.convs.back();
}

// VGG-19 first ten convolutions + the two CPM adapters; BODY_25 replaces the
// ReLUs from conv4_2 on with PReLUs.
void add_trunk(PoseFamily& f, int late_act) {
  add(f, "conv1_1", 3, 64, 3, kActRelu, 0);
  add(f, "conv1_2", 64, 64, 3, kActRelu, 0);
  add(f, "conv2_1", 64, 128, 3, kActRelu, 1);
  add(f, "conv2_2", 128, 128, 3, kActRelu, 1);
  add(f, "conv3_1", 128, 256, 3, kActRelu, 2);
  add(f, "conv3_2", 256, 256, 3, kActRelu, 2);
  add(f, "conv3_3", 256, 256, 3, kActRelu, 2);
  add(f, "conv3_4", 256, 256, 3, kActRelu, 2);
  add(f, "conv4_1", 256, 512, 3, kActRelu, 3);
  add(f, "conv4_2", 512, 512, 3, late_act, 3);
  add(f, "conv4_3_CPM", 512, 256, 3, late_act, 3);
  add(f, "conv4_4_CPM", 256, 128, 3, late_act, 3);
}

// COCO: stage 1 (3x3 convs) and stages 2..S (7x7 convs) whose input is the
// concat [L1, L2, trunk] of the previous stage's outputs and the trunk.
void build_coco(PoseFamily& f) {
  add_trunk(f, kActRelu);
  const int outs[2] = {f.paf_channels, f.heat_channels};
  for (int b = 0; b < 2; ++b) {
    const std::string L = b == 0 ? "_L1" : "_L2";
    add(f, "conv5_1_CPM" + L, 128, 128, 3, kActRelu, 3);
    add(f, "conv5_2_CPM" + L, 128, 128, 3, kActRelu, 3);
    add(f, "conv5_3_CPM" + L, 128, 128, 3, kActRelu, 3);
    add(f, "conv5_4_CPM" + L, 128, 512, 1, kActRelu, 3);
    add(f, "conv5_5_CPM" + L, 512, outs[b], 1, kActNone, 3);
  }
  const int branches = f.paf_channels + f.heat_channels;
  const int cat = branches + f.trunk_channels;  // 185
  // internal concat layout (netspec.hpp): [trunk | L1 at kCocoPaf | L2 at
  // kCocoHeat]; Caffe order is [L1, L2, trunk]
  if (f.trunk_channels != kCocoPaf || kCocoPaf + f.paf_channels > kCocoHeat ||
      kCocoHeat + f.heat_channels > kCocoCatChannels)
    fail(AVEC_ERR_INVALID_MODEL, "COCO stage concat layout does not fit");
  std::vector<int> map(cat);
  for (int ci = 0; ci < cat; ++ci)
    map[ci] = ci < f.paf_channels ? kCocoPaf + ci
              : ci < branches     ? kCocoHeat + (ci - f.paf_channels)
                                  : ci - branches;
  for (int t = 2; t <= f.stages; ++t) {
    for (int b = 0; b < 2; ++b) {
      const std::string sfx = "_stage" + std::to_string(t) + (b == 0 ? "_L1" : "_L2");
      ConvDef& m1 = add(f, "Mconv1" + sfx, cat, 128, 7, kActRelu, 3);
      m1.cin_map = map;
      m1.cin_pad = 192;
      for (int i = 2; i <= 5; ++i) add(f, "Mconv" + std::to_string(i) + sfx, 128, 128, 7, kActRelu, 3);
      add(f, "Mconv6" + sfx, 128, 128, 1, kActRelu, 3);
      add(f, "Mconv7" + sfx, 128, outs[b], 1, kActNone, 3);
    }
  }
}

// one BODY_25 stage: 5 dense blocks of three 3x3 convs (width w, PReLU) whose
// outputs concatenate to 3w, then Mconv6 (1x1, PReLU) and Mconv7 (1x1 head)
void add_b25_stage(PoseFamily& f, const std::string& sfx, int cin, int w, int c6, int out,
                   const std::vector<int>& map, int cin_pad) {
  for (int blk = 1; blk <= 5; ++blk) {
    for (int j = 0; j < 3; ++j) {
      const int ci = j > 0 ? w : (blk == 1 ? cin : 3 * w);
      ConvDef& d = add(f, "Mconv" + std::to_string(blk) + sfx + "_" + std::to_string(j), ci, w, 3,
                       kActPrelu, 3);
      if (blk == 1 && j == 0) {
        d.cin_map = map;
        d.cin_pad = cin_pad;
      }
    }
  }
  add(f, "Mconv6" + sfx, 3 * w, c6, 1, kActPrelu, 3);
  add(f, "Mconv7" + sfx, c6, out, 1, kActNone, 3);
}

void build_body25(PoseFamily& f) {
  f.paf_channels = 52;   // 26 limbs x 2 (L2 branch)
  f.heat_channels = 26;  // 25 parts + background (L1 branch)
  add_trunk(f, kActPrelu);
  const int T = f.trunk_channels, P = f.paf_channels, Hc = f.heat_channels;
  // [trunk, PAF] (Caffe concat_stageN_L2 / concat_stage0_L1) read from window [32, 216):
  // PAF at 0..51, trunk at 56..183 inside the window
  std::vector<int> tp(T + P);
  for (int ci = 0; ci < T + P; ++ci) tp[ci] = ci < T ? (kB25Trunk - kB25Paf) + ci : ci - T;
  // [trunk, heat, PAF] (concat_stage1_L1) read from window [0, 216)
  std::vector<int> thp(T + Hc + P);
  for (int ci = 0; ci < T + Hc + P; ++ci)
    thp[ci] = ci < T ? kB25Trunk + ci : ci < T + Hc ? kB25Heat + (ci - T) : kB25Paf + (ci - T - Hc);
  add_b25_stage(f, "_stage0_L2", T, 96, 256, P, {}, 0);
  for (int t = 1; t <= 3; ++t) add_b25_stage(f, "_stage" + std::to_string(t) + "_L2", T + P, 128, 512, P, tp, 192);
  add_b25_stage(f, "_stage0_L1", T + P, 96, 256, Hc, tp, 192);
  add_b25_stage(f, "_stage1_L1", T + Hc + P, 128, 512, Hc, thp, 256);
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
    } else if (key == "input") {
      std::string dt;
      ls >> dt;
      if (dt != "bf16" && dt != "tf32") fail(AVEC_ERR_INVALID_MODEL, "input must be bf16 or tf32");
      f.input_tf32 = dt == "tf32";
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
  } else if (f.family == "openpose_body25") {
    build_body25(f);
  } else {
    fail(AVEC_ERR_INVALID_MODEL, "unknown pose-net family: " + f.family);
  }
  return f;
}

// splitmix64 stream per layer; u in [0,1) with 24 bits; w = (2u-1)*sqrt(6/fan_in),
// bias = (2u-1)*0.05, PReLU slope = 0.25 * (1 + (2u-1)*0.5)
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
    auto unit = [&]() { return double(next() >> 40) * (1.0 / 16777216.0); };
    const double fan_in = double(c.cin) * c.k * c.k;
    const double a = std::sqrt(6.0 / fan_in);
    const uint64_t nw = uint64_t(c.cout) * c.cin * c.k * c.k;
    for (uint64_t i = 0; i < nw; ++i) out[off++] = float((2.0 * unit() - 1.0) * a);
    for (int i = 0; i < c.cout; ++i) out[off++] = float((2.0 * unit() - 1.0) * 0.05);
    if (c.act == kActPrelu)
      for (int i = 0; i < c.cout; ++i) out[off++] = float(0.25 * (1.0 + (2.0 * unit() - 1.0) * 0.5));
  }
}

}  // namespace avec
