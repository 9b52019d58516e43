// Pose-network specs carried in ModelDescriptor.structure.
//
// The reference treats `structure` as opaque bytes (wire.hpp:75) and its
// harness fills it with random data (harness.cpp:355-370). A structure that
// starts with the line "avecnet 1" selects a pose network instead:
//
//     avecnet 1
//     family openpose_coco        # or openpose_body25
//     init he_uniform 1           # weights when the upload carries none (seed)
//
// Weights, when present, are the Caffe-order fp32 blob: for every conv layer
// in prototxt order, W[cout][cin][kh][kw], bias[cout], and — for layers with a
// PReLU — the per-channel slopes[cout].
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace avec {

enum ConvAct : int { kActNone = 0, kActRelu = 1, kActPrelu = 2 };

struct ConvDef {
  std::string name;
  int cin, cout, k;
  int act;    // ConvAct
  int level;  // log2 of the downsampling at which the layer runs
  // Stage-input layers read a concat buffer whose internal channel order
  // differs from Caffe's concat order: cin_map[ci] = internal channel (relative
  // to the layer's input window) of Caffe input channel ci; empty = identity.
  std::vector<int> cin_map;
  int cin_pad = 0;  // internal input width (multiple of 64); 0 = round_up(cin, 64)
};

struct PoseFamily {
  std::string family;
  int stages = 6;            // COCO: total stages (>= 2)
  int paf_channels = 38;     // COCO L1 / BODY_25 L2 branch
  int heat_channels = 19;    // COCO L2 / BODY_25 L1 branch (parts + background)
  int trunk_channels = 128;
  std::vector<ConvDef> convs;  // weights-blob order
  uint64_t init_seed = 1;
  // "input tf32": conv1_1 takes the fp32 frames as tf32 operands (10-bit
  // mantissa) instead of bf16 (7-bit); every later layer stays bf16
  bool input_tf32 = false;
  int out_channels() const { return heat_channels + paf_channels; }
  uint64_t weight_floats() const;
  bool body25() const { return family == "openpose_body25"; }
};

// true if the structure bytes are an avecnet spec (then parse() must succeed)
bool is_avecnet(const uint8_t* s, size_t n);
// throws Error{AVEC_ERR_INVALID_MODEL} on malformed specs
PoseFamily parse_avecnet(const uint8_t* s, size_t n);
// deterministic He-uniform init, Caffe order; out has weight_floats() entries
void synth_weights(const PoseFamily& f, float* out);

// Stage-concat buffer layouts. Each head slot starts on an 8-channel boundary
// and owns the channels up to the next one (the pixel-major epilogue stores
// 8-channel-granular TMA boxes).
// COCO (192 channels): [trunk 0..127 | PAF 128..165 | pad | heat 168..186 | pad]
constexpr int kCocoCatChannels = 192;
constexpr int kCocoPaf = 128, kCocoHeat = 168;
// BODY_25 (256 channels):
//   [heat 0..25 | pad | PAF 32..83 | pad | trunk 88..215 | pad]
// so every stage input is ONE contiguous, 16-byte aligned channel window:
// PAF stages 1..3 and heat stage 0 read [32, 216), heat stage 1 reads [0, 216).
constexpr int kB25CatChannels = 256;
constexpr int kB25Heat = 0, kB25Paf = 32, kB25Trunk = 88;

}  // namespace avec
