// Pose-network specs carried in ModelDescriptor.structure.
//
// The reference treats `structure` as opaque bytes (wire.hpp:75) and its
// harness fills it with random data (harness.cpp:355-370). A structure that
// starts with the line "avecnet 1" selects the pose network instead:
//
//     avecnet 1
//     family openpose_coco        # VGG19[:10] + CPM + 6 stages, 19 heat + 38 PAF
//     init he_uniform 1           # weights when the upload carries none (seed)
//
// Weights, when present, are the Caffe-order fp32 blob: for every conv layer
// in prototxt order, W[cout][cin][kh][kw] then bias[cout].
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace avec {

struct ConvDef {
  std::string name;
  int cin, cout, k;
  int relu;
  int level;  // log2 of the downsampling at which the layer runs
};

struct PoseFamily {
  std::string family;
  int stages = 6;
  int paf_channels = 38;   // L1 branch
  int heat_channels = 19;  // L2 branch (18 parts + background)
  int trunk_channels = 128;
  std::vector<ConvDef> convs;  // weights-blob order
  uint64_t init_seed = 1;
  int out_channels() const { return heat_channels + paf_channels; }
  uint64_t weight_floats() const;
};

// true if the structure bytes are an avecnet spec (then parse() must succeed)
bool is_avecnet(const uint8_t* s, size_t n);
// throws Error{AVEC_ERR_INVALID_MODEL} on malformed specs
PoseFamily parse_avecnet(const uint8_t* s, size_t n);
// deterministic He-uniform init, Caffe order; out has weight_floats() entries
void synth_weights(const PoseFamily& f, float* out);

}  // namespace avec
