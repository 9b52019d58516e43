// The reference-side binding a maintainer of accelfwd would add: an
// accelfwd::backend::Backend (proj/include/accelfwd/backend.hpp:64-78) that
// forwards to the B200 engine through its C-ABI (include/avec_cuda.h).
// Reproduced in INTEGRATION.md; compiled here against the reference library
// to run the reference's OWN Server on the B200 (ref_b200_server.cpp).
#pragma once

#include <stdexcept>
#include <string>

#include "accelfwd/backend.hpp"
#include "accelfwd/error.hpp"
#include "avec_cuda.h"

namespace accelfwd::backend {

class B200Backend final : public Backend {
 public:
  explicit B200Backend(int device = 0) {
    if (avec_ctx_create(device, 2, &ctx_) != AVEC_OK)
      raise(ErrorCode::invalid_model, std::string("B200 unavailable: ") + avec_last_error());
    label_ = avec_ctx_label(ctx_);
  }
  ~B200Backend() override { avec_ctx_destroy(ctx_); }

  ModelHandle register_model(const ModelDescriptor& m) override {
    std::uint64_t h = 0;
    check(avec_model_register(ctx_, m.digest.data(), m.name.data(), m.name.size(), m.structure.data(),
                              m.structure.size(), m.weights.data(), m.weights.size(), m.output_divisor, &h));
    return {h};
  }

  Heatmap forward(ModelHandle model, const Frame& f) override {
    const auto& d = f.dims;
    std::uint64_t k = 0;
    check(avec_output_elems(ctx_, model.id, d.batch, d.channels, d.height, d.width, &k));
    Heatmap h;
    h.data.resize(k);
    check(avec_forward(ctx_, model.id, d.batch, d.channels, d.height, d.width, f.data.data(), f.data.size(),
                       h.data.data(), h.data.size(), nullptr));
    return h;
  }

  std::string_view label() const override { return label_; }

 private:
  // AVEC_* codes -> the exceptions MockPoseBackend throws (backend.cpp:43-93)
  static void check(int rc) {
    if (rc == AVEC_OK) return;
    const std::string msg = avec_last_error();
    switch (rc) {
      // a shape the net rejects comes from the client's own FrameData/Resolution; the
      // reference Server only catches accelfwd::Error (server.cpp:315, 334), so it must
      // not leave as std::invalid_argument (that would terminate the server)
      case AVEC_ERR_INVALID_ARGUMENT: raise(ErrorCode::invariant_violation, msg);
      case AVEC_ERR_UNKNOWN_MODEL: raise(ErrorCode::unknown_model, msg);
      case AVEC_ERR_INVALID_MODEL: raise(ErrorCode::invalid_model, msg);
      case AVEC_ERR_DEGENERATE_OUTPUT: raise(ErrorCode::degenerate_output, msg);
      default: raise(ErrorCode::invariant_violation, "B200: " + msg);  // -> WireError::internal
    }
  }
  avec_ctx* ctx_ = nullptr;
  std::string label_;
};

}  // namespace accelfwd::backend
