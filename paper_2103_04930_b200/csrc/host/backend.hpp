// Compute plugin contract of the destination server, mirroring
// accelfwd::backend::Backend (proj/include/accelfwd/backend.hpp:64-78):
// register_model (idempotent per digest, handles from 1), forward, label.
//
// The B200 server needs two more things from a backend, both with defaults so
// any reference-style backend still plugs in:
//  * forward_into: zero-copy forward from the session's pinned ingest buffer
//    into its pinned egress buffer, returning the device-measured compute
//    seconds shipped as ForwardResult.compute_s (wire.hpp:122);
//  * concurrency: how many forwards may run at once (GPUs x slots), so the
//    dispatcher can keep every device busy while preserving FIFO dispatch.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "wire.hpp"

namespace avec::backend {

// reference ErrorCode values a backend raises (error.hpp:8-41)
enum class ErrorCode { invalid_model, unknown_model, degenerate_output, internal, bad_config };

struct Error : std::runtime_error {
  ErrorCode code;
  Error(ErrorCode c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct Frame {
  wire::Dims dims;
  std::vector<float> data;  // flattened, batch-major
};

struct Heatmap {
  std::vector<float> data;
  std::uint64_t elem_count() const { return data.size(); }
};

struct ModelHandle {
  std::uint64_t id = 0;  // valid ids start at 1
  bool operator==(const ModelHandle&) const = default;
};

// A session's pipelined cycle (receive / H2D / compute / D2H overlap): begun
// when a FrameData header arrives with the dims the session's previous cycle
// had, fed as the payload lands in the pinned frame buffer, finished by the
// dispatcher (or aborted when Resolution disagrees with the guess).
class Pipeline {
 public:
  virtual ~Pipeline() = default;
  // false: declined (e.g. the device is busy with other cycles, where whole
  // batches use it better); the cycle then takes the dispatcher's normal path
  virtual bool begin(ModelHandle model, const wire::Dims& dims, const float* in, float* out, std::uint64_t n_out) = 0;
  // build what a cycle of these dims needs (plans, staging) off the critical
  // path; the server calls it from a helper thread before speculating
  virtual void prepare(ModelHandle /*model*/, const wire::Dims& /*dims*/) {}
  virtual void feed(std::uint64_t landed_bytes) = 0;
  virtual double finish() = 0;  // blocks; device compute seconds of the cycle
  virtual void abort() = 0;
};

class Backend {
 public:
  virtual ~Backend() = default;

  // Throws Error{invalid_model}.
  virtual ModelHandle register_model(const wire::ModelDescriptor& model) = 0;
  // Throws Error{unknown_model | degenerate_output | internal}, std::invalid_argument.
  virtual Heatmap forward(ModelHandle model, const Frame& frame) = 0;
  virtual std::string_view label() const = 0;

  // ---- B200 server extensions (defaults go through forward()) ----
  virtual bool zero_copy() const { return false; }
  virtual std::uint64_t output_elems(ModelHandle, const wire::Dims&) {
    throw Error(ErrorCode::internal, "output_elems unsupported by this backend");
  }
  virtual double forward_into(ModelHandle, const wire::Dims&, const float*, std::uint64_t, float*,
                              std::uint64_t) {
    throw Error(ErrorCode::internal, "forward_into unsupported by this backend");
  }
  // the server's call: `session` lets a multi-device backend pin sessions
  virtual double forward_session(std::uint64_t /*session*/, ModelHandle h, const wire::Dims& d, const float* in,
                                 std::uint64_t n_in, float* out, std::uint64_t n_out) {
    return forward_into(h, d, in, n_in, out, n_out);
  }
  virtual int concurrency() const { return 1; }
  virtual int devices() const { return 1; }
  // per-session pipelined cycles; nullptr: the backend has none
  virtual std::unique_ptr<Pipeline> open_pipeline(std::uint64_t /*session*/) { return nullptr; }
  // host memory for ingest/egress staging (pinned when the backend can)
  virtual void* alloc_host(std::size_t bytes);
  virtual void free_host(void* p);
};

}  // namespace avec::backend
