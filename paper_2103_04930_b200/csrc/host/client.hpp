// Minimal native client of the AVEC wire protocol (reference:
// proj/src/client.cpp Session::ensure_model / forward) used by avec-loadgen to
// measure through-the-wire frames/s. FrameData goes out as header + caller's
// buffer in one writev.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "channel.hpp"
#include "record.hpp"
#include "wire.hpp"

namespace avec::client {

struct RemoteError : std::runtime_error {
  std::uint32_t code;
  RemoteError(std::uint32_t c, const std::string& m) : std::runtime_error(m), code(c) {}
};

class Session {
 public:
  static Session connect(const std::string& endpoint, double timeout_s = 5.0);
  explicit Session(std::unique_ptr<net::Stream> stream);

  void handshake(std::uint32_t version = wire::kProtocolVersion);
  // true on a cache hit (no upload)
  bool ensure_model(const wire::ModelDescriptor& model);
  // one cycle; result floats into `out`; returns the server's compute seconds
  double forward(const float* data, std::uint32_t elems, std::uint32_t width, std::uint32_t height,
                 std::vector<float>& out);
  // the same cycle timed like the reference client (proj/src/client.cpp:160-195)
  record::CycleTiming forward_timed(const float* data, std::uint32_t elems, std::uint32_t width,
                                    std::uint32_t height, std::vector<float>& out);
  void close() { ch_->close(); }
  std::uint64_t bytes_sent() const { return ch_->bytes_sent(); }
  std::uint64_t bytes_received() const { return ch_->bytes_received(); }

 private:
  std::unique_ptr<net::Channel> ch_;
};

}  // namespace avec::client
