// Framed messages over a Stream (reference: proj/include/accelfwd/channel.hpp).
//
// Same decode/poison contract as accelfwd::net::MessageChannel
// (proj/src/channel.cpp:21-54): an unknown tag or malformed payload poisons
// the stream; EOF inside a frame poisons it too. The B200-specific part is the
// ingest path: a FrameData payload (the frame tensor, tens of MB) is read from
// the socket directly into memory handed out by a FrameSink — the session's
// pinned staging buffer that the H2D copy reads — instead of through a 256 KiB
// vector per read, a reassembly buffer and a std::vector<float> copy
// (transport.cpp:62-77, channel.cpp:44-52, wire.cpp:326-333).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "net.hpp"
#include "wire.hpp"

namespace avec::net {

struct ProtocolError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class FrameSink {
 public:
  virtual ~FrameSink() = default;
  // destination for `elems` floats of an incoming FrameData (valid until the
  // next call); nullptr makes the channel buffer the message instead
  virtual float* frame_buffer(std::uint32_t elems) = 0;
  // same for an incoming ForwardResult (clients); default: buffer it
  virtual float* result_buffer(std::uint32_t /*elems*/) { return nullptr; }
  // a streamed FrameData has `bytes` of its payload in the frame buffer
  // (called after every socket read; lets the server start copies early)
  virtual void frame_progress(std::size_t /*bytes*/) {}
};

class Channel {
 public:
  explicit Channel(std::unique_ptr<Stream> stream);

  void send(const wire::Message& m);
  // header bytes followed by a payload region, one gather write
  void send_parts(const void* head, std::size_t head_len, const void* payload, std::size_t payload_len);

  // Blocks for the next message. Throws NetError{disconnected|timeout} and
  // ProtocolError (the stream is then poisoned and every later call throws).
  wire::Message recv(FrameSink* sink = nullptr);

  std::uint64_t bytes_sent() const { return sent_; }
  std::uint64_t bytes_received() const { return received_; }
  void set_recv_timeout(double s) { stream_->set_recv_timeout(s); }
  void shutdown_read() { stream_->shutdown_read(); }
  void close() { stream_->close(); }

 private:
  // make at least n bytes available in the buffer; false on clean EOF
  bool fill(std::size_t n);
  [[noreturn]] void poison(const char* why);
  std::size_t avail() const { return tail_ - head_; }
  const std::uint8_t* data() const { return buf_.data() + head_; }

  std::unique_ptr<Stream> stream_;
  std::vector<std::uint8_t> buf_;
  std::size_t head_ = 0, tail_ = 0;
  bool poisoned_ = false;
  std::uint64_t sent_ = 0, received_ = 0;
};

}  // namespace avec::net
