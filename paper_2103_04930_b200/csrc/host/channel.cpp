#include "channel.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>

namespace avec::net {

namespace {
constexpr std::size_t kReadAhead = 64 * 1024;  // small messages: one read, many frames
}

Channel::Channel(std::unique_ptr<Stream> stream) : stream_(std::move(stream)) {
  buf_.resize(kReadAhead);
}

void Channel::send(const wire::Message& m) {
  auto bytes = wire::encode(m);
  stream_->write_all(bytes.data(), bytes.size());
  sent_ += bytes.size();
}

void Channel::send_parts(const void* head, std::size_t head_len, const void* payload,
                         std::size_t payload_len) {
  iovec iov[2] = {{const_cast<void*>(head), head_len}, {const_cast<void*>(payload), payload_len}};
  stream_->write_all(iov, payload_len ? 2 : 1);
  sent_ += head_len + payload_len;
}

void Channel::poison(const char* why) {
  poisoned_ = true;
  head_ = tail_ = 0;
  throw ProtocolError(why);
}

bool Channel::fill(std::size_t n) {
  if (avail() >= n) return true;
  if (head_ > 0) {  // compact
    std::memmove(buf_.data(), buf_.data() + head_, avail());
    tail_ -= head_;
    head_ = 0;
  }
  if (buf_.size() < n) buf_.resize(std::max(n, buf_.size() * 2));
  while (avail() < n) {
    std::size_t got = stream_->read_some(buf_.data() + tail_, buf_.size() - tail_);
    if (got == 0) return false;
    tail_ += got;
    received_ += got;
  }
  return true;
}

wire::Message Channel::recv(FrameSink* sink) {
  using wire::DecodeStatus;
  if (poisoned_) throw ProtocolError("stream already poisoned");
  auto eof = [&]() -> wire::Message {
    poisoned_ = avail() > 0;  // EOF inside a frame
    throw NetError(NetError::disconnected, "peer closed the connection");
  };
  if (!fill(4)) eof();
  std::uint32_t len;
  std::memcpy(&len, data(), 4);
  if (len < 1 || len > wire::kMaxFrameLen) poison("malformed message payload");
  if (!fill(5)) eof();
  const std::uint8_t tag = data()[4];
  if (tag < std::uint8_t(wire::Tag::hello) || tag > std::uint8_t(wire::Tag::error))
    poison("unknown message tag");

  // streamed FrameData: header + count, then the floats straight into the sink
  if (sink && tag == std::uint8_t(wire::Tag::frame_data) && len >= 5) {
    if (!fill(9)) eof();
    std::uint32_t count;
    std::memcpy(&count, data() + 5, 4);
    if (count >= 1 && std::uint64_t(len) == 5 + 4 * std::uint64_t(count)) {
      if (float* dst = sink->frame_buffer(count)) {
        head_ += 9;
        const std::size_t want = 4 * std::size_t(count);
        const std::size_t have = std::min(avail(), want);
        std::memcpy(dst, data(), have);
        head_ += have;
        std::size_t done = have;
        auto* out = reinterpret_cast<std::uint8_t*>(dst);
        if (done) sink->frame_progress(done);
        while (done < want) {
          const std::size_t got = stream_->read_some(out + done, want - done);
          if (got == 0) {
            poisoned_ = true;
            throw NetError(NetError::disconnected, "peer closed the connection");
          }
          done += got;
          received_ += got;
          sink->frame_progress(done);
        }
        wire::FrameData fd;
        fd.elem_count = count;
        fd.streamed = dst;
        return fd;
      }
    }
    // inconsistent counts: buffer the whole frame and let the decoder reject it
  }

  // streamed ForwardResult (client side): preamble, then floats into the sink
  if (sink && tag == std::uint8_t(wire::Tag::forward_result) && len >= 13) {
    if (!fill(17)) eof();
    double compute_s;
    std::uint32_t count;
    std::memcpy(&compute_s, data() + 5, 8);
    std::memcpy(&count, data() + 13, 4);
    if (count >= 1 && std::uint64_t(len) == 13 + 4 * std::uint64_t(count) && std::isfinite(compute_s) &&
        compute_s >= 0) {
      if (float* dst = sink->result_buffer(count)) {
        head_ += 17;
        const std::size_t want = 4 * std::size_t(count);
        const std::size_t have = std::min(avail(), want);
        std::memcpy(dst, data(), have);
        head_ += have;
        std::size_t done = have;
        auto* out = reinterpret_cast<std::uint8_t*>(dst);
        while (done < want) {
          const std::size_t got = stream_->read_some(out + done, want - done);
          if (got == 0) {
            poisoned_ = true;
            throw NetError(NetError::disconnected, "peer closed the connection");
          }
          done += got;
          received_ += got;
        }
        wire::ForwardResult fr;
        fr.compute_s = compute_s;
        fr.elem_count = count;  // payload is in the sink; fr.data stays empty
        return fr;
      }
    }
  }

  if (!fill(wire::kHeaderBytes + std::size_t(len))) eof();
  auto r = wire::decode({data(), wire::kHeaderBytes + std::size_t(len)});
  if (r.status != DecodeStatus::ok)
    poison(r.status == DecodeStatus::unknown_tag ? "unknown message tag" : "malformed message payload");
  head_ += r.consumed;
  return std::move(*r.message);
}

}  // namespace avec::net
