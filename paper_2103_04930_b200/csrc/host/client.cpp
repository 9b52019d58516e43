#include "client.hpp"

#include <algorithm>
#include <chrono>

namespace avec::client {

using namespace wire;

Session Session::connect(const std::string& endpoint, double timeout_s) {
  Session s(net::connect_tcp(endpoint, timeout_s));
  s.handshake();
  return s;
}

Session::Session(std::unique_ptr<net::Stream> stream)
    : ch_(std::make_unique<net::Channel>(std::move(stream))) {}

namespace {
[[noreturn]] void remote(const ErrorMsg& e) {
  throw RemoteError(e.code, std::string("destination reported ") + wire_error_name(e.code) + ": " + e.message);
}
}  // namespace

void Session::handshake(std::uint32_t version) {
  ch_->send(Hello{version});
  Message m = ch_->recv();
  if (const auto* ack = std::get_if<HelloAck>(&m)) {
    if (ack->version != version) throw std::runtime_error("destination speaks another protocol version");
    return;
  }
  if (const auto* e = std::get_if<ErrorMsg>(&m)) remote(*e);
  throw std::runtime_error("unexpected handshake reply");
}

bool Session::ensure_model(const ModelDescriptor& model) {
  ch_->send(ModelCheck{model.digest});
  Message m = ch_->recv();
  if (const auto* e = std::get_if<ErrorMsg>(&m)) remote(*e);
  if (const auto* ack = std::get_if<ModelAck>(&m)) {
    if (ack->digest != model.digest) throw std::runtime_error("acknowledged digest differs");
    return true;
  }
  if (!std::get_if<ModelNeeded>(&m)) throw std::runtime_error("unexpected reply to ModelCheck");
  ModelUpload up;
  up.digest = model.digest;
  up.output_divisor = model.output_divisor;
  up.name = model.name;
  up.structure = model.structure;
  up.weights = model.weights;
  ch_->send(Message(std::move(up)));
  Message m2 = ch_->recv();
  if (const auto* e = std::get_if<ErrorMsg>(&m2)) remote(*e);
  const auto* ack = std::get_if<ModelAck>(&m2);
  if (!ack || ack->digest != model.digest) throw std::runtime_error("upload was not acknowledged");
  return false;
}

namespace {
// receive the ForwardResult floats straight into the caller's vector
struct VectorSink final : net::FrameSink {
  std::vector<float>& v;
  explicit VectorSink(std::vector<float>& out) : v(out) {}
  float* frame_buffer(std::uint32_t) override { return nullptr; }
  float* result_buffer(std::uint32_t elems) override {
    if (v.size() != elems) v.resize(elems);
    return v.data();
  }
};
}  // namespace

double Session::forward(const float* data, std::uint32_t elems, std::uint32_t width,
                        std::uint32_t height, std::vector<float>& out) {
  return forward_timed(data, elems, width, height, out).compute_s;
}

record::CycleTiming Session::forward_timed(const float* data, std::uint32_t elems, std::uint32_t width,
                                           std::uint32_t height, std::vector<float>& out) {
  using clk = std::chrono::steady_clock;
  const std::uint64_t sent0 = ch_->bytes_sent(), recv0 = ch_->bytes_received();
  const auto t0 = clk::now();
  const auto head = frame_data_header(elems);
  ch_->send_parts(head.data(), head.size(), data, std::size_t(elems) * 4);
  ch_->send(Resolution{width, height});
  ch_->send(FrameSize{elems});
  const auto sent_at = clk::now();
  VectorSink sink(out);
  Message m = ch_->recv(&sink);
  if (const auto* e = std::get_if<ErrorMsg>(&m)) remote(*e);
  auto* fr = std::get_if<ForwardResult>(&m);
  if (!fr) throw std::runtime_error("expected ForwardResult");
  if (!fr->data.empty()) out = std::move(fr->data);  // not streamed (small replies)
  const auto recv_at = clk::now();
  const double send_s = std::chrono::duration<double>(sent_at - t0).count();
  const double wait_s = std::chrono::duration<double>(recv_at - sent_at).count();
  record::CycleTiming t;
  t.compute_s = fr->compute_s;
  // the destination may start computing before sent_at is stamped: clamp so
  // gpu + communication never exceeds the cycle
  t.gpu_s = std::min(fr->compute_s, wait_s);
  t.communication_s = send_s + (wait_s - t.gpu_s);
  t.other_s = std::max(0.0, std::chrono::duration<double>(clk::now() - t0).count() - t.communication_s - t.gpu_s);
  t.bytes_sent = ch_->bytes_sent() - sent0;
  t.bytes_received = ch_->bytes_received() - recv0;
  return t;
}

}  // namespace avec::client
