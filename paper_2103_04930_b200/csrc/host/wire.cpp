// Wire codec. Behaviour (lengths, validation, poison rules) matches the
// reference codec proj/src/wire.cpp; the implementation is our own.
#include "wire.hpp"

#include <openssl/evp.h>

#include <bit>
#include <cmath>
#include <cstring>
#include <stdexcept>

static_assert(std::endian::native == std::endian::little, "little-endian host required");

namespace avec::wire {

std::uint64_t output_elems(std::uint64_t input_elems, double divisor) {
  if (!(divisor > 0.0)) throw std::invalid_argument("output divisor must be > 0");
  return static_cast<std::uint64_t>(std::llround(static_cast<double>(input_elems) / divisor));
}

std::uint64_t transfer_size(const Dims& dims, double divisor) {
  const std::uint64_t e = dims.elem_count();
  return 12 + 4 * e + 4 * output_elems(e, divisor);
}

namespace {
struct EvpCtx {
  EVP_MD_CTX* c = EVP_MD_CTX_new();
  ~EvpCtx() { EVP_MD_CTX_free(c); }
};
}  // namespace

static Digest sha256_parts(std::initializer_list<std::span<const std::uint8_t>> parts) {
  EvpCtx ctx;
  Digest d{};
  unsigned n = 0;
  if (!ctx.c || EVP_DigestInit_ex(ctx.c, EVP_sha256(), nullptr) != 1)
    throw std::runtime_error("sha256 init failed");
  for (auto p : parts)
    if (EVP_DigestUpdate(ctx.c, p.data(), p.size()) != 1) throw std::runtime_error("sha256 update failed");
  if (EVP_DigestFinal_ex(ctx.c, d.data(), &n) != 1 || n != 32) throw std::runtime_error("sha256 final failed");
  return d;
}

Digest sha256(std::span<const std::uint8_t> data) { return sha256_parts({data}); }

std::string hex(const Digest& d) {
  static constexpr char k[] = "0123456789abcdef";
  std::string s(64, '0');
  for (int i = 0; i < 32; ++i) {
    s[2 * i] = k[d[i] >> 4];
    s[2 * i + 1] = k[d[i] & 15];
  }
  return s;
}

Digest model_digest(std::span<const std::uint8_t> structure, std::span<const std::uint8_t> weights,
                    double output_divisor) {
  std::uint8_t c[8];
  std::memcpy(c, &output_divisor, 8);
  return sha256_parts({structure, weights, std::span<const std::uint8_t>(c, 8)});
}

ModelDescriptor make_model(std::string name, std::vector<std::uint8_t> structure,
                           std::vector<std::uint8_t> weights, double output_divisor) {
  if (!(output_divisor > 0.0)) throw std::invalid_argument("output divisor must be > 0");
  ModelDescriptor m;
  m.digest = model_digest(structure, weights, output_divisor);
  m.name = std::move(name);
  m.structure = std::move(structure);
  m.weights = std::move(weights);
  m.output_divisor = output_divisor;
  return m;
}

// ------------------------------------------------------------------ encode
namespace {

class Builder {
 public:
  explicit Builder(Tag tag, std::uint64_t payload) {
    const std::uint64_t len = 1 + payload;
    if (len > kMaxFrameLen) throw std::length_error("encoded frame would exceed 2^31-1 bytes");
    out.reserve(kHeaderBytes + len);
    put32(static_cast<std::uint32_t>(len));
    out.push_back(static_cast<std::uint8_t>(tag));
  }
  void put32(std::uint32_t v) { raw(&v, 4); }
  void put64(std::uint64_t v) { raw(&v, 8); }
  void putf64(double v) { raw(&v, 8); }
  void bytes(const void* p, std::size_t n) { raw(p, n); }
  void raw(const void* p, std::size_t n) {
    const auto* b = static_cast<const std::uint8_t*>(p);
    out.insert(out.end(), b, b + n);
  }
  std::vector<std::uint8_t> out;
};

}  // namespace

std::vector<std::uint8_t> encode(const Message& m) {
  return std::visit(
      [](const auto& v) -> std::vector<std::uint8_t> {
        using T = std::decay_t<decltype(v)>;
        if constexpr (std::is_same_v<T, Hello> || std::is_same_v<T, HelloAck>) {
          Builder b(std::is_same_v<T, Hello> ? Tag::hello : Tag::hello_ack, 4);
          b.put32(v.version);
          return std::move(b.out);
        } else if constexpr (std::is_same_v<T, FrameSize>) {
          if (v.elem_count < 1) throw std::invalid_argument("FrameSize is zero");
          Builder b(Tag::frame_size, 4);
          b.put32(v.elem_count);
          return std::move(b.out);
        } else if constexpr (std::is_same_v<T, Resolution>) {
          if (v.width < 1 || v.height < 1 || v.width > kMaxSide || v.height > kMaxSide)
            throw std::invalid_argument("Resolution out of range");
          Builder b(Tag::resolution, 8);
          b.put32(v.width);
          b.put32(v.height);
          return std::move(b.out);
        } else if constexpr (std::is_same_v<T, FrameData>) {
          if (!v.streamed && v.data.size() != v.elem_count)
            throw std::invalid_argument("FrameData element count mismatch");
          if (v.elem_count < 1) throw std::invalid_argument("FrameData is empty");
          Builder b(Tag::frame_data, 4 + 4 * std::uint64_t(v.elem_count));
          b.put32(v.elem_count);
          b.bytes(v.floats(), 4 * std::size_t(v.elem_count));
          return std::move(b.out);
        } else if constexpr (std::is_same_v<T, ForwardResult>) {
          if (v.data.size() != v.elem_count)
            throw std::invalid_argument("ForwardResult element count mismatch");
          if (v.elem_count < 1) throw std::invalid_argument("ForwardResult is empty");
          if (!std::isfinite(v.compute_s) || v.compute_s < 0)
            throw std::invalid_argument("ForwardResult compute seconds invalid");
          Builder b(Tag::forward_result, 12 + 4 * std::uint64_t(v.elem_count));
          b.putf64(v.compute_s);
          b.put32(v.elem_count);
          b.bytes(v.data.data(), 4 * v.data.size());
          return std::move(b.out);
        } else if constexpr (std::is_same_v<T, ModelCheck> || std::is_same_v<T, ModelNeeded> ||
                             std::is_same_v<T, ModelAck>) {
          Tag t = std::is_same_v<T, ModelCheck> ? Tag::model_check
                  : std::is_same_v<T, ModelNeeded> ? Tag::model_needed : Tag::model_ack;
          Builder b(t, 32);
          b.bytes(v.digest.data(), 32);
          return std::move(b.out);
        } else if constexpr (std::is_same_v<T, ModelUpload>) {
          if (!(v.output_divisor > 0.0) || !std::isfinite(v.output_divisor))
            throw std::invalid_argument("ModelUpload divisor invalid");
          Builder b(Tag::model_upload, 32 + 8 + 4 + v.name.size() + 4 + v.structure.size() + 8 +
                                           v.weights.size());
          b.bytes(v.digest.data(), 32);
          b.putf64(v.output_divisor);
          b.put32(static_cast<std::uint32_t>(v.name.size()));
          b.bytes(v.name.data(), v.name.size());
          b.put32(static_cast<std::uint32_t>(v.structure.size()));
          b.bytes(v.structure.data(), v.structure.size());
          b.put64(v.weights.size());
          b.bytes(v.weights.data(), v.weights.size());
          return std::move(b.out);
        } else {
          static_assert(std::is_same_v<T, ErrorMsg>);
          Builder b(Tag::error, 8 + v.message.size());
          b.put32(v.code);
          b.put32(static_cast<std::uint32_t>(v.message.size()));
          b.bytes(v.message.data(), v.message.size());
          return std::move(b.out);
        }
      },
      m);
}

std::array<std::uint8_t, 17> forward_result_header(double compute_s, std::uint32_t k) {
  if (k < 1) throw std::invalid_argument("ForwardResult is empty");
  if (!std::isfinite(compute_s) || compute_s < 0)
    throw std::invalid_argument("ForwardResult compute seconds invalid");
  std::array<std::uint8_t, 17> h{};
  const std::uint64_t len = 1 + 8 + 4 + 4 * std::uint64_t(k);
  if (len > kMaxFrameLen) throw std::length_error("encoded frame would exceed 2^31-1 bytes");
  const std::uint32_t l32 = static_cast<std::uint32_t>(len);
  std::memcpy(h.data(), &l32, 4);
  h[4] = static_cast<std::uint8_t>(Tag::forward_result);
  std::memcpy(h.data() + 5, &compute_s, 8);
  std::memcpy(h.data() + 13, &k, 4);
  return h;
}

std::array<std::uint8_t, 9> frame_data_header(std::uint32_t k) {
  if (k < 1) throw std::invalid_argument("FrameData is empty");
  std::array<std::uint8_t, 9> h{};
  const std::uint64_t len = 1 + 4 + 4 * std::uint64_t(k);
  if (len > kMaxFrameLen) throw std::length_error("encoded frame would exceed 2^31-1 bytes");
  const std::uint32_t l32 = static_cast<std::uint32_t>(len);
  std::memcpy(h.data(), &l32, 4);
  h[4] = static_cast<std::uint8_t>(Tag::frame_data);
  std::memcpy(h.data() + 5, &k, 4);
  return h;
}

// ------------------------------------------------------------------ decode
namespace {

struct Cursor {
  const std::uint8_t* p;
  std::size_t left;
  template <class T>
  bool get(T& v) {
    if (left < sizeof(T)) return false;
    std::memcpy(&v, p, sizeof(T));
    p += sizeof(T);
    left -= sizeof(T);
    return true;
  }
  bool take(std::size_t n, const std::uint8_t*& out) {
    if (left < n) return false;
    out = p;
    p += n;
    left -= n;
    return true;
  }
  bool done() const { return left == 0; }
};

DecodeResult bad() { return {DecodeStatus::malformed_payload, std::nullopt, 0}; }

std::optional<Message> parse_payload(Tag tag, Cursor c) {
  const std::uint8_t* raw = nullptr;
  switch (tag) {
    case Tag::hello:
    case Tag::hello_ack: {
      std::uint32_t v;
      if (!c.get(v) || !c.done()) return std::nullopt;
      if (tag == Tag::hello) return Message(Hello{v});
      return Message(HelloAck{v});
    }
    case Tag::frame_size: {
      FrameSize v;
      if (!c.get(v.elem_count) || !c.done() || v.elem_count < 1) return std::nullopt;
      return Message(v);
    }
    case Tag::resolution: {
      Resolution v;
      if (!c.get(v.width) || !c.get(v.height) || !c.done()) return std::nullopt;
      if (v.width < 1 || v.height < 1 || v.width > kMaxSide || v.height > kMaxSide) return std::nullopt;
      return Message(v);
    }
    case Tag::frame_data: {
      FrameData v;
      if (!c.get(v.elem_count) || v.elem_count < 1) return std::nullopt;
      if (!c.take(4 * std::size_t(v.elem_count), raw) || !c.done()) return std::nullopt;
      v.data.resize(v.elem_count);
      std::memcpy(v.data.data(), raw, 4 * std::size_t(v.elem_count));
      return Message(std::move(v));
    }
    case Tag::forward_result: {
      ForwardResult v;
      if (!c.get(v.compute_s) || !c.get(v.elem_count)) return std::nullopt;
      if (!std::isfinite(v.compute_s) || v.compute_s < 0 || v.elem_count < 1) return std::nullopt;
      if (!c.take(4 * std::size_t(v.elem_count), raw) || !c.done()) return std::nullopt;
      v.data.resize(v.elem_count);
      std::memcpy(v.data.data(), raw, 4 * std::size_t(v.elem_count));
      return Message(std::move(v));
    }
    case Tag::model_check:
    case Tag::model_needed:
    case Tag::model_ack: {
      Digest d;
      if (!c.take(32, raw) || !c.done()) return std::nullopt;
      std::memcpy(d.data(), raw, 32);
      if (tag == Tag::model_check) return Message(ModelCheck{d});
      if (tag == Tag::model_needed) return Message(ModelNeeded{d});
      return Message(ModelAck{d});
    }
    case Tag::model_upload: {
      ModelUpload v;
      std::uint32_t nl = 0, sl = 0;
      std::uint64_t wl = 0;
      if (!c.take(32, raw)) return std::nullopt;
      std::memcpy(v.digest.data(), raw, 32);
      if (!c.get(v.output_divisor) || !std::isfinite(v.output_divisor) || !(v.output_divisor > 0.0))
        return std::nullopt;
      if (!c.get(nl) || !c.take(nl, raw)) return std::nullopt;
      v.name.assign(reinterpret_cast<const char*>(raw), nl);
      if (!c.get(sl) || !c.take(sl, raw)) return std::nullopt;
      v.structure.assign(raw, raw + sl);
      if (!c.get(wl) || wl > c.left || !c.take(std::size_t(wl), raw) || !c.done()) return std::nullopt;
      v.weights.assign(raw, raw + wl);
      return Message(std::move(v));
    }
    case Tag::error: {
      ErrorMsg v;
      std::uint32_t ml = 0;
      if (!c.get(v.code) || !c.get(ml) || !c.take(ml, raw) || !c.done()) return std::nullopt;
      v.message.assign(reinterpret_cast<const char*>(raw), ml);
      return Message(std::move(v));
    }
  }
  return std::nullopt;
}

}  // namespace

DecodeResult decode(std::span<const std::uint8_t> buf) {
  if (buf.size() < kHeaderBytes) return {};
  std::uint32_t len;
  std::memcpy(&len, buf.data(), 4);
  if (len < 1 || len > kMaxFrameLen) return bad();
  if (buf.size() < kHeaderBytes + 1) return {};
  const std::uint8_t tag = buf[4];
  if (tag < std::uint8_t(Tag::hello) || tag > std::uint8_t(Tag::error))
    return {DecodeStatus::unknown_tag, std::nullopt, 0};
  if (buf.size() < kHeaderBytes + len) return {};
  auto m = parse_payload(static_cast<Tag>(tag), Cursor{buf.data() + 5, std::size_t(len) - 1});
  if (!m) return bad();
  return {DecodeStatus::ok, std::move(m), kHeaderBytes + len};
}

Tag tag_of(const Message& m) {
  static constexpr Tag order[] = {Tag::hello,       Tag::hello_ack,   Tag::frame_size,
                                  Tag::resolution,  Tag::frame_data,  Tag::forward_result,
                                  Tag::model_check, Tag::model_needed, Tag::model_upload,
                                  Tag::model_ack,   Tag::error};
  return order[m.index()];
}

const char* tag_name(Tag t) noexcept {
  static constexpr const char* names[] = {"Hello",       "HelloAck",    "FrameSize", "Resolution",
                                          "FrameData",   "ForwardResult", "ModelCheck",
                                          "ModelNeeded", "ModelUpload", "ModelAck",  "Error"};
  const unsigned i = unsigned(t) - 1;
  return i < 11 ? names[i] : "?";
}

const char* wire_error_name(std::uint32_t code) noexcept {
  static constexpr const char* names[] = {"protocol",      "busy",          "too_large", "version",
                                          "unknown_model", "invalid_model", "internal"};
  return code >= 1 && code <= 7 ? names[code - 1] : "?";
}

}  // namespace avec::wire
