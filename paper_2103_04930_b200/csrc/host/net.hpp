// Byte streams for the destination server: TCP (TCP_NODELAY, SO_RCVTIMEO) and
// an in-process duplex pipe. Reference: proj/include/accelfwd/transport.hpp.
//
// Unlike the reference Transport (which returns a freshly allocated, zeroed
// 256 KiB vector per read, transport.cpp:62-77), a Stream reads INTO a caller
// buffer, so the channel can land FrameData payloads directly in pinned
// staging memory and send ForwardResult payloads from it with one writev.
#pragma once

#include <sys/uio.h>

#include <atomic>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>

namespace avec::net {

// failure kinds the channel/server distinguish (reference ErrorCode subset)
struct NetError : std::runtime_error {
  enum Kind { disconnected, timeout, connect_failed, bind_failed } kind;
  NetError(Kind k, const std::string& m) : std::runtime_error(m), kind(k) {}
};

class Stream {
 public:
  virtual ~Stream() = default;
  // Reads 1..max bytes; returns 0 on orderly EOF. Throws NetError{timeout}.
  virtual std::size_t read_some(void* dst, std::size_t max) = 0;
  virtual void write_all(const iovec* iov, int n) = 0;
  void write_all(const void* p, std::size_t n) {
    iovec v{const_cast<void*>(p), n};
    write_all(&v, 1);
  }
  virtual void set_recv_timeout(double seconds) = 0;
  virtual void shutdown_read() = 0;  // unblocks readers; further reads see EOF
  virtual void close() = 0;
};

// "host:port"; throws NetError{connect_failed}
std::unique_ptr<Stream> connect_tcp(const std::string& endpoint, double timeout_s);

class TcpListener {
 public:
  TcpListener(const std::string& host, std::uint16_t port);  // throws NetError{bind_failed}
  ~TcpListener();
  TcpListener(const TcpListener&) = delete;
  TcpListener& operator=(const TcpListener&) = delete;
  std::uint16_t port() const { return port_; }
  std::unique_ptr<Stream> accept();  // nullptr once closed
  // wakes a blocked accept (from any thread); the descriptor itself is
  // released by the destructor, after the accepting thread is gone, so it
  // can never be reused under a concurrent accept
  void close();

 private:
  int fd_ = -1;  // set in the constructor, released in the destructor
  std::atomic<bool> closed_{false};
  std::uint16_t port_ = 0;
};

struct StreamPair {
  std::unique_ptr<Stream> first, second;
};
StreamPair make_pipe();

}  // namespace avec::net
