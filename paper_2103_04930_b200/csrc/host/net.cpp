#include "net.hpp"

#include <arpa/inet.h>
#include <fcntl.h>
#include <netdb.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <poll.h>
#include <sys/socket.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <vector>

namespace avec::net {

namespace {

[[noreturn]] void sys_fail(NetError::Kind k, const std::string& what) {
  throw NetError(k, what + ": " + std::strerror(errno));
}

class TcpStream final : public Stream {
 public:
  explicit TcpStream(int fd) : fd_(fd) {
    int one = 1;
    setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof one);
    // frames are tens of MB. An explicit SO_RCVBUF/SO_SNDBUF turns off the
    // kernel's buffer autotuning and is capped at net.core.[rw]mem_max, so it
    // is only set when asked for (AVEC_SOCKBUF=<bytes>)
    static const int buf = [] {
      const char* e = std::getenv("AVEC_SOCKBUF");
      return e ? std::atoi(e) : 0;
    }();
    if (buf > 0) {
      setsockopt(fd, SOL_SOCKET, SO_RCVBUF, &buf, sizeof buf);
      setsockopt(fd, SOL_SOCKET, SO_SNDBUF, &buf, sizeof buf);
    }
  }
  ~TcpStream() override { close(); }

  std::size_t read_some(void* dst, std::size_t max) override {
    for (;;) {
      const int fd = fd_.load();
      if (fd < 0) return 0;
      const ssize_t n = ::recv(fd, dst, max, 0);
      if (n >= 0) return std::size_t(n);
      if (errno == EINTR) continue;
      if (errno == EAGAIN || errno == EWOULDBLOCK) throw NetError(NetError::timeout, "recv timed out");
      if (errno == ECONNRESET || errno == EBADF) return 0;
      sys_fail(NetError::disconnected, "recv");
    }
  }

  void write_all(const iovec* iov_in, int n) override {
    std::vector<iovec> iov(iov_in, iov_in + n);
    std::size_t i = 0;
    while (i < iov.size()) {
      msghdr msg{};
      msg.msg_iov = iov.data() + i;
      msg.msg_iovlen = iov.size() - i;
      const int fd = fd_.load();
      if (fd < 0) throw NetError(NetError::disconnected, "send on closed socket");
      ssize_t w = ::sendmsg(fd, &msg, MSG_NOSIGNAL);
      if (w < 0) {
        if (errno == EINTR) continue;
        sys_fail(NetError::disconnected, "send");
      }
      std::size_t left = std::size_t(w);
      while (i < iov.size() && left >= iov[i].iov_len) left -= iov[i++].iov_len;
      if (i < iov.size()) {
        iov[i].iov_base = static_cast<char*>(iov[i].iov_base) + left;
        iov[i].iov_len -= left;
      }
    }
  }

  void set_recv_timeout(double s) override {
    timeval tv{};
    if (s > 0) {
      tv.tv_sec = time_t(s);
      tv.tv_usec = suseconds_t((s - double(tv.tv_sec)) * 1e6);
    }
    setsockopt(fd_.load(), SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof tv);
  }
  void shutdown_read() override { ::shutdown(fd_.load(), SHUT_RD); }
  void close() override {
    int fd = fd_.exchange(-1);
    if (fd >= 0) ::close(fd);
  }

 private:
  std::atomic<int> fd_;
};

sockaddr_in resolve(const std::string& host, std::uint16_t port, NetError::Kind k) {
  sockaddr_in a{};
  a.sin_family = AF_INET;
  a.sin_port = htons(port);
  if (inet_pton(AF_INET, host.c_str(), &a.sin_addr) == 1) return a;
  addrinfo hints{}, *res = nullptr;
  hints.ai_family = AF_INET;
  hints.ai_socktype = SOCK_STREAM;
  if (getaddrinfo(host.c_str(), nullptr, &hints, &res) != 0 || !res)
    throw NetError(k, "cannot resolve host " + host);
  a.sin_addr = reinterpret_cast<sockaddr_in*>(res->ai_addr)->sin_addr;
  freeaddrinfo(res);
  return a;
}

// ---- in-process pipe: one byte queue per direction ----
struct ByteQueue {
  std::mutex m;
  std::condition_variable cv;
  std::deque<std::vector<std::uint8_t>> chunks;
  std::size_t head = 0;  // consumed bytes of chunks.front()
  bool writer_closed = false, reader_closed = false;
};

class PipeStream final : public Stream {
 public:
  PipeStream(std::shared_ptr<ByteQueue> rx, std::shared_ptr<ByteQueue> tx)
      : rx_(std::move(rx)), tx_(std::move(tx)) {}
  ~PipeStream() override { close(); }

  std::size_t read_some(void* dst, std::size_t max) override {
    std::unique_lock<std::mutex> lk(rx_->m);
    auto ready = [&] { return !rx_->chunks.empty() || rx_->writer_closed || rx_->reader_closed; };
    if (timeout_ > 0) {
      if (!rx_->cv.wait_for(lk, std::chrono::duration<double>(timeout_), ready))
        throw NetError(NetError::timeout, "recv timed out");
    } else {
      rx_->cv.wait(lk, ready);
    }
    if (rx_->reader_closed || rx_->chunks.empty()) return 0;
    auto& front = rx_->chunks.front();
    const std::size_t n = std::min(max, front.size() - rx_->head);
    std::memcpy(dst, front.data() + rx_->head, n);
    rx_->head += n;
    if (rx_->head == front.size()) {
      rx_->chunks.pop_front();
      rx_->head = 0;
    }
    return n;
  }

  void write_all(const iovec* iov, int n) override {
    std::size_t total = 0;
    for (int i = 0; i < n; ++i) total += iov[i].iov_len;
    if (!total) return;
    std::vector<std::uint8_t> chunk(total);
    std::size_t off = 0;
    for (int i = 0; i < n; ++i) {
      std::memcpy(chunk.data() + off, iov[i].iov_base, iov[i].iov_len);
      off += iov[i].iov_len;
    }
    std::lock_guard<std::mutex> lk(tx_->m);
    if (tx_->writer_closed || tx_->reader_closed) throw NetError(NetError::disconnected, "pipe closed");
    tx_->chunks.push_back(std::move(chunk));
    tx_->cv.notify_all();
  }

  void set_recv_timeout(double s) override { timeout_ = s; }
  void shutdown_read() override {
    std::lock_guard<std::mutex> lk(rx_->m);
    rx_->reader_closed = true;
    rx_->cv.notify_all();
  }
  void close() override {
    {
      std::lock_guard<std::mutex> lk(tx_->m);
      tx_->writer_closed = true;
      tx_->cv.notify_all();
    }
    shutdown_read();
  }

 private:
  std::shared_ptr<ByteQueue> rx_, tx_;
  double timeout_ = 0;
};

}  // namespace

std::unique_ptr<Stream> connect_tcp(const std::string& endpoint, double timeout_s) {
  const auto colon = endpoint.rfind(':');
  if (colon == std::string::npos || colon + 1 == endpoint.size())
    throw NetError(NetError::connect_failed, "endpoint must be host:port, got " + endpoint);
  int port = -1;
  try {
    port = std::stoi(endpoint.substr(colon + 1));
  } catch (...) {
  }
  if (port < 1 || port > 65535) throw NetError(NetError::connect_failed, "bad port in " + endpoint);
  sockaddr_in a = resolve(endpoint.substr(0, colon), std::uint16_t(port), NetError::connect_failed);
  const int fd = ::socket(AF_INET, SOCK_STREAM, 0);
  if (fd < 0) sys_fail(NetError::connect_failed, "socket");
  const int flags = fcntl(fd, F_GETFL, 0);
  fcntl(fd, F_SETFL, flags | O_NONBLOCK);
  int rc = ::connect(fd, reinterpret_cast<sockaddr*>(&a), sizeof a);
  if (rc != 0 && errno != EINPROGRESS) {
    ::close(fd);
    sys_fail(NetError::connect_failed, "connect to " + endpoint);
  }
  if (rc != 0) {
    pollfd p{fd, POLLOUT, 0};
    const int pr = ::poll(&p, 1, timeout_s > 0 ? int(timeout_s * 1000) : -1);
    int err = 0;
    socklen_t len = sizeof err;
    if (pr > 0) getsockopt(fd, SOL_SOCKET, SO_ERROR, &err, &len);
    if (pr <= 0 || err) {
      ::close(fd);
      throw NetError(NetError::connect_failed,
                     "connect to " + endpoint + (pr == 0 ? " timed out" : " failed"));
    }
  }
  fcntl(fd, F_SETFL, flags);
  return std::make_unique<TcpStream>(fd);
}

TcpListener::TcpListener(const std::string& host, std::uint16_t port) {
  sockaddr_in a = resolve(host, port, NetError::bind_failed);
  fd_ = ::socket(AF_INET, SOCK_STREAM, 0);
  if (fd_ < 0) sys_fail(NetError::bind_failed, "socket");
  int one = 1;
  setsockopt(fd_, SOL_SOCKET, SO_REUSEADDR, &one, sizeof one);
  if (::bind(fd_, reinterpret_cast<sockaddr*>(&a), sizeof a) != 0 || ::listen(fd_, 64) != 0) {
    const int e = errno;
    ::close(fd_);
    fd_ = -1;
    errno = e;
    sys_fail(NetError::bind_failed, "bind/listen " + host);
  }
  sockaddr_in b{};
  socklen_t len = sizeof b;
  getsockname(fd_, reinterpret_cast<sockaddr*>(&b), &len);
  port_ = ntohs(b.sin_port);
}

TcpListener::~TcpListener() {
  close();
  if (fd_ >= 0) ::close(fd_);
  fd_ = -1;
}

std::unique_ptr<Stream> TcpListener::accept() {
  for (;;) {
    if (closed_.load()) return nullptr;
    const int c = ::accept(fd_, nullptr, nullptr);
    if (c >= 0) {
      if (closed_.load()) {
        ::close(c);
        return nullptr;
      }
      return std::make_unique<TcpStream>(c);
    }
    if (errno == EINTR) continue;
    return nullptr;
  }
}

void TcpListener::close() {
  if (!closed_.exchange(true) && fd_ >= 0) ::shutdown(fd_, SHUT_RDWR);  // wakes accept()
}

StreamPair make_pipe() {
  auto a = std::make_shared<ByteQueue>(), b = std::make_shared<ByteQueue>();
  return {std::make_unique<PipeStream>(a, b), std::make_unique<PipeStream>(b, a)};
}

}  // namespace avec::net
