// Raw loopback TCP bandwidth (the host-ingest ceiling of the wire configs):
// N connections, each sends MB megabytes in 8 MB writes; prints the aggregate.
//   g++ -O2 -std=c++17 -pthread -o build/loopback_bw tools/loopback_bw.cpp && build/loopback_bw 8 2048
#include <arpa/inet.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <unistd.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 1;
  long mb = argc > 2 ? atol(argv[2]) : 2048;
  int ls = socket(AF_INET, SOCK_STREAM, 0);
  sockaddr_in a{}; a.sin_family = AF_INET; a.sin_addr.s_addr = htonl(INADDR_LOOPBACK); a.sin_port = 0;
  bind(ls, (sockaddr*)&a, sizeof a); listen(ls, 64);
  socklen_t l = sizeof a; getsockname(ls, (sockaddr*)&a, &l);
  std::vector<std::thread> th;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) {
    th.emplace_back([&] {
      int c = socket(AF_INET, SOCK_STREAM, 0); int one = 1; setsockopt(c, IPPROTO_TCP, TCP_NODELAY, &one, sizeof one);
      connect(c, (sockaddr*)&a, sizeof a);
      std::vector<char> buf(8 << 20, 1);
      long left = mb << 20;
      while (left > 0) { long w = write(c, buf.data(), std::min<long>(left, buf.size())); if (w <= 0) break; left -= w; }
      close(c);
    });
    int s = accept(ls, nullptr, nullptr);
    th.emplace_back([s] {
      std::vector<char> buf(64 << 20);
      while (read(s, buf.data(), buf.size()) > 0) {}
      close(s);
    });
  }
  for (auto& t : th) t.join();
  double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  printf("%d connections: %.2f GB/s aggregate (%.2f per connection)\n", n, n * mb / 1024.0 / sec, mb / 1024.0 / sec);
}
