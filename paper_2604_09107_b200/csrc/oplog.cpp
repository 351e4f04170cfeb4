// Sequenced operation log for the multi-process registry.
//
// The reference runs one metadata server that clients dial at any time
// (StreamServerHost / StreamControl, transport_stream.cpp:582-797).  Here
// every process keeps a replica of the registry (csrc/registry.cpp) and the
// replicas stay identical by applying one totally ordered log of registry
// operations (a replicated state machine).  The log server assigns the
// order: a process appends its operation and learns its sequence number; every
// process tails the log and applies entries in sequence order.  A process
// that starts late fetches the log from entry 0 and replays it, so it joins
// with exactly the registry state the others have -- including replicas that
// are still filling, which it may then be planned onto and chase.
//
// Wire (little-endian, one TCP connection per client, requests serialised):
//   request  := magic u32 ("RSLG") | kind u8 | ...
//     APPEND (1): len u64 | bytes            -> seq u64
//     FETCH  (2): from u64 | wait_ms u32 | max u32
//                 -> count u64 | count x (len u64 | bytes)
//   FETCH long-polls up to wait_ms for an entry at or after `from`.
#include <arpa/inet.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ros_b200.h"
#include "common.hpp"

namespace {

constexpr std::uint32_t kLogMagic = 0x474C5352;  // "RSLG"
constexpr std::uint64_t kMaxEntry = 256ull << 20;

bool send_all(int fd, const void* p, std::size_t n) {
  const auto* b = static_cast<const std::uint8_t*>(p);
  while (n) {
    const ssize_t k = ::send(fd, b, n, MSG_NOSIGNAL);
    if (k <= 0) return false;
    b += k;
    n -= static_cast<std::size_t>(k);
  }
  return true;
}

bool recv_all(int fd, void* p, std::size_t n) {
  auto* b = static_cast<std::uint8_t*>(p);
  while (n) {
    const ssize_t k = ::recv(fd, b, n, 0);
    if (k <= 0) return false;
    b += k;
    n -= static_cast<std::size_t>(k);
  }
  return true;
}

template <class T>
bool send_pod(int fd, const T& v) {
  return send_all(fd, &v, sizeof(v));
}
template <class T>
bool recv_pod(int fd, T* v) {
  return recv_all(fd, v, sizeof(T));
}

int st(rsb::Status s) { return static_cast<int>(s); }

}  // namespace

struct rs_oplog_server {
  std::mutex m;
  std::condition_variable cv;
  std::vector<std::string> log;
  int lfd = -1;
  int port = 0;
  std::atomic<bool> stop{false};
  std::thread acceptor;
  std::mutex conns_m;
  std::vector<std::thread> conns;
  std::vector<int> fds;

  void serve(int fd) {
    for (;;) {
      std::uint32_t magic = 0;
      std::uint8_t kind = 0;
      if (!recv_pod(fd, &magic) || magic != kLogMagic || !recv_pod(fd, &kind)) break;
      if (kind == 1) {
        std::uint64_t len = 0;
        if (!recv_pod(fd, &len) || len > kMaxEntry) break;
        std::string e(len, '\0');
        if (len && !recv_all(fd, e.data(), len)) break;
        std::uint64_t seq;
        {
          std::lock_guard lk(m);
          seq = log.size();
          log.push_back(std::move(e));
        }
        cv.notify_all();
        if (!send_pod(fd, seq)) break;
      } else if (kind == 2) {
        std::uint64_t from = 0;
        std::uint32_t wait_ms = 0, max = 0;
        if (!recv_pod(fd, &from) || !recv_pod(fd, &wait_ms) || !recv_pod(fd, &max)) break;
        std::vector<std::string> out;
        {
          std::unique_lock lk(m);
          cv.wait_for(lk, std::chrono::milliseconds(wait_ms), [&] { return stop.load() || log.size() > from; });
          for (std::uint64_t i = from; i < log.size() && out.size() < max; ++i) out.push_back(log[i]);
        }
        std::uint64_t n = out.size();
        bool good = send_pod(fd, n);
        for (const auto& e : out) {
          const std::uint64_t len = e.size();
          good = good && send_pod(fd, len) && send_all(fd, e.data(), e.size());
        }
        if (!good) break;
      } else {
        break;
      }
    }
    ::close(fd);
  }
};

struct rs_oplog {
  int fd = -1;
  std::vector<std::string> last;  // entries of the latest fetch
};

extern "C" {

int rs_oplog_serve(const char* host, int port, int* bound_port, rs_oplog_server** out) {
  if (!host || !out) return st(rsb::Status::invalid_argument);
  auto* s = new rs_oplog_server();
  s->lfd = ::socket(AF_INET, SOCK_STREAM, 0);
  int one = 1;
  setsockopt(s->lfd, SOL_SOCKET, SO_REUSEADDR, &one, sizeof(one));
  sockaddr_in a{};
  a.sin_family = AF_INET;
  a.sin_port = htons(static_cast<std::uint16_t>(port));
  if (inet_pton(AF_INET, host, &a.sin_addr) != 1 ||
      ::bind(s->lfd, reinterpret_cast<sockaddr*>(&a), sizeof(a)) != 0 || ::listen(s->lfd, 64) != 0) {
    ::close(s->lfd);
    delete s;
    return st(rsb::Status::server_unavailable);
  }
  socklen_t al = sizeof(a);
  getsockname(s->lfd, reinterpret_cast<sockaddr*>(&a), &al);
  s->port = ntohs(a.sin_port);
  s->acceptor = std::thread([s] {
    while (!s->stop) {
      const int fd = ::accept(s->lfd, nullptr, nullptr);
      if (fd < 0) {
        if (s->stop) return;
        continue;
      }
      int one = 1;
      setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
      std::lock_guard lk(s->conns_m);
      s->fds.push_back(fd);
      s->conns.emplace_back([s, fd] { s->serve(fd); });
    }
  });
  if (bound_port) *bound_port = s->port;
  *out = s;
  return 0;
}

void rs_oplog_server_stop(rs_oplog_server* s) {
  if (!s) return;
  s->stop = true;
  s->cv.notify_all();
  ::shutdown(s->lfd, SHUT_RDWR);
  ::close(s->lfd);
  if (s->acceptor.joinable()) s->acceptor.join();
  {
    std::lock_guard lk(s->conns_m);
    for (int fd : s->fds) ::shutdown(fd, SHUT_RDWR);
  }
  for (auto& t : s->conns)
    if (t.joinable()) t.join();
  delete s;
}

uint64_t rs_oplog_server_size(rs_oplog_server* s) {
  if (!s) return 0;
  std::lock_guard lk(s->m);
  return s->log.size();
}

int rs_oplog_connect(const char* host, int port, double timeout_s, rs_oplog** out) {
  if (!host || !out) return st(rsb::Status::invalid_argument);
  sockaddr_in a{};
  a.sin_family = AF_INET;
  a.sin_port = htons(static_cast<std::uint16_t>(port));
  if (inet_pton(AF_INET, host, &a.sin_addr) != 1) return st(rsb::Status::invalid_argument);
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(timeout_s);
  for (;;) {
    const int fd = ::socket(AF_INET, SOCK_STREAM, 0);
    if (fd >= 0 && ::connect(fd, reinterpret_cast<sockaddr*>(&a), sizeof(a)) == 0) {
      int one = 1;
      setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
      auto* l = new rs_oplog();
      l->fd = fd;
      *out = l;
      return 0;
    }
    if (fd >= 0) ::close(fd);
    if (std::chrono::steady_clock::now() > deadline) return st(rsb::Status::server_unavailable);
    std::this_thread::sleep_for(std::chrono::milliseconds(10));
  }
}

int rs_oplog_append(rs_oplog* l, const void* entry, size_t len, uint64_t* seq) {
  if (!l || (len && !entry) || !seq || len > kMaxEntry) return st(rsb::Status::invalid_argument);
  const std::uint8_t kind = 1;
  const std::uint64_t n = len;
  if (!send_pod(l->fd, kLogMagic) || !send_pod(l->fd, kind) || !send_pod(l->fd, n) ||
      !send_all(l->fd, entry, len) || !recv_pod(l->fd, seq))
    return st(rsb::Status::server_unavailable);
  return 0;
}

int rs_oplog_fetch(rs_oplog* l, uint64_t from, int wait_ms, uint32_t max_entries, uint64_t* count) {
  if (!l || !count) return st(rsb::Status::invalid_argument);
  const std::uint8_t kind = 2;
  const auto w = static_cast<std::uint32_t>(wait_ms < 0 ? 0 : wait_ms);
  std::uint64_t n = 0;
  if (!send_pod(l->fd, kLogMagic) || !send_pod(l->fd, kind) || !send_pod(l->fd, from) || !send_pod(l->fd, w) ||
      !send_pod(l->fd, max_entries) || !recv_pod(l->fd, &n) || n > max_entries)
    return st(rsb::Status::server_unavailable);
  l->last.assign(n, std::string());
  for (auto& e : l->last) {
    std::uint64_t len = 0;
    if (!recv_pod(l->fd, &len) || len > kMaxEntry) return st(rsb::Status::protocol_error);
    e.resize(len);
    if (len && !recv_all(l->fd, e.data(), len)) return st(rsb::Status::server_unavailable);
  }
  *count = n;
  return 0;
}

int rs_oplog_entry(rs_oplog* l, uint64_t i, const void** data, size_t* len) {
  if (!l || !data || !len || i >= l->last.size()) return st(rsb::Status::invalid_argument);
  *data = l->last[i].data();
  *len = l->last[i].size();
  return 0;
}

void rs_oplog_close(rs_oplog* l) {
  if (!l) return;
  if (l->fd >= 0) {
    ::shutdown(l->fd, SHUT_RDWR);
    ::close(l->fd);
  }
  delete l;
}

}  // extern "C"
