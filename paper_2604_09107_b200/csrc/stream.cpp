#include "stream.hpp"

#include <arpa/inet.h>
#include <netdb.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace rsb {

namespace {

bool debug() {
  static const bool d = std::getenv("RSB_DEBUG") != nullptr;
  return d;
}

constexpr std::uint32_t kReqMagic = 0x32505352;  // "RSP2"
constexpr std::uint32_t kEnd = 0xffffffffu;
constexpr std::uint32_t kFrameBatches = 32;  // up to 32 watermark batches per frame
constexpr std::size_t kStageBytes = 8u << 20;  // per staging buffer (frames are cut to fit)
constexpr int kSlots = 16;                     // concurrent connections with staging

// Connections per source: frame k of the stream travels on connection
// k % streams (one TCP stream is bound by one core's copy; RSB_TCP_STREAMS).
// Loopback on the B200 box, 1 GiB: 1 stream 6.9 GB/s, 2: 10-13, 4: 16-19,
// 8: 21.6.  (A same-GPU stall with 4 connections was a hardware work queue
// shared by the server's staging copy and an event queued behind the
// reader's waiting kernel; Client::launch_fill queues nothing behind a
// TCP-fed kernel.)
std::uint32_t tcp_streams() {
  static const std::uint32_t n = [] {
    const char* e = std::getenv("RSB_TCP_STREAMS");
    const int v = e ? std::atoi(e) : 4;
    return static_cast<std::uint32_t>(std::clamp(v, 1, 8));
  }();
  return n;
}

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
template <class T>
bool send_vec(int fd, const std::vector<T>& v) {
  const auto n = static_cast<std::uint32_t>(v.size());
  return send_pod(fd, n) && (n == 0 || send_all(fd, v.data(), n * sizeof(T)));
}
template <class T>
bool recv_vec(int fd, std::vector<T>* v) {
  std::uint32_t n = 0;
  if (!recv_pod(fd, &n) || n > (1u << 28)) return false;  // a header table, not a payload
  v->resize(n);
  return n == 0 || recv_all(fd, v->data(), n * sizeof(T));
}

void tune(int fd) {
  int one = 1;
  setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
  static const int buf = [] {  // socket buffers (0: kernel autotuning); RSB_TCP_BUF
    const char* e = std::getenv("RSB_TCP_BUF");
    return e ? std::atoi(e) : 8 << 20;
  }();
  if (buf > 0) {
    setsockopt(fd, SOL_SOCKET, SO_SNDBUF, &buf, sizeof(buf));
    setsockopt(fd, SOL_SOCKET, SO_RCVBUF, &buf, sizeof(buf));
  }
}

// One batch's byte range inside its item.
struct BatchSpan {
  std::uint32_t item = 0;
  std::uint64_t off = 0, len = 0;
};

// Byte offset inside item i of its item-relative chunk c (the item's length
// at or past its last chunk): uniform chunks, or the item's runs when it is
// a member-cut group.
std::uint64_t chunk_offset(const ChunkMap& cm, std::uint32_t i, std::uint64_t c, std::uint64_t item_len) {
  if (!cm.cut(i)) return std::min<std::uint64_t>(c * cm.chunk_len[i], item_len);
  for (const ChunkPart& r : cm.parts[i]) {
    const std::uint64_t n = (r.len + r.chunk_len - 1) / r.chunk_len;
    if (c < r.first + n) return r.off + std::min<std::uint64_t>((c - r.first) * r.chunk_len, r.len);
  }
  return item_len;
}

std::vector<BatchSpan> batch_spans(const ChunkMap& cm, const std::vector<std::uint64_t>& item_len) {
  std::vector<BatchSpan> out(cm.n_batches());
  for (std::uint32_t i = 0; i + 1 < cm.chunk0.size(); ++i) {
    const std::uint32_t b0 = cm.chunk0[i] / dev::kBatchChunks;
    const std::uint32_t nb = (cm.count[i] + dev::kBatchChunks - 1) / dev::kBatchChunks;
    for (std::uint32_t k = 0; k < nb; ++k) {
      const std::uint64_t off = chunk_offset(cm, i, std::uint64_t(k) * dev::kBatchChunks, item_len[i]);
      const std::uint64_t end = chunk_offset(cm, i, std::uint64_t(k + 1) * dev::kBatchChunks, item_len[i]);
      out[b0 + k] = {i, off, end > off ? end - off : 0};
    }
  }
  return out;
}

// A member-cut item's runs on the wire: per item a run count, then every
// run as (offset, length, chunk length, first chunk).
void flatten_runs(const ChunkMap& cm, std::vector<std::uint32_t>* nruns, std::vector<std::uint64_t>* runs) {
  nruns->assign(cm.chunk_len.size(), 0);
  runs->clear();
  for (std::size_t i = 0; i < cm.chunk_len.size(); ++i) {
    if (!cm.cut(i)) continue;
    (*nruns)[i] = static_cast<std::uint32_t>(cm.parts[i].size());
    for (const ChunkPart& r : cm.parts[i]) runs->insert(runs->end(), {r.off, r.len, r.chunk_len, r.first});
  }
}

}  // namespace

// ------------------------------------------------------------------ server

StreamServer::StreamServer(ServeRegistry* serves) : serves_(serves) {}

StreamServer::~StreamServer() { stop(); }

Result<int> StreamServer::start(const std::string& host, int port) {
  if (listen_fd_ >= 0) return port_;
  listen_fd_ = ::socket(AF_INET, SOCK_STREAM, 0);
  if (listen_fd_ < 0) return Status::transfer_failed;
  int one = 1;
  setsockopt(listen_fd_, SOL_SOCKET, SO_REUSEADDR, &one, sizeof(one));
  sockaddr_in a{};
  a.sin_family = AF_INET;
  a.sin_port = htons(static_cast<std::uint16_t>(port));
  if (inet_pton(AF_INET, host.c_str(), &a.sin_addr) != 1 ||
      ::bind(listen_fd_, reinterpret_cast<sockaddr*>(&a), sizeof(a)) != 0 ||
      ::listen(listen_fd_, 64) != 0) {
    ::close(listen_fd_);
    listen_fd_ = -1;
    return Status::transfer_failed;
  }
  socklen_t len = sizeof(a);
  getsockname(listen_fd_, reinterpret_cast<sockaddr*>(&a), &len);
  port_ = ntohs(a.sin_port);
  for (int i = 0; i < kSlots; ++i) {
    auto sl = std::make_unique<Slot>();
    sl->bytes = kStageBytes;
    if (cudaHostAlloc(&sl->stage[0], kStageBytes, cudaHostAllocPortable) != cudaSuccess ||
        cudaHostAlloc(&sl->stage[1], kStageBytes, cudaHostAllocPortable) != cudaSuccess ||
        cudaStreamCreateWithFlags(&sl->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&sl->ev[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&sl->ev[1], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      break;
    }
    free_slots_.push_back(sl.get());
    slots_.push_back(std::move(sl));
  }
  acceptor_ = std::thread([this] { accept_loop(); });
  return port_;
}

void StreamServer::stop() {
  if (listen_fd_ < 0) return;
  stop_ = true;
  ::shutdown(listen_fd_, SHUT_RDWR);
  ::close(listen_fd_);
  listen_fd_ = -1;
  if (acceptor_.joinable()) acceptor_.join();
  {
    std::lock_guard lk(conns_mu_);
    for (auto& t : conns_)
      if (t.joinable()) t.join();
    conns_.clear();
  }
  for (auto& sl : slots_) {
    cudaStreamSynchronize(sl->stream);
    cudaEventDestroy(sl->ev[0]);
    cudaEventDestroy(sl->ev[1]);
    cudaStreamDestroy(sl->stream);
    cudaFreeHost(sl->stage[0]);
    cudaFreeHost(sl->stage[1]);
  }
  cudaGetLastError();
  slots_.clear();
  free_slots_.clear();
}

StreamServer::Slot* StreamServer::take_slot() {
  for (;;) {
    {
      std::lock_guard lk(slots_mu_);
      if (!free_slots_.empty()) {
        Slot* s = free_slots_.back();
        free_slots_.pop_back();
        return s;
      }
      if (slots_.empty() || stop_) return nullptr;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

void StreamServer::give_slot(Slot* s) {
  std::lock_guard lk(slots_mu_);
  free_slots_.push_back(s);
}

void StreamServer::accept_loop() {
  while (!stop_) {
    const int fd = ::accept(listen_fd_, nullptr, nullptr);
    if (fd < 0) {
      if (stop_) return;
      continue;
    }
    tune(fd);
    std::lock_guard lk(conns_mu_);
    conns_.emplace_back([this, fd] { serve_conn(fd); });
  }
}

void StreamServer::serve_conn(int fd) {
  auto finish = [&](std::uint32_t status) {
    send_pod(fd, status);
    ::close(fd);
  };
  std::uint32_t magic = 0, klen = 0, stripe = 0, stripes = 1;
  VersionId version = 0;
  if (!recv_pod(fd, &magic)) return (void)::close(fd);
  if (magic == 0x50445352u) {  // "RSDP": a reference StreamData peer (rsdp.cpp)
    std::uint8_t first4[4];
    std::memcpy(first4, &magic, 4);
    return serve_rsdp(fd, serves_, first4);
  }
  if (magic != kReqMagic || !recv_pod(fd, &klen) || klen > 4096) return (void)::close(fd);
  std::string key(klen, '\0');
  if (!recv_all(fd, key.data(), klen) || !recv_pod(fd, &version) || !recv_pod(fd, &stripe) ||
      !recv_pod(fd, &stripes) || stripes == 0 || stripe >= stripes)
    return (void)::close(fd);
  auto st = serves_->find(key);
  if (!st) return finish(static_cast<std::uint32_t>(Status::not_serving));
  // snapshot of the serve state (addresses in this process)
  ChunkMap cm;
  std::vector<std::uint64_t> ptrs, lens;
  std::uint64_t digests = 0, flags = 0;
  std::uint32_t epoch = 0;
  bool complete = false;
  int device = -1;
  {
    std::lock_guard lk(st->m);
    if (!st->serving || st->version != version || st->imported)
      return finish(static_cast<std::uint32_t>(Status::not_serving));
    cm = st->cmap;
    ptrs = st->item_ptrs;
    std::uint64_t prev = 0;
    for (auto e : st->item_ends) {
      lens.push_back(e - prev);
      prev = e;
    }
    digests = st->digests;
    flags = st->flags;
    epoch = st->epoch;
    complete = st->complete;
    device = st->device;
  }
  if (device >= 0) cudaSetDevice(device);
  // a member-cut item streams by its runs, which an imported state (another
  // process's replica) does not carry: such an item is not served from here
  for (std::size_t i = 0; i < cm.chunk_len.size(); ++i)
    if (cm.chunk_len[i] == 0 && !cm.cut(i)) return finish(static_cast<std::uint32_t>(Status::invalid_argument));
  const auto spans = batch_spans(cm, lens);
  for (const auto& sp : spans)
    if (sp.len > kStageBytes) return finish(static_cast<std::uint32_t>(Status::invalid_argument));
  // header (on the first connection of a source only): chunk map, item
  // lengths, chunk-digest table
  if (stripe == 0) {
    std::vector<std::uint64_t> dig(cm.n_chunks());
    if (!dig.empty() && cudaMemcpy(dig.data(), reinterpret_cast<const void*>(digests), dig.size() * 8,
                                   cudaMemcpyDefault) != cudaSuccess)
      return finish(static_cast<std::uint32_t>(Status::transfer_failed));
    std::vector<std::uint32_t> nruns;
    std::vector<std::uint64_t> runs;
    flatten_runs(cm, &nruns, &runs);
    if (!send_pod(fd, std::uint32_t{0}) || !send_vec(fd, cm.chunk0) || !send_vec(fd, cm.chunk_len) ||
        !send_vec(fd, cm.count) || !send_vec(fd, lens) || !send_vec(fd, nruns) || !send_vec(fd, runs) ||
        !send_vec(fd, dig))
      return (void)::close(fd);
  } else if (!send_pod(fd, std::uint32_t{0})) {
    return (void)::close(fd);
  }
  // payload: frames of up to kFrameBatches consecutive batches of one item,
  // each sent once the source has verified it (double-buffered D2H staging)
  const auto t_slot = std::chrono::steady_clock::now();
  Slot* slot = take_slot();
  if (!slot) return (void)::close(fd);
  if (debug()) {
    const double w = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_slot).count();
    if (w > 0.01) std::fprintf(stderr, "[rsb] stream server: stripe %u waited %.3f s for staging\n", stripe, w);
  }
  void* const* stage = slot->stage;
  cudaStream_t cs = slot->stream;
  cudaEvent_t* ev = slot->ev;
  std::vector<std::uint32_t> fl(complete ? 0 : cm.n_batches());
  auto landed = [&](std::uint32_t b) {  // the source verified batch b
    if (complete) return true;
    auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(60);
    while (fl[b] != epoch) {
      cudaMemcpy(fl.data() + b, reinterpret_cast<const std::uint32_t*>(flags) + b,
                 (fl.size() - b) * 4, cudaMemcpyDefault);
      if (fl[b] == epoch) break;
      if (std::chrono::steady_clock::now() > deadline || (fl[b] & dev::kAbort)) return false;
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    return true;
  };
  struct Frame {
    std::uint32_t b0 = 0, nb = 0;
    std::uint64_t len = 0;
  };
  std::vector<Frame> frames;  // this connection's: frame k of the stream if k % stripes == stripe
  for (std::uint32_t b = 0, k = 0; b < spans.size();) {
    if (spans[b].len == 0) {
      ++b;
      continue;
    }
    Frame f{b, 0, 0};
    while (b < spans.size() && f.nb < kFrameBatches && spans[b].len &&
           spans[b].item == spans[f.b0].item && f.len + spans[b].len <= kStageBytes) {
      f.len += spans[b].len;
      ++f.nb;
      ++b;
    }
    if (k++ % stripes == stripe) frames.push_back(f);
  }
  bool good = true;
  auto issue = [&](std::size_t k) {
    const Frame& f = frames[k];
    for (std::uint32_t b = f.b0; b < f.b0 + f.nb; ++b)
      if (!landed(b)) return false;
    const BatchSpan& s0 = spans[f.b0];
    return cudaMemcpyAsync(stage[k & 1], reinterpret_cast<const std::uint8_t*>(ptrs[s0.item]) + s0.off,
                           f.len, cudaMemcpyDefault, cs) == cudaSuccess &&
           cudaEventRecord(ev[k & 1], cs) == cudaSuccess;
  };
  if (!frames.empty()) good = issue(0);
  for (std::size_t k = 0; good && k < frames.size(); ++k) {
    if (k + 1 < frames.size()) good = issue(k + 1);
    const auto t_wait = std::chrono::steady_clock::now();
    if (!good || cudaEventSynchronize(ev[k & 1]) != cudaSuccess) {
      good = false;
      break;
    }
    if (debug()) {
      const double w = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_wait).count();
      if (w > 0.01)
        std::fprintf(stderr, "[rsb] stream server: stripe %u frame %zu D2H waited %.3f s\n", stripe, k, w);
    }
    const Frame& f = frames[k];
    good = send_pod(fd, f.b0) && send_pod(fd, f.nb) && send_pod(fd, f.len) &&
           send_all(fd, stage[k & 1], f.len);
  }
  if (debug())
    std::fprintf(stderr, "[rsb] stream server: %s v%llu stripe %u/%u: %zu frames %s\n", key.c_str(),
                 static_cast<unsigned long long>(version), stripe, stripes, frames.size(),
                 good ? "sent" : "aborted");
  if (good) {
    send_pod(fd, kEnd);
    send_pod(fd, std::uint32_t{0});
    send_pod(fd, std::uint64_t{0});
  }
  cudaStreamSynchronize(cs);
  cudaGetLastError();
  give_slot(slot);
  ::close(fd);
}

// ------------------------------------------------------------------ reader

StreamSource::~StreamSource() {
  for (int fd : fds_)
    if (fd >= 0) ::shutdown(fd, SHUT_RDWR);
  for (auto& t : rx_)
    if (t.joinable()) t.join();
  for (int fd : fds_)
    if (fd >= 0) ::close(fd);
}

Status StreamSource::open(const std::string& endpoint, const std::string& key, VersionId version,
                          double timeout_s, std::vector<std::unique_ptr<HostBuf>>* pool) {
  // endpoint "tcp:host:port"
  const auto p1 = endpoint.find(':'), p2 = endpoint.rfind(':');
  if (endpoint.rfind("tcp:", 0) != 0 || p2 == p1) return Status::invalid_argument;
  const std::string host = endpoint.substr(p1 + 1, p2 - p1 - 1);
  const int port = std::atoi(endpoint.c_str() + p2 + 1);
  sockaddr_in a{};
  a.sin_family = AF_INET;
  a.sin_port = htons(static_cast<std::uint16_t>(port));
  if (inet_pton(AF_INET, host.c_str(), &a.sin_addr) != 1) return Status::invalid_argument;
  // An assigned upstream that is not serving yet is waited for, not
  // condemned (as on the in-box path, Client::resolve_source).
  auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(timeout_s);
  const auto klen = static_cast<std::uint32_t>(key.size());
  const std::uint32_t streams = tcp_streams();
  auto connect_stripe = [&](std::uint32_t stripe, int* out) -> Status {
    for (;;) {
      int fd = ::socket(AF_INET, SOCK_STREAM, 0);
      std::uint32_t status = static_cast<std::uint32_t>(Status::not_serving);
      if (fd >= 0 && ::connect(fd, reinterpret_cast<sockaddr*>(&a), sizeof(a)) == 0) {
        tune(fd);
        if (!send_pod(fd, kReqMagic) || !send_pod(fd, klen) || !send_all(fd, key.data(), klen) ||
            !send_pod(fd, version) || !send_pod(fd, stripe) || !send_pod(fd, streams) ||
            !recv_pod(fd, &status))
          status = static_cast<std::uint32_t>(Status::transfer_failed);
        if (status == 0) {
          *out = fd;
          return Status::ok;
        }
      }
      if (fd >= 0) ::close(fd);
      if (status != static_cast<std::uint32_t>(Status::not_serving)) return static_cast<Status>(status);
      if (std::chrono::steady_clock::now() > deadline) return Status::not_serving;
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
  };
  fds_.assign(streams, -1);
  if (Status s = connect_stripe(0, &fds_[0]); !ok(s)) return s;
  ChunkMap cm;
  std::vector<std::uint64_t> lens, dig;
  const int fd0 = fds_[0];
  std::vector<std::uint32_t> nruns;
  std::vector<std::uint64_t> runs;
  if (!recv_vec(fd0, &cm.chunk0) || !recv_vec(fd0, &cm.chunk_len) || !recv_vec(fd0, &cm.count) ||
      !recv_vec(fd0, &lens) || !recv_vec(fd0, &nruns) || !recv_vec(fd0, &runs) || !recv_vec(fd0, &dig))
    return Status::protocol_error;
  // the runs of member-cut items, as the header states them
  if (nruns.size() != cm.chunk_len.size()) return Status::protocol_error;
  {
    std::uint64_t total = 0;
    for (auto n : nruns) total += n;
    if (runs.size() != 4 * total) return Status::protocol_error;
    cm.parts.assign(nruns.size(), {});
    std::size_t at = 0;
    for (std::size_t i = 0; i < nruns.size(); ++i)
      for (std::uint32_t k = 0; k < nruns[i]; ++k, at += 4) {
        if (runs[at + 2] == 0 || runs[at + 2] > (1u << 30) || runs[at + 3] > (1u << 30))
          return Status::protocol_error;
        cm.parts[i].push_back(ChunkPart{runs[at], runs[at + 1], static_cast<std::uint32_t>(runs[at + 2]),
                                        static_cast<std::uint32_t>(runs[at + 3])});
      }
  }
  if (!valid_header(cm, lens) || dig.size() != cm.n_chunks()) return Status::protocol_error;
  // every stripe's socket gives up when its source stays silent well past
  // the pull timeout (the kernel has failed by then; finish() shuts it too)
  const double rx_s = 2 * timeout_s + 1;
  timeval tv{static_cast<time_t>(rx_s), static_cast<suseconds_t>((rx_s - std::floor(rx_s)) * 1e6)};
  setsockopt(fd0, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof(tv));
  for (std::uint32_t k = 1; k < streams; ++k) {
    if (Status s = connect_stripe(k, &fds_[k]); !ok(s)) return s;
    setsockopt(fds_[k], SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof(tv));
  }
  item_len_ = lens;
  // pinned, device-mapped landing for the stream + digests + watermarks
  item_off_.resize(lens.size());
  std::uint64_t tot = 0;
  for (std::size_t i = 0; i < lens.size(); ++i) {
    item_off_[i] = tot;
    tot += (lens[i] + 255) / 256 * 256;
  }
  static const bool no_pool = std::getenv("RSB_TCP_NOPOOL") != nullptr;  // diagnostic
  auto take = [&](std::size_t n, std::unique_ptr<HostBuf>* out) -> Status {
    if (pool && !no_pool)
      for (auto it = pool->begin(); it != pool->end(); ++it)
        if ((*it)->n >= n) {
          *out = std::move(*it);
          pool->erase(it);
          return Status::ok;
        }
    *out = std::make_unique<HostBuf>();
    return (*out)->alloc(n);
  };
  if (Status s = take(tot, &data_); !ok(s)) return s;
  const std::size_t nb = cm.n_batches();
  if (Status s = take(dig.size() * 8 + nb * 4 + 16, &tables_); !ok(s)) return s;
  auto* tb = static_cast<std::uint8_t*>(tables_->p);
  if (!dig.empty()) std::memcpy(tb, dig.data(), dig.size() * 8);
  std::memset(tb + dig.size() * 8, 0, nb * 4);
  view_.cmap = cm;
  view_.item_ptrs.resize(lens.size());
  for (std::size_t i = 0; i < lens.size(); ++i)
    view_.item_ptrs[i] = reinterpret_cast<std::uint64_t>(data_->p) + item_off_[i];
  view_.digests = reinterpret_cast<std::uint64_t>(tb);
  view_.flags = reinterpret_cast<std::uint64_t>(tb + dig.size() * 8);
  view_.epoch = 1;
  view_.total = tot;
  for (int fd : fds_) rx_.emplace_back([this, fd] { receive_loop(fd); });
  return Status::ok;
}

bool StreamSource::valid_header(const ChunkMap& cm, const std::vector<std::uint64_t>& lens) {
  // The header comes off the wire: every table the receive threads index
  // must agree with the item count, and the chunk map must be the batch
  // aligned, monotone partition of the item lengths (ChunkMap::from_lens).
  const std::size_t n = lens.size();
  if (cm.chunk0.size() != n + 1 || cm.chunk_len.size() != n || cm.count.size() != n ||
      cm.chunk0[0] != 0 || cm.chunk0.back() > (1u << 30))
    return false;
  if (!cm.parts.empty() && cm.parts.size() != n) return false;
  for (std::size_t i = 0; i < n; ++i) {
    const std::uint32_t cl = cm.chunk_len[i];
    if (cm.chunk0[i] % dev::kBatchChunks != 0) return false;
    if (cl == 0) {
      // member-cut: runs back to back from byte 0, covering the item, their
      // chunks numbered consecutively from 0
      if (!cm.cut(i)) return false;
      std::uint64_t off = 0, first = 0;
      for (const ChunkPart& r : cm.parts[i]) {
        if (r.off != off || r.first != first || r.chunk_len == 0 || r.len == 0) return false;
        off += r.len;
        first += (r.len + r.chunk_len - 1) / r.chunk_len;
      }
      if (off != lens[i] || first != cm.count[i]) return false;
    } else {
      if (cm.cut(i)) return false;
      if (cm.count[i] != (lens[i] + cl - 1) / cl) return false;
    }
    if (std::uint64_t(cm.chunk0[i]) + cm.count[i] > cm.chunk0[i + 1]) return false;
  }
  return true;
}

void StreamSource::receive_loop(int fd) {
  const ChunkMap& cm = view_.cmap;
  // item of every batch and the batch's offset inside it
  std::vector<std::uint32_t> item_of(cm.n_batches(), 0);
  std::vector<std::uint64_t> off_of(cm.n_batches(), 0);
  for (std::uint32_t i = 0; i + 1 < cm.chunk0.size(); ++i) {
    const std::uint32_t b0 = cm.chunk0[i] / dev::kBatchChunks;
    const std::uint32_t nb = (cm.count[i] + dev::kBatchChunks - 1) / dev::kBatchChunks;
    for (std::uint32_t k = 0; k < nb; ++k) {
      item_of[b0 + k] = i;
      off_of[b0 + k] = chunk_offset(cm, i, std::uint64_t(k) * dev::kBatchChunks, item_len_[i]);
    }
  }
  auto* flags = reinterpret_cast<std::uint32_t*>(view_.flags);
  auto* base = static_cast<std::uint8_t*>(data_->p);
  auto fail = [&](Status st) {
    int expect = 0;
    rx_status_.compare_exchange_strong(expect, static_cast<int>(st));
    abort_all();
  };
  for (;;) {
    std::uint32_t b0 = 0, nb = 0;
    std::uint64_t len = 0;
    if (!recv_pod(fd, &b0) || !recv_pod(fd, &nb) || !recv_pod(fd, &len)) return fail(Status::transfer_failed);
    if (b0 == kEnd) break;
    // a frame is a run of whole batches of one item, exactly their bytes
    if (nb == 0 || b0 >= item_of.size() || nb > item_of.size() - b0) return fail(Status::protocol_error);
    const std::uint32_t i = item_of[b0];
    if (item_of[b0 + nb - 1] != i || (b0 + nb - 1) * std::uint64_t(dev::kBatchChunks) >=
                                         std::uint64_t(cm.chunk0[i]) + cm.count[i])
      return fail(Status::protocol_error);
    const std::uint64_t end = chunk_offset(
        cm, i, std::uint64_t(b0 + nb) * dev::kBatchChunks - cm.chunk0[i], item_len_[i]);
    if (off_of[b0] >= end && item_len_[i] != 0) return fail(Status::protocol_error);
    if (len != end - off_of[b0]) return fail(Status::protocol_error);
    if (!recv_all(fd, base + item_off_[i] + off_of[b0], len)) return fail(Status::transfer_failed);
    received_ += len;
    // the bytes are in memory before the watermarks the GPU polls (x86
    // stores are ordered; the kernel reads the flag with ld.acquire.sys)
    std::atomic_thread_fence(std::memory_order_release);
    for (std::uint32_t b = b0; b < b0 + nb; ++b)
      __atomic_store_n(&flags[b], 1u, __ATOMIC_RELEASE);
  }
}

void StreamSource::abort_all() {
  if (debug()) std::fprintf(stderr, "[rsb] stream source: receive failed (%d)\n", rx_status_.load());
  // the kernel chasing these watermarks stops at once (not_serving)
  auto* flags = reinterpret_cast<std::uint32_t*>(view_.flags);
  for (std::uint32_t b = 0; b < view_.cmap.n_batches(); ++b)
    if (__atomic_load_n(&flags[b], __ATOMIC_ACQUIRE) != 1u)
      __atomic_store_n(&flags[b], 1u | dev::kAbort, __ATOMIC_RELEASE);
}

std::pair<std::uint32_t, std::uint32_t> StreamSource::flag_summary() const {
  const auto* flags = reinterpret_cast<const std::uint32_t*>(view_.flags);
  std::uint32_t set = 0, first = ~0u;
  for (std::uint32_t b = 0; b < view_.cmap.n_batches(); ++b) {
    if (__atomic_load_n(&flags[b], __ATOMIC_ACQUIRE) == 1u) ++set;
    else if (first == ~0u) first = b;
  }
  return {set, first};
}

void StreamSource::release(std::vector<std::unique_ptr<HostBuf>>* pool) {
  for (auto& t : rx_)
    if (t.joinable()) t.join();
  if (!pool) return;
  for (auto* b : {&data_, &tables_})
    if (*b && pool->size() < 4) pool->push_back(std::move(*b));
}

Status StreamSource::finish(bool kernel_ok) {
  // A fill that failed (checksum, timeout) does not wait for the rest of the
  // stream: the receive threads return at once on the shut sockets.
  if (!kernel_ok)
    for (int fd : fds_)
      if (fd >= 0) ::shutdown(fd, SHUT_RDWR);
  for (auto& t : rx_)
    if (t.joinable()) t.join();
  return static_cast<Status>(rx_status_.load());
}

}  // namespace rsb
