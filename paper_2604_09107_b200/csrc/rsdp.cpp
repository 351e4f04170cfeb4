// The reference's bulk-data wire (RSDP, transport_stream.hpp:36-76), served
// from B200 serve states, so a reference StreamData reader can pull a
// version a B200 replica holds in HBM (or in a pinned host retention lane).
//
//   header  := magic "RSDP" u32be | wire_version u16be (1) | kind u16be |
//              body_len u64be                              (16 bytes)
//   pull_req / query_req bodies: the tagged fields of codec.hpp
//     (tag u8 | type u8 | payload; u64 = 8 bytes big-endian, bytes = u32be
//     length + raw) -- 1 model, 2 replica, 3 version, 4 shard, 5 offset
//     (query: min_items), 6 max_bytes
//   pull_resp  := status u8 | progress u64be | complete u8 | payload_len
//                 u64be | payload (the item stream [offset, offset+len))
//   query_resp := status u8 | progress u64be | complete u8
//
// Semantics follow StreamDataServer::handle_pull / handle_query
// (transport_stream.cpp:355-411): compute_slice (transport.cpp:32-49) over
// the serve state's verified item prefix; a query long-polls up to 1 s for
// progress >= min_items.  A B200 serve state's verified prefix is read from
// its device watermarks, so a filling B200 replica is chased over RSDP just
// as a reference source would be.
#include <sys/socket.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "stream.hpp"

namespace rsb {
namespace {

constexpr std::uint32_t kRsdpMagic = 0x52534450;  // "RSDP"
constexpr std::uint16_t kRsdpVersion = 1;
constexpr std::uint64_t kRsdpMaxBody = 256ull << 20;  // kMaxDataBody
constexpr std::uint16_t kPullReq = 1, kPullResp = 2, kQueryReq = 3, kQueryResp = 4;
constexpr std::size_t kPullPrefix = 1 + 8 + 1 + 8;

bool read_exact(int fd, void* p, std::size_t n) {
  auto* b = static_cast<std::uint8_t*>(p);
  while (n) {
    const ssize_t k = ::recv(fd, b, n, 0);
    if (k <= 0) return false;
    b += k;
    n -= static_cast<std::size_t>(k);
  }
  return true;
}

bool write_exact(int fd, const void* p, std::size_t n) {
  const auto* b = static_cast<const std::uint8_t*>(p);
  while (n) {
    const ssize_t k = ::send(fd, b, n, MSG_NOSIGNAL);
    if (k <= 0) return false;
    b += k;
    n -= static_cast<std::size_t>(k);
  }
  return true;
}

std::uint64_t load_be(const std::uint8_t* p, int n) {
  std::uint64_t v = 0;
  for (int i = 0; i < n; ++i) v = (v << 8) | p[i];
  return v;
}

void put_be(std::string& out, std::uint64_t v, int n) {
  for (int i = n - 1; i >= 0; --i) out.push_back(static_cast<char>((v >> (8 * i)) & 0xff));
}

// codec.hpp tagged fields: the strings and u64s of a request body.
struct Fields {
  std::string str[7];
  std::uint64_t u64[7] = {};
  bool have[7] = {};
  bool parse(std::string_view d) {
    std::size_t i = 0;
    const auto* p = reinterpret_cast<const std::uint8_t*>(d.data());
    while (i < d.size()) {
      if (d.size() - i < 2) return false;
      const std::uint8_t tag = p[i], type = p[i + 1];
      i += 2;
      if (type == 1) {  // wt_u64
        if (d.size() - i < 8) return false;
        if (tag < 7) {
          u64[tag] = load_be(p + i, 8);
          have[tag] = true;
        }
        i += 8;
      } else if (type == 2) {  // wt_bytes
        if (d.size() - i < 4) return false;
        const std::uint64_t n = load_be(p + i, 4);
        i += 4;
        if (d.size() - i < n) return false;
        if (tag < 7) {
          str[tag].assign(d.data() + i, n);
          have[tag] = true;
        }
        i += n;
      } else if (type == 3) {  // wt_list (not used by data requests): skip
        if (d.size() - i < 4) return false;
        const std::uint64_t cnt = load_be(p + i, 4);
        i += 4;
        for (std::uint64_t k = 0; k < cnt; ++k) {
          if (d.size() - i < 4) return false;
          const std::uint64_t n = load_be(p + i, 4);
          i += 4 + n;
          if (i > d.size()) return false;
        }
      } else {
        return false;
      }
    }
    return true;
  }
};

std::string header(std::uint16_t kind, std::uint64_t body_len) {
  std::string h;
  put_be(h, kRsdpMagic, 4);
  put_be(h, kRsdpVersion, 2);
  put_be(h, kind, 2);
  put_be(h, body_len, 8);
  return h;
}

// Copies on a private non-blocking stream per device: a copy on the legacy
// default stream would queue behind a persistent pull kernel on that GPU
// (possibly the very fill this reader chases).
struct Copier {
  std::vector<std::pair<int, cudaStream_t>> streams;
  ~Copier() {
    for (auto& [d, st] : streams) {
      cudaSetDevice(d);
      cudaStreamDestroy(st);
    }
  }
  bool copy(void* dst, const void* src, std::size_t n, int device) {
    if (device >= 0) cudaSetDevice(device);
    cudaStream_t st = nullptr;
    for (auto& [d, x] : streams)
      if (d == device) st = x;
    if (!st) {
      if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return false;
      streams.emplace_back(device, st);
    }
    const bool good = cudaMemcpyAsync(dst, src, n, cudaMemcpyDefault, st) == cudaSuccess &&
                      cudaStreamSynchronize(st) == cudaSuccess;
    if (!good) cudaGetLastError();
    return good;
  }
};

// A snapshot of a serve state with its verified item prefix.
struct Snap {
  bool found = false, serving = false, complete = false;
  VersionId version = 0;
  std::uint64_t progress = 0;
  std::vector<std::uint64_t> item_ends, item_ptrs;
  int device = -1;
};

Snap snapshot(ServeRegistry* serves, const std::string& key, Copier& cp) {
  Snap s;
  auto st = serves->find(key);
  if (!st || serves->is_silent(key)) return s;
  ChunkMap cm;
  std::uint64_t flags = 0;
  std::uint32_t epoch = 0;
  {
    std::lock_guard lk(st->m);
    if (st->imported) return s;  // another process's state: served there
    s.found = true;
    s.serving = st->serving;
    s.complete = st->complete;
    s.version = st->version;
    s.item_ends = st->item_ends;
    s.item_ptrs = st->item_ptrs;
    s.device = st->device;
    s.progress = st->complete ? st->item_ends.size() : st->progress;
    cm = st->cmap;
    flags = st->flags;
    epoch = st->epoch;
  }
  if (!s.complete && flags && cm.chunk0.size() == s.item_ends.size() + 1) {
    // a filling replica: its verified prefix is in the device watermarks
    std::vector<std::uint32_t> f(cm.n_batches());
    if (!f.empty() && cp.copy(f.data(), reinterpret_cast<const void*>(flags), f.size() * 4, s.device)) {
      std::uint64_t items = 0;
      for (std::size_t i = 0; i + 1 < cm.chunk0.size(); ++i) {
        const std::uint32_t b0 = cm.chunk0[i] / dev::kBatchChunks;
        const std::uint32_t nb = (cm.count[i] + dev::kBatchChunks - 1) / dev::kBatchChunks;
        bool done = true;
        for (std::uint32_t b = b0; b < b0 + nb && done; ++b) done = f[b] == epoch;
        if (!done) break;
        items = i + 1;
      }
      s.progress = std::max(s.progress, items);
    }
  }
  return s;
}

bool handle_pull(int fd, ServeRegistry* serves, const Fields& f, Copier& cp) {
  for (int t = 1; t <= 6; ++t)
    if (!f.have[t]) return false;
  const Snap s =
      snapshot(serves, ServeRegistry::key(f.str[1], f.str[2], static_cast<std::uint32_t>(f.u64[4])), cp);
  const std::uint64_t offset = f.u64[5], max_bytes = f.u64[6];
  Status st = Status::ok;
  std::uint64_t bytes = 0;
  if (!s.found || !s.serving || s.version != f.u64[3]) {
    st = Status::not_serving;
  } else {
    const std::uint64_t safe = s.progress ? s.item_ends[s.progress - 1] : 0;
    if (offset < safe) bytes = std::min(max_bytes, safe - offset);
    bytes = std::min<std::uint64_t>(bytes, kRsdpMaxBody - kPullPrefix);  // one body
  }
  std::string prefix;
  prefix.push_back(static_cast<char>(st));
  put_be(prefix, ok(st) ? s.progress : 0, 8);
  prefix.push_back(ok(st) && s.complete ? 1 : 0);
  put_be(prefix, bytes, 8);
  const std::string h = header(kPullResp, prefix.size() + bytes);
  if (!write_exact(fd, h.data(), h.size()) || !write_exact(fd, prefix.data(), prefix.size())) return false;
  if (!bytes) return true;
  // copy_slice_locked over the item spans, staged D2H in 8 MiB pieces
  std::vector<std::uint8_t> buf(std::min<std::uint64_t>(bytes, 8u << 20));
  std::size_t idx = std::upper_bound(s.item_ends.begin(), s.item_ends.end(), offset) - s.item_ends.begin();
  std::uint64_t pos = offset, left = bytes;
  while (left && idx < s.item_ends.size()) {
    const std::uint64_t start = idx ? s.item_ends[idx - 1] : 0;
    const std::uint64_t in_item = pos - start;
    const std::uint64_t take = std::min({left, s.item_ends[idx] - pos, std::uint64_t(buf.size())});
    if (!cp.copy(buf.data(), reinterpret_cast<const void*>(s.item_ptrs[idx] + in_item), take, s.device))
      return false;  // the reader sees a short body: transfer_failed
    if (!write_exact(fd, buf.data(), take)) return false;
    pos += take;
    left -= take;
    if (pos == s.item_ends[idx]) ++idx;
  }
  return left == 0;
}

bool handle_query(int fd, ServeRegistry* serves, const Fields& f, Copier& cp) {
  for (int t = 1; t <= 5; ++t)
    if (!f.have[t]) return false;
  const std::string key = ServeRegistry::key(f.str[1], f.str[2], static_cast<std::uint32_t>(f.u64[4]));
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(1);  // query_bound
  Status st = Status::ok;
  Snap s;
  for (;;) {
    s = snapshot(serves, key, cp);
    if (!s.found || !s.serving || s.version != f.u64[3]) {
      st = Status::not_serving;
      break;
    }
    if (s.complete || s.progress >= f.u64[5] || std::chrono::steady_clock::now() >= deadline) break;
    std::this_thread::sleep_for(std::chrono::milliseconds(10));
  }
  std::string body;
  body.push_back(static_cast<char>(st));
  put_be(body, ok(st) ? s.progress : 0, 8);
  body.push_back(ok(st) && s.complete ? 1 : 0);
  const std::string h = header(kQueryResp, body.size());
  return write_exact(fd, h.data(), h.size()) && write_exact(fd, body.data(), body.size());
}

}  // namespace

void serve_rsdp(int fd, ServeRegistry* serves, const std::uint8_t first4[4]) {
  std::vector<char> body;
  Copier cp;
  for (bool first = true;; first = false) {
    std::uint8_t h[16];
    if (first) {
      std::memcpy(h, first4, 4);
      if (!read_exact(fd, h + 4, 12)) break;
    } else if (!read_exact(fd, h, 16)) {
      break;
    }
    if (load_be(h, 4) != kRsdpMagic || load_be(h + 4, 2) != kRsdpVersion) break;
    const std::uint64_t len = load_be(h + 8, 8);
    if (len > kRsdpMaxBody) break;
    body.resize(len);
    if (len && !read_exact(fd, body.data(), len)) break;
    Fields f;
    if (!f.parse(std::string_view(body.data(), body.size()))) break;
    const auto kind = static_cast<std::uint16_t>(load_be(h + 6, 2));
    bool good = false;
    if (kind == kPullReq) good = handle_pull(fd, serves, f, cp);
    else if (kind == kQueryReq) good = handle_query(fd, serves, f, cp);
    if (!good) break;
  }
  ::close(fd);
}

}  // namespace rsb
