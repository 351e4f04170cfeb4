#include "client.hpp"

#include "stream.hpp"

#include <cuda.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>

namespace rsb {

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

Status cuda_status(cudaError_t e, const char* what = nullptr, int line = 0) {
  if (e == cudaSuccess) return Status::ok;
  static const bool debug = std::getenv("RSB_DEBUG") != nullptr;
  if (debug && what)
    std::fprintf(stderr, "[rsb] client.cpp:%d %s -> %s\n", line, what, cudaGetErrorString(e));
  return Status::transfer_failed;
}

#define RS_CUDA(expr)                                          \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return cuda_status(_e, #expr, __LINE__); \
  } while (0)

// cuMemGetAddressRange through the runtime's driver entry point (no libcuda
// link dependency, so the library still loads on a GPU-less host).
using GetRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
GetRangeFn get_range_fn() {
  static GetRangeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<GetRangeFn>(nullptr);
    return reinterpret_cast<GetRangeFn>(p);
  }();
  return fn;
}

// Binary writer/reader for serve-state export blobs.
struct W {
  std::string s;
  template <class T>
  void pod(const T& v) {
    s.append(reinterpret_cast<const char*>(&v), sizeof(T));
  }
  void str(const std::string& v) {
    pod(static_cast<std::uint32_t>(v.size()));
    s.append(v);
  }
  template <class T>
  void vec(const std::vector<T>& v) {
    pod(static_cast<std::uint32_t>(v.size()));
    s.append(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(T));
  }
};
struct R {
  const char* p;
  std::size_t n, i = 0;
  bool ok = true;
  template <class T>
  T pod() {
    T v{};
    if (i + sizeof(T) > n) {
      ok = false;
      return v;
    }
    std::memcpy(static_cast<void*>(&v), p + i, sizeof(T));
    i += sizeof(T);
    return v;
  }
  std::string str() {
    auto len = pod<std::uint32_t>();
    if (!ok || i + len > n) {
      ok = false;
      return {};
    }
    std::string v(p + i, len);
    i += len;
    return v;
  }
  template <class T>
  std::vector<T> vec() {
    auto len = pod<std::uint32_t>();
    std::vector<T> v;
    if (!ok || i + std::size_t(len) * sizeof(T) > n) {
      ok = false;
      return v;
    }
    v.resize(len);
    std::memcpy(static_cast<void*>(v.data()), p + i, std::size_t(len) * sizeof(T));
    i += std::size_t(len) * sizeof(T);
    return v;
  }
};

constexpr std::uint32_t kBlobMagic = 0x31425352;  // "RSB1"

// IPC mappings opened in this process.  An exported allocation is mapped
// once per reader device and kept while some imported serve state refers to
// it; when the last such state moves to other allocations (its owner re-bound
// or re-published and freed the old tables) the mappings are closed -- the
// owner's allocator may hand the same addresses out again, and a stale
// mapping of them would make the new handle unmappable.
struct IpcEntry {
  int refs = 0;                 // imported serve states referring to the allocation
  std::map<int, void*> mapped;  // reader device -> mapped base
};
std::mutex g_ipc_mu;
std::map<std::string, IpcEntry> g_ipc;

std::string ipc_key(const cudaIpcMemHandle_t& h) {
  return std::string(reinterpret_cast<const char*>(&h), sizeof(h));
}

Result<std::uint64_t> open_ipc(const cudaIpcMemHandle_t& h, int device) {
  std::lock_guard lk(g_ipc_mu);
  IpcEntry& e = g_ipc[ipc_key(h)];
  auto it = e.mapped.find(device);
  if (it != e.mapped.end()) return reinterpret_cast<std::uint64_t>(it->second);
  DeviceGuard g(device);
  void* p = nullptr;
  if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    return Status::not_serving;
  }
  e.mapped[device] = p;
  return reinterpret_cast<std::uint64_t>(p);
}

// An imported state now refers to `now` instead of `before`.
void retarget_ipc(const std::vector<ServeState::Alloc>& before,
                  const std::vector<ServeState::Alloc>& now) {
  std::set<std::string> b, n;
  for (const auto& a : before) b.insert(ipc_key(a.handle));
  for (const auto& a : now) n.insert(ipc_key(a.handle));
  std::lock_guard lk(g_ipc_mu);
  for (const auto& k : n)
    if (!b.count(k)) ++g_ipc[k].refs;
  for (const auto& k : b) {
    if (n.count(k)) continue;
    auto it = g_ipc.find(k);
    if (it == g_ipc.end() || --it->second.refs > 0) continue;
    for (auto& [dev, p] : it->second.mapped) {
      DeviceGuard g(dev);
      cudaIpcCloseMemHandle(p);
      cudaGetLastError();
    }
    g_ipc.erase(it);
  }
}

// Host (retention offload) segments mapped into this process by name, kept
// while an imported serve state refers to them.
struct HostEntry {
  int refs = 0;
  void* p = nullptr;
  std::size_t n = 0;
};
std::mutex g_host_mu;
std::map<std::string, HostEntry> g_host;

Result<std::uint64_t> open_host(const std::string& name, std::size_t n) {
  std::lock_guard lk(g_host_mu);
  HostEntry& e = g_host[name];
  if (e.p) return reinterpret_cast<std::uint64_t>(e.p);
  const int fd = shm_open(name.c_str(), O_RDWR, 0);
  if (fd < 0) return Status::not_serving;
  void* p = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return Status::not_serving;
  if (cudaHostRegister(p, n, cudaHostRegisterPortable | cudaHostRegisterMapped) != cudaSuccess) {
    cudaGetLastError();
    munmap(p, n);
    return Status::not_serving;
  }
  e.p = p;
  e.n = n;
  return reinterpret_cast<std::uint64_t>(p);
}

void retarget_host(const std::string& before, const std::string& now) {
  if (before == now) return;
  std::lock_guard lk(g_host_mu);
  if (!now.empty()) ++g_host[now].refs;
  if (before.empty()) return;
  auto it = g_host.find(before);
  if (it == g_host.end() || --it->second.refs > 0) return;
  if (it->second.p) {
    cudaHostUnregister(it->second.p);
    cudaGetLastError();
    munmap(it->second.p, it->second.n);
  }
  g_host.erase(it);
}

}  // namespace

// ------------------------------------------------------------------ DevBuf

HostBuf::~HostBuf() {
  if (!p) return;
  cudaHostUnregister(p);
  cudaGetLastError();
  munmap(p, n);
  shm_unlink(name.c_str());
}

Status HostBuf::alloc(std::size_t bytes) {
  static std::atomic<std::uint64_t> ctr{0};
  name = "/rsb-" + std::to_string(getpid()) + "-" + std::to_string(ctr++);
  n = bytes ? bytes : 1;
  const int fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
  if (fd < 0) return Status::offload_failed;
  const bool sized = ftruncate(fd, static_cast<off_t>(n)) == 0;
  void* q = sized ? mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd, 0)
                  : MAP_FAILED;
  close(fd);
  if (q == MAP_FAILED) {
    shm_unlink(name.c_str());
    return Status::offload_failed;
  }
  if (cudaHostRegister(q, n, cudaHostRegisterPortable | cudaHostRegisterMapped) != cudaSuccess) {
    cudaGetLastError();
    munmap(q, n);
    shm_unlink(name.c_str());
    return Status::offload_failed;
  }
  p = q;
  return Status::ok;
}

DevBuf::~DevBuf() {
  if (p) {
    DeviceGuard g(dev);
    cudaFree(p);
  }
}

namespace {
// RSB_TIMING=1: host wall time of the replicate phases on stderr (diagnostic)
struct PhaseClock {
  bool on = std::getenv("RSB_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[rsb] %s %.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};
}  // namespace

Status DevBuf::alloc(int device, std::size_t bytes) {
  if (p && n >= bytes && dev == device) return Status::ok;
  if (p) {
    DeviceGuard g(dev);
    cudaFree(p);
    p = nullptr;
  }
  DeviceGuard g(device);
  dev = device;
  n = bytes ? bytes : 16;
  if (cudaMalloc(&p, n) != cudaSuccess) {
    p = nullptr;
    n = 0;
    return Status::transfer_failed;
  }
  return Status::ok;
}

// ---------------------------------------------------------------- ChunkMap

ChunkMap ChunkMap::uniform(const Manifest& m, std::uint64_t chunk_bytes) {
  return from_lens(m, std::vector<std::uint32_t>(m.items().size(),
                                                 static_cast<std::uint32_t>(chunk_bytes)));
}

ChunkMap ChunkMap::from_lens(const Manifest& m, const std::vector<std::uint32_t>& lens,
                             const std::vector<std::uint32_t>& member_lens) {
  ChunkMap c;
  std::uint32_t next = 0;
  const auto& items = m.items();
  c.parts.resize(items.size());
  for (std::size_t i = 0; i < items.size(); ++i) {
    std::uint32_t n = 0, cl32 = 0;
    if (i < lens.size() && lens[i] == 0 && items[i].is_group && !member_lens.empty()) {
      // member-cut group: one run per member, in packing order
      std::vector<GroupMember> mem = m.groups[items[i].index].members;
      std::sort(mem.begin(), mem.end(),
                [](const GroupMember& a, const GroupMember& b) { return a.offset < b.offset; });
      for (const auto& g : mem) {
        const std::uint64_t len = m.entries[g.entry].length;
        const std::uint64_t cl = g.entry < member_lens.size() && member_lens[g.entry] ? member_lens[g.entry] : 4096;
        c.parts[i].push_back(ChunkPart{g.offset, len, static_cast<std::uint32_t>(cl), n});
        n += static_cast<std::uint32_t>((len + cl - 1) / cl);
      }
    } else {
      const std::uint64_t cl = i < lens.size() && lens[i] ? lens[i] : 4096;
      n = static_cast<std::uint32_t>((items[i].length + cl - 1) / cl);
      cl32 = static_cast<std::uint32_t>(cl);
    }
    c.chunk0.push_back(next);
    c.chunk_len.push_back(cl32);
    c.count.push_back(n);
    next += (n + dev::kBatchChunks - 1) / dev::kBatchChunks * dev::kBatchChunks;
  }
  c.chunk0.push_back(next);
  return c;
}

ChunkMap ChunkMap::from_layout(const Manifest& m, const ShardLayout& lay, std::uint64_t chunk_bytes,
                               std::uint32_t align) {
  return from_lens(m, lay.chunk_len, member_chunk_lens(m, lay.geo, chunk_bytes, align));
}

// Item-for-item segments of item `item` (one per chunk run); dst 0: hash only.
void append_identity(std::vector<dev::ItemDesc>* out, std::uint64_t src, std::uint64_t dst,
                     std::uint64_t len, const ChunkMap& cm, std::size_t item) {
  for (const ChunkPart& r : cm.runs(item, len)) {
    dev::ItemDesc d{};
    d.src = src + r.off;
    d.dst = dst ? dst + r.off : 0;
    d.len = r.len;
    d.chunk0 = cm.chunk0[item] + r.first;
    d.chunk_len = r.chunk_len;
    d.src_chunk0 = d.chunk0;
    d.q = 1;
    d.m = 1;
    d.src_id = 0;
    out->push_back(d);
  }
}

// ----------------------------------------------------------- ServeRegistry

std::string ServeRegistry::key(const std::string& model, const std::string& replica,
                               std::uint32_t shard) {
  return model + "|" + replica + "|" + std::to_string(shard);
}

std::shared_ptr<ServeState> ServeRegistry::ensure(const std::string& k) {
  std::lock_guard lk(m_);
  auto& slot = map_[k];
  if (!slot) slot = std::make_shared<ServeState>();
  return slot;
}

std::shared_ptr<ServeState> ServeRegistry::find(const std::string& k) const {
  std::lock_guard lk(m_);
  auto it = map_.find(k);
  return it == map_.end() ? nullptr : it->second;
}

void ServeRegistry::erase(const std::string& k) {
  std::shared_ptr<ServeState> st;
  {
    std::lock_guard lk(m_);
    auto it = map_.find(k);
    if (it == map_.end()) return;
    st = it->second;
    map_.erase(it);
  }
  std::lock_guard lk(st->m);
  if (st->imported) {
    retarget_ipc(st->allocs, {});
    retarget_host(st->host_name, {});
  }
  st->allocs.clear();
}

void ServeRegistry::set_silent(const std::string& model, const std::string& replica, bool on) {
  std::lock_guard lk(m_);
  const std::string prefix = model + "|" + replica + "|";
  if (on) silent_.insert(prefix);
  else silent_.erase(prefix);
}

bool ServeRegistry::is_silent(const std::string& k) const {
  std::lock_guard lk(m_);
  for (const auto& p : silent_)
    if (k.compare(0, p.size(), p) == 0) return true;
  return false;
}

Result<std::string> ServeRegistry::export_state(const std::string& k) {
  auto st = find(k);
  if (!st) return Status::not_found;
  std::lock_guard lk(st->m);
  if (st->imported) return Status::invalid_state;
  if (!st->host_name.empty()) {  // a retention offload: named shared memory
    std::vector<std::pair<std::uint32_t, std::uint64_t>> item_loc(st->item_ptrs.size());
    for (std::size_t i = 0; i < st->item_ptrs.size(); ++i) item_loc[i] = {0, st->item_ptrs[i] - st->host_base};
    W w;
    w.pod(kBlobMagic);
    w.str(k);
    w.pod(st->version);
    w.pod(static_cast<std::uint8_t>(st->serving));
    w.pod(static_cast<std::uint8_t>(st->complete));
    w.pod(st->progress);
    w.pod(st->epoch);
    w.pod(st->device);
    w.pod(static_cast<std::int32_t>(getpid()));
    w.vec(st->item_ends);
    w.vec(st->cmap.chunk0);
    w.vec(st->cmap.chunk_len);
    w.vec(st->cmap.count);
    w.vec(std::vector<ServeState::Alloc>{});
    w.vec(item_loc);
    w.pod(std::pair<std::uint32_t, std::uint64_t>{0, st->digests - st->host_base});
    w.pod(std::pair<std::uint32_t, std::uint64_t>{0, 0});
    w.str(st->host_name);
    w.pod(st->host_size);
    return w.s;
  }
  auto range = get_range_fn();
  if (!range) return Status::transfer_failed;
  DeviceGuard g(st->device);
  std::vector<ServeState::Alloc> allocs;
  std::map<std::uint64_t, std::uint32_t> by_base;
  auto locate = [&](std::uint64_t ptr, std::pair<std::uint32_t, std::uint64_t>* loc) -> Status {
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, static_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
      return Status::invalid_argument;
    auto it = by_base.find(base);
    if (it == by_base.end()) {
      ServeState::Alloc a{};
      if (cudaIpcGetMemHandle(&a.handle, reinterpret_cast<void*>(base)) != cudaSuccess)
        return Status::invalid_argument;
      a.size = size;
      it = by_base.emplace(base, static_cast<std::uint32_t>(allocs.size())).first;
      allocs.push_back(a);
    }
    *loc = {it->second, ptr - base};
    return Status::ok;
  };
  std::vector<std::pair<std::uint32_t, std::uint64_t>> item_loc(st->item_ptrs.size());
  for (std::size_t i = 0; i < st->item_ptrs.size(); ++i)
    if (Status s = locate(st->item_ptrs[i], &item_loc[i]); !ok(s)) return s;
  std::pair<std::uint32_t, std::uint64_t> dl{0, 0}, fl{0, 0};
  if (Status s = locate(st->digests, &dl); !ok(s)) return s;
  if (Status s = locate(st->flags, &fl); !ok(s)) return s;
  W w;
  w.pod(kBlobMagic);
  w.str(k);
  w.pod(st->version);
  w.pod(static_cast<std::uint8_t>(st->serving));
  w.pod(static_cast<std::uint8_t>(st->complete));
  w.pod(st->progress);
  w.pod(st->epoch);
  w.pod(st->device);
  w.pod(static_cast<std::int32_t>(getpid()));
  w.vec(st->item_ends);
  w.vec(st->cmap.chunk0);
  w.vec(st->cmap.chunk_len);
  w.vec(st->cmap.count);
  w.vec(allocs);
  w.vec(item_loc);
  w.pod(dl);
  w.pod(fl);
  w.str(std::string());
  w.pod(std::uint64_t{0});
  return w.s;
}

Status ServeRegistry::import_state(const std::string& blob) {
  R r{blob.data(), blob.size()};
  if (r.pod<std::uint32_t>() != kBlobMagic) return Status::protocol_error;
  std::string k = r.str();
  auto version = r.pod<VersionId>();
  bool serving = r.pod<std::uint8_t>() != 0;
  bool complete = r.pod<std::uint8_t>() != 0;
  auto progress = r.pod<std::uint64_t>();
  auto epoch = r.pod<std::uint32_t>();
  auto device = r.pod<int>();
  auto pid = r.pod<std::int32_t>();
  auto ends = r.vec<std::uint64_t>();
  auto c0 = r.vec<std::uint32_t>();
  auto cl = r.vec<std::uint32_t>();
  auto cc = r.vec<std::uint32_t>();
  auto allocs = r.vec<ServeState::Alloc>();
  auto item_loc = r.vec<std::pair<std::uint32_t, std::uint64_t>>();
  auto dl = r.pod<std::pair<std::uint32_t, std::uint64_t>>();
  auto fl = r.pod<std::pair<std::uint32_t, std::uint64_t>>();
  std::string host_name = r.str();
  auto host_size = r.pod<std::uint64_t>();
  if (!r.ok) return Status::protocol_error;
  if (pid == getpid()) return Status::ok;  // our own state: nothing to import
  auto st = ensure(k);
  std::lock_guard lk(st->m);
  st->imported = true;
  st->serving = serving;
  st->complete = complete;
  st->version = version;
  st->progress = progress;
  st->epoch = epoch;
  st->device = device;
  st->pid = pid;
  st->item_ends = std::move(ends);
  st->cmap.chunk0 = std::move(c0);
  st->cmap.chunk_len = std::move(cl);
  st->cmap.count = std::move(cc);
  retarget_ipc(st->imported ? st->allocs : std::vector<ServeState::Alloc>{}, allocs);
  retarget_host(st->imported ? st->host_name : std::string(), host_name);
  st->host_name = std::move(host_name);
  st->host_size = host_size;
  st->allocs = std::move(allocs);
  st->item_loc = std::move(item_loc);
  st->digests_loc = dl;
  st->flags_loc = fl;
  return Status::ok;
}

// --------------------------------------------------------- address mapping

Status enable_peer(int reader_device, int owner_device) {
  if (reader_device == owner_device) return Status::ok;
  static std::mutex mu;
  static std::set<std::pair<int, int>> done;
  std::lock_guard lk(mu);
  if (done.count({reader_device, owner_device})) return Status::ok;
  int can = 0;
  cudaDeviceCanAccessPeer(&can, reader_device, owner_device);
  if (!can) return Status::not_serving;
  DeviceGuard g(reader_device);
  cudaError_t e = cudaDeviceEnablePeerAccess(owner_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    e = cudaSuccess;
  }
  if (e != cudaSuccess) return Status::not_serving;
  done.insert({reader_device, owner_device});
  return Status::ok;
}

Status map_source(const std::shared_ptr<ServeState>& st, int reader_device, SourceView* out) {
  std::lock_guard lk(st->m);
  out->device = st->host_name.empty() ? st->device : -1;
  out->cmap = st->cmap;
  out->epoch = st->epoch;
  out->total = st->item_ends.empty() ? 0 : st->item_ends.back();
  if (!st->imported) {
    if (st->device >= 0)  // a host lane (device < 0) needs no peer mapping
      if (Status s = enable_peer(reader_device, st->device); !ok(s)) return s;
    out->item_ptrs = st->item_ptrs;
    out->digests = st->digests;
    out->flags = st->flags;
    return Status::ok;
  }
  if (!st->host_name.empty()) {  // another process's retention offload
    auto b = open_host(st->host_name, st->host_size);
    if (!b) return b.status();
    out->item_ptrs.resize(st->item_loc.size());
    for (std::size_t i = 0; i < st->item_loc.size(); ++i) out->item_ptrs[i] = *b + st->item_loc[i].second;
    out->digests = *b + st->digests_loc.second;
    out->flags = 0;
    return Status::ok;
  }
  std::vector<std::uint64_t> bases(st->allocs.size());
  for (std::size_t a = 0; a < st->allocs.size(); ++a) {
    auto b = open_ipc(st->allocs[a].handle, reader_device);
    if (!b) return b.status();
    bases[a] = *b;
  }
  out->item_ptrs.resize(st->item_loc.size());
  for (std::size_t i = 0; i < st->item_loc.size(); ++i)
    out->item_ptrs[i] = bases[st->item_loc[i].first] + st->item_loc[i].second;
  out->digests = bases[st->digests_loc.first] + st->digests_loc.second;
  out->flags = bases[st->flags_loc.first] + st->flags_loc.second;
  return Status::ok;
}

// ------------------------------------------------------------------ Client

Client::Client(Registry* reg, ServeRegistry* serves, std::string model, std::string replica,
               std::uint32_t num_shards, ClientConfig cfg)
    : reg_(reg),
      serves_(serves),
      model_(std::move(model)),
      replica_(std::move(replica)),
      num_shards_(num_shards),
      cfg_(std::move(cfg)) {
  shards_.resize(num_shards_);
  for (std::uint32_t i = 0; i < num_shards_; ++i) shards_[i].idx = i;
}

Client::~Client() {
  if (fin_thread_.joinable()) fin_thread_.join();
  join_seed();
  stop_serving();
  for (auto& sh : shards_) {
    if (sh.device < 0) continue;
    DeviceGuard g(sh.device);
    if (sh.ev0) cudaEventDestroy(sh.ev0);
    if (sh.ev1) cudaEventDestroy(sh.ev1);
    if (sh.own_stream && sh.stream) cudaStreamDestroy(sh.stream);
    if (sh.poll) cudaStreamDestroy(sh.poll);
    if (sh.k6) cudaStreamDestroy(sh.k6);
    if (sh.dma) {
      cudaStreamSynchronize(sh.dma);
      cudaStreamDestroy(sh.dma);
    }
    dev::free_pull_plan(sh.device, &sh.plan);
    dev::free_pull_plan(sh.device, &sh.hash_plan);
    dev::free_pull_plan(sh.device, &sh.fuse_plan);
    dev::free_pull_plan(sh.device, &sh.seed_plan);
    if (sh.seed_ev) cudaEventDestroy(sh.seed_ev);
    if (sh.seed_stream) cudaStreamDestroy(sh.seed_stream);
    for (auto& [v, lane] : sh.seed_lanes) serves_->erase(lane.key);
  }
}

Status Client::register_tensor(std::uint32_t shard, const std::string& name, void* ptr,
                               std::uint64_t len, const Geometry& geo, bool cast) {
  // validation order of ClientCore::register_tensor (client_core.cpp:534-553)
  if (closed_) return Status::closed;
  if (shard >= num_shards_ || name.empty() || name.find('|') != std::string::npos)
    return Status::invalid_argument;
  if (!ptr || len == 0) return Status::invalid_argument;
  if (cast && (len % 2 || (geo.has() && geo.nc % 2))) return Status::invalid_argument;  // bf16
  if (geo.has() && (geo.nr * geo.nc != len || geo.r0 + geo.nr > geo.rows ||
                    geo.c0 + geo.nc > geo.row_bytes))
    return Status::invalid_argument;
  if (published_ || current_) return Status::invalid_state;
  Shard& sh = shards_[shard];
  if (sh.by_name.count(name)) return Status::already_exists;
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, ptr) != cudaSuccess || attr.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    return Status::invalid_argument;  // registered regions live in device memory
  }
  if (sh.device < 0) sh.device = attr.device;
  if (sh.device != attr.device) return Status::invalid_argument;  // one device per shard
  if (sh.endpoint.empty()) sh.endpoint = "cuda:" + std::to_string(sh.device);
  sh.by_name[name] = static_cast<std::uint32_t>(sh.regs.size());
  sh.regs.push_back({name, static_cast<std::uint8_t*>(ptr), len, geo, cast});
  return Status::ok;
}

namespace {
struct Fnv {
  std::uint64_t h = 1469598103934665603ull;
  void mix(const void* p, std::size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  }
};
}  // namespace

Client::ShardHash Client::shard_hash(std::uint32_t shard) const {
  // FNV-1a over (shard, name, length, geometry) of the shard's regions
  ShardHash out;
  if (shard >= num_shards_) return out;
  const Shard& sh = shards_[shard];
  Fnv f;
  f.mix(&sh.idx, sizeof(sh.idx));
  for (const auto& r : sh.regs) {
    out.geometry |= r.geo.has();
    out.cast |= r.cast;
    f.mix(r.name.data(), r.name.size());
    const std::uint64_t v[7] = {r.len, r.geo.rows, r.geo.row_bytes, r.geo.r0,
                                r.geo.nr, r.geo.c0, r.geo.nc};
    f.mix(v, sizeof(v));
  }
  out.hash = f.h;
  return out;
}

std::string Client::combine_layout_key(const std::vector<ShardHash>& shards) {
  // plain replicas (no geometry anywhere) keep the reference's single slicing ""
  bool any = false, cast = false;
  Fnv f;
  for (const auto& s : shards) {
    any |= s.geometry;
    cast |= s.cast;
    f.mix(&s.hash, sizeof(s.hash));
  }
  const std::string mark = cast ? "!" : "";
  if (!any) return mark;
  char buf[32];
  std::snprintf(buf, sizeof(buf), "L%016llx", static_cast<unsigned long long>(f.h));
  return mark + buf;
}

std::string Client::layout_key() const {
  std::vector<ShardHash> hs;
  for (std::uint32_t i = 0; i < num_shards_; ++i) hs.push_back(shard_hash(i));
  return combine_layout_key(hs);
}

bool Client::terminal() const {
  for (const auto& sh : shards_)
    for (const auto& r : sh.regs)
      if (r.cast) return true;
  return false;
}

void Client::set_shard_endpoint(std::uint32_t shard, std::string ep) {
  if (shard < num_shards_) shards_[shard].endpoint = std::move(ep);
}

void Client::set_stream(std::uint32_t shard, cudaStream_t s) {
  if (shard >= num_shards_) return;
  Shard& sh = shards_[shard];
  if (sh.own_stream && sh.stream) {
    DeviceGuard g(sh.device);
    cudaStreamDestroy(sh.stream);
  }
  sh.stream = s;
  sh.own_stream = false;
}

int Client::grid(const Shard& sh) const {
  const int sms = dev::pull_grid(sh.device);
  return cfg_.grid_sms ? std::min<int>(sms, static_cast<int>(cfg_.grid_sms)) : sms;
}

Status Client::ensure_stream(Shard& sh) {
  if (sh.device < 0) return Status::invalid_state;
  DeviceGuard g(sh.device);
  if (!sh.stream) {
    RS_CUDA(cudaStreamCreateWithFlags(&sh.stream, cudaStreamNonBlocking));
    sh.own_stream = true;
  }
  if (!sh.ev0) RS_CUDA(cudaEventCreate(&sh.ev0));
  if (!sh.ev1) RS_CUDA(cudaEventCreate(&sh.ev1));
  return Status::ok;
}

Status Client::open() {
  std::vector<std::string> eps;
  for (auto& sh : shards_) {
    if (sh.device < 0) return Status::invalid_state;  // nothing registered on a shard
    eps.push_back(sh.endpoint);
  }
  std::vector<std::string> dman, dlay;
  if (Status s = derived_blobs(&dman, &dlay); !ok(s)) return s;
  Status s = reg_->open(model_, replica_, num_shards_, cfg_.dc, eps, layout_key(), dman, dlay);
  if (ok(s) && !retain_.empty()) s = reg_->set_retention(model_, replica_, retain_);
  if (ok(s) && cfg_.offload_seed) s = reg_->set_offload_seed(model_, replica_, true);
  if (ok(s)) opened_ = true;
  return s;
}

// ---- publish --------------------------------------------------------------

Status Client::build_payload(Shard& sh, VersionId v, std::shared_ptr<Payload>* out) {
  if (Status s = ensure_stream(sh); !ok(s)) return s;
  DeviceGuard g(sh.device);
  const std::size_t n = sh.regs.size();
  auto p = std::make_shared<Payload>();
  PhaseClock pc;
  RS_CUDA(cudaEventRecord(sh.ev0, sh.stream));

  // Entry digests (K6).
  std::vector<std::uint64_t> ptrs(n), lens(n), dig(n, 0);
  for (std::size_t i = 0; i < n; ++i) {
    ptrs[i] = reinterpret_cast<std::uint64_t>(sh.regs[i].ptr);
    lens[i] = sh.regs[i].len;
  }
  // Early publish: the big entries (>= tiny_threshold: items of their own)
  // are digested on sh.k6 in the background (launched below, beside the
  // chunk-table hash pass); the manifest carries 0 for them until then.
  std::vector<std::uint32_t> now, later;
  for (std::uint32_t i = 0; i < n; ++i)
    (cfg_.early_publish && lens[i] >= cfg_.limits.tiny_threshold ? later : now).push_back(i);
  // The background digest stream and its tables exist from the first
  // publish in either mode (sized for every entry), so an early publish --
  // the latency-critical one -- creates and allocates nothing: stream
  // creation + cudaMalloc were measured at 0.8-52 ms there.
  if (!sh.k6) RS_CUDA(cudaStreamCreateWithFlags(&sh.k6, cudaStreamNonBlocking));
  if (Status s = sh.k6_tables.alloc(sh.device, std::max<std::size_t>(3 * n, 1) * 8); !ok(s)) return s;
  pc.mark("build_payload: k6 stream + tables");
  // Library buffers of a publish are reused across publishes (a cudaFree
  // synchronizes the device and was measured taking up to 0.44 s here).
  DevBuf& tab = sh.dig_tables;
  if (Status s = tab.alloc(sh.device, std::max<std::size_t>(3 * n, 1) * 8); !ok(s)) return s;
  auto* d = static_cast<std::uint64_t*>(tab.p);
  if (!now.empty()) {
    const std::size_t nn = now.size();
    std::vector<std::uint64_t> np(nn), nl(nn), nd(nn);
    for (std::size_t k = 0; k < nn; ++k) {
      np[k] = ptrs[now[k]];
      nl[k] = lens[now[k]];
    }
    RS_CUDA(cudaMemcpyAsync(d, np.data(), nn * 8, cudaMemcpyHostToDevice, sh.stream));
    RS_CUDA(cudaMemcpyAsync(d + nn, nl.data(), nn * 8, cudaMemcpyHostToDevice, sh.stream));
    RS_CUDA(dev::launch_span_digests(d, d + nn, d + 2 * nn, static_cast<int>(nn), sh.stream));
    ++stats_.kernel_launches;
    RS_CUDA(cudaMemcpyAsync(nd.data(), d + 2 * nn, nn * 8, cudaMemcpyDeviceToHost, sh.stream));
    pc.mark("build_payload: small-entry digests queued");
    RS_CUDA(cudaStreamSynchronize(sh.stream));
    for (std::size_t k = 0; k < nn; ++k) dig[now[k]] = nd[k];
    stats_.h2d_bytes += 16 * nn;
    stats_.d2h_bytes += 8 * nn;
  }
  pc.mark("build_payload: entry digests");
  std::vector<EntryInfo> infos(n);
  for (std::size_t i = 0; i < n; ++i) infos[i] = {sh.regs[i].name, lens[i], dig[i]};
  auto mr = assemble(infos, cfg_.limits);
  if (!mr) return mr.status();
  p->manifest = std::move(*mr);

  // Tiny-tensor groups: pack (K3) then digest (K6) the staging buffer.
  const std::size_t ng = p->manifest.groups.size();
  if (ng) {
    std::vector<std::uint64_t> srcs, dsts, ls, gp(ng), gl(ng), gd(ng);
    for (std::size_t gi = 0; gi < ng; ++gi) {
      const auto& grp = p->manifest.groups[gi];
      // the payload being replaced has drained (see alloc_tables): its
      // group staging is taken over when large enough
      std::unique_ptr<DevBuf> buf;
      if (sh.holding && gi < sh.holding->group_bufs.size() && sh.holding->group_bufs[gi] &&
          sh.holding->group_bufs[gi]->n >= grp.packed_length && sh.holding->group_bufs[gi]->dev == sh.device)
        buf = std::move(sh.holding->group_bufs[gi]);
      else
        buf = std::make_unique<DevBuf>();
      if (Status s = buf->alloc(sh.device, grp.packed_length); !ok(s)) return s;
      for (const auto& mem : grp.members) {
        srcs.push_back(ptrs[mem.entry]);
        dsts.push_back(reinterpret_cast<std::uint64_t>(buf->p) + mem.offset);
        ls.push_back(lens[mem.entry]);
      }
      gp[gi] = reinterpret_cast<std::uint64_t>(buf->p);
      gl[gi] = grp.packed_length;
      p->group_bufs.push_back(std::move(buf));
    }
    if (Status s = copy_spans(sh, srcs, dsts, ls); !ok(s)) return s;
    DevBuf& gt = sh.group_tables;
    if (Status s = gt.alloc(sh.device, 3 * ng * 8); !ok(s)) return s;
    auto* g2 = static_cast<std::uint64_t*>(gt.p);
    RS_CUDA(cudaMemcpyAsync(g2, gp.data(), ng * 8, cudaMemcpyHostToDevice, sh.stream));
    RS_CUDA(cudaMemcpyAsync(g2 + ng, gl.data(), ng * 8, cudaMemcpyHostToDevice, sh.stream));
    RS_CUDA(dev::launch_span_digests(g2, g2 + ng, g2 + 2 * ng, static_cast<int>(ng), sh.stream));
    ++stats_.kernel_launches;
    RS_CUDA(cudaMemcpyAsync(gd.data(), g2 + 2 * ng, ng * 8, cudaMemcpyDeviceToHost, sh.stream));
    RS_CUDA(cudaStreamSynchronize(sh.stream));
    stats_.h2d_bytes += 16 * ng;
    stats_.d2h_bytes += 8 * ng;
    for (std::size_t gi = 0; gi < ng; ++gi)
      p->manifest.set_group_digest(static_cast<std::uint32_t>(gi), gd[gi]);
  }

  pc.mark("build_payload: groups");
  // Serving addresses per item, chunk map, chunk digest table + watermarks.
  const auto& items = p->manifest.items();
  p->item_ptrs.resize(items.size());
  for (std::size_t i = 0; i < items.size(); ++i)
    p->item_ptrs[i] = items[i].is_group
                          ? reinterpret_cast<std::uint64_t>(p->group_bufs[items[i].index]->p)
                          : ptrs[items[i].index];
  // Chunk lengths from the regions' geometry (layout.hpp chunk rule).
  ShardLayout lay;
  for (const auto& r : sh.regs) lay.geo.push_back(r.geo);
  lay.chunk_len = item_chunk_lens(p->manifest, lay.geo, cfg_.chunk_bytes, cfg_.reshard_align);
  p->cmap = ChunkMap::from_layout(p->manifest, lay, cfg_.chunk_bytes, cfg_.reshard_align);
  p->layout = lay.encode();
  if (Status s = alloc_tables(sh, *p, 0); !ok(s)) return s;
  pc.mark("build_payload: tables");
  p->epoch = ++sh.epoch_ctr;
  // Chunk digest table of the published bytes (hash-only pull), and every
  // watermark set: a complete source.
  std::vector<std::uint32_t> all(items.size());
  for (std::size_t i = 0; i < items.size(); ++i) all[i] = static_cast<std::uint32_t>(i);
  if (Status s = hash_items(sh, *p, all); !ok(s)) return s;
  RS_CUDA(cudaEventRecord(sh.ev1, sh.stream));
  pc.mark("build_payload: hash pass queued");
  if (!later.empty()) {
    // launched only now, after every allocation of this publish (the hash
    // pass's plan included): a device allocation issued while it runs would
    // serialise the rest behind it.  It starts behind the hash pass: its
    // CTAs (one per entry, hundreds of ms each) dispatched first would hold
    // the SMs' shared memory and keep the persistent hash pass from
    // launching until they drain (seen: publish 4 ms -> 89 ms, one run in two)
    const std::size_t nl = later.size();
    std::vector<std::uint64_t> lp(nl), ll(nl);
    for (std::size_t k = 0; k < nl; ++k) {
      lp[k] = ptrs[later[k]];
      ll[k] = lens[later[k]];
    }
    auto* kd = static_cast<std::uint64_t*>(sh.k6_tables.p);
    RS_CUDA(cudaStreamWaitEvent(sh.k6, sh.ev1, 0));  // behind the hash pass (and all prior work)
    RS_CUDA(cudaMemcpyAsync(kd, lp.data(), nl * 8, cudaMemcpyHostToDevice, sh.k6));
    RS_CUDA(cudaMemcpyAsync(kd + nl, ll.data(), nl * 8, cudaMemcpyHostToDevice, sh.k6));
    RS_CUDA(dev::launch_span_digests(kd, kd + nl, kd + 2 * nl, static_cast<int>(nl), sh.k6));
    ++stats_.kernel_launches;
    stats_.h2d_bytes += 16 * nl;
  }

  pc.mark("build_payload: K6 queued");
  RS_CUDA(cudaStreamSynchronize(sh.stream));
  pc.mark("build_payload: hash pass done");
  float ms = 0;
  cudaEventElapsedTime(&ms, sh.ev0, sh.ev1);
  stats_.last_publish_ms = ms;
  p->encoded = p->manifest.encode();
  p->provisional = !later.empty();
  p->deferred = std::move(later);
  *out = std::move(p);
  return Status::ok;
}

// ---- early publish: background digests ------------------------------------

void Client::start_finalize(VersionId v) {
  struct Work {
    int device;
    cudaStream_t k6;
    const std::uint64_t* out;
    std::vector<std::uint32_t> deferred;
    Manifest manifest;
  };
  std::vector<std::optional<Work>> work(num_shards_);
  bool any = false;
  for (auto& sh : shards_) {
    if (sh.device < 0 || !sh.holding || sh.holding->deferred.empty()) continue;
    const auto nl = sh.holding->deferred.size();
    work[sh.idx] = Work{sh.device, sh.k6, static_cast<const std::uint64_t*>(sh.k6_tables.p) + 2 * nl,
                        sh.holding->deferred, sh.holding->manifest};
    any = true;
  }
  if (!any) return;
  if (fin_thread_.joinable()) fin_thread_.join();  // a previous publish's (normally joined already)
  bool all_local = true;
  std::vector<std::string> held(num_shards_);  // shards with nothing deferred: final already
  for (std::uint32_t i = 0; i < num_shards_; ++i) {
    all_local &= is_local(i);
    if (!work[i] && is_local(i) && shards_[i].holding) held[i] = shards_[i].holding->encoded;
  }
  {
    std::lock_guard lk(fin_m_);
    fin_running_ = true;
    fin_v_ = v;
    fin_status_ = Status::ok;
    fin_manifests_.assign(num_shards_, std::string());
  }
  // the thread touches no Client state but the fin_ fields and the registry
  fin_thread_ = std::thread([this, v, all_local, work = std::move(work), held = std::move(held)]() mutable {
    std::vector<std::string> finals = std::move(held);
    Status st = Status::ok;
    for (std::uint32_t i = 0; i < num_shards_; ++i) {
      if (!work[i]) continue;
      Work& w = *work[i];
      DeviceGuard g(w.device);
      std::vector<std::uint64_t> dg(w.deferred.size());
      if (cudaMemcpyAsync(dg.data(), w.out, dg.size() * 8, cudaMemcpyDeviceToHost, w.k6) != cudaSuccess ||
          cudaStreamSynchronize(w.k6) != cudaSuccess) {
        st = Status::transfer_failed;
        continue;
      }
      for (std::size_t k = 0; k < dg.size(); ++k) w.manifest.set_entry_digest(w.deferred[k], dg[k]);
      finals[i] = w.manifest.encode();
    }
    // the in-process registry takes the final bytes now; a replica split over
    // processes commits them through its caller (rs_server_finalize)
    if (ok(st) && all_local) st = reg_->finalize_manifests(model_, replica_, v, finals);
    std::lock_guard lk(fin_m_);
    fin_status_ = st;
    fin_manifests_ = std::move(finals);
    fin_running_ = false;
  });
}

Status Client::join_finalize() {
  if (fin_thread_.joinable()) fin_thread_.join();
  std::lock_guard lk(fin_m_);
  if (fin_manifests_.empty()) return fin_status_;
  for (auto& sh : shards_) {
    if (sh.idx >= fin_manifests_.size() || !sh.holding || sh.holding->deferred.empty()) continue;
    const std::string& fb = fin_manifests_[sh.idx];
    if (!ok(fin_status_) || fb.empty()) continue;
    auto m = Manifest::decode(fb);
    if (!m || !m->same_structure(sh.holding->manifest)) continue;
    sh.holding->manifest = std::move(*m);
    sh.holding->encoded = fb;
    sh.holding->provisional = false;
    sh.holding->deferred.clear();
  }
  fin_manifests_.clear();
  return fin_status_;
}

Status Client::finalize_publish(double wait_s, std::vector<std::string>* manifests) {
  (void)wait_s;  // the digests are a bounded kernel: the join always returns
  Status st = join_finalize();
  if (ok(st) && publish_pending()) st = Status::invalid_state;  // no committed publish to finish
  if (manifests) {
    manifests->clear();
    for (auto& sh : shards_) manifests->push_back(sh.device >= 0 && sh.holding ? sh.holding->encoded : "");
  }
  return st;
}

Status Client::adopt_final(Shard& sh, double wait_s) {
  if (!sh.holding || !sh.holding->provisional) return Status::ok;
  if (!sh.holding->deferred.empty()) return join_finalize();  // this publisher's own digests
  const std::optional<VersionId> v = current_ ? current_ : sh.partial_version;
  if (!v) return Status::not_found;
  auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(wait_s);
  for (;;) {
    std::string bytes;
    bool fin = false;
    if (Status s = reg_->replica_manifest(model_, replica_, *v, sh.idx, &bytes, &fin); !ok(s)) return s;
    if (fin) {
      auto m = Manifest::decode(bytes);
      if (!m || !m->same_structure(sh.holding->manifest)) return Status::manifest_conflict;
      sh.holding->manifest = std::move(*m);
      sh.holding->encoded = bytes;
      sh.holding->provisional = false;
      return Status::ok;
    }
    if (std::chrono::steady_clock::now() > deadline) return Status::timeout;
    std::this_thread::sleep_for(std::chrono::milliseconds(1));
  }
}

Status Client::alloc_tables(Shard& sh, Payload& p, std::uint32_t extra_chunks) {
  DeviceGuard g(sh.device);
  const std::uint32_t nc = p.cmap.n_chunks() + extra_chunks;
  const std::uint32_t nb = (nc + dev::kBatchChunks - 1) / dev::kBatchChunks;
  if (sh.holding && sh.holding.get() != &p && sh.holding->digests.n >= std::size_t(nc) * 8 &&
      sh.holding->flags.n >= std::size_t(nb) * 4) {
    // The payload being replaced has drained (an unpublish or update settles
    // only with no readers left): keep its tables -- same allocations, so
    // the IPC mappings other processes hold stay valid and nothing re-pins.
    p.digests = std::move(sh.holding->digests);
    p.flags = std::move(sh.holding->flags);
  } else {
    if (Status s = p.digests.alloc(sh.device, std::size_t(nc) * 8); !ok(s)) return s;
    if (Status s = p.flags.alloc(sh.device, std::size_t(nb) * 4); !ok(s)) return s;
  }
  RS_CUDA(cudaMemsetAsync(p.flags.p, 0, std::size_t(nb) * 4, sh.stream));
  RS_CUDA(cudaMemsetAsync(p.digests.p, 0, std::size_t(nc) * 8, sh.stream));
  return Status::ok;
}

Status Client::hash_items(Shard& sh, Payload& p, const std::vector<std::uint32_t>& which,
                          const std::uint32_t* guard) {
  // Hash-only pull over some of the payload's own items: fills their chunk
  // digests and releases their watermarks in the current epoch.
  if (which.empty() || p.cmap.n_chunks() == 0) return Status::ok;
  DeviceGuard g(sh.device);
  const auto& items = p.manifest.items();
  std::vector<dev::ItemDesc> descs;
  for (std::uint32_t i : which) append_identity(&descs, p.item_ptrs[i], 0, items[i].length, p.cmap, i);
  const dev::SrcDesc self{nullptr, nullptr, 0, 0};
  dev::PullParams pp{};
  RS_CUDA(dev::upload_pull_plan(sh.device, sh.stream, descs.data(),
                                static_cast<std::uint32_t>(descs.size()), &self, 1,
                                p.cmap.n_chunks(), &sh.hash_plan, &pp));
  pp.first_batch = descs.front().chunk0 / dev::kBatchChunks;
  pp.dst_digests = static_cast<std::uint64_t*>(p.digests.p);
  pp.dst_flags = static_cast<std::uint32_t*>(p.flags.p);
  pp.dst_epoch = p.epoch;
  pp.timeout_ns = static_cast<std::uint64_t>(cfg_.pull_timeout_s * 1e9);
  pp.guard = guard;
  RS_CUDA(dev::launch_pull(pp, grid(sh), sh.stream));
  stats_.kernel_launches += dev::pull_has_work(pp) ? 1 : 0;
  stats_.h2d_bytes += sh.hash_plan.h2d_bytes;
  return Status::ok;
}

Status Client::prepare_publish(VersionId v, std::vector<std::string>* manifests,
                               std::vector<std::string>* layouts) {
  if (terminal()) return Status::invalid_state;  // regions hold a cast, not the version
  join_finalize();  // the previous publish's background digests
  manifests->clear();
  if (layouts) layouts->clear();
  for (auto& sh : shards_) {
    if (sh.device < 0) {  // another process publishes it
      manifests->emplace_back();
      if (layouts) layouts->emplace_back();
      continue;
    }
    std::shared_ptr<Payload> p;
    PhaseClock pc;
    if (Status s = build_payload(sh, v, &p); !ok(s)) return s;
    pc.mark("publish: build_payload");
    sh.holding = std::move(p);
    pc.mark("publish: drop the previous payload");
    manifests->push_back(sh.holding->encoded);
    if (layouts) layouts->push_back(sh.holding->layout);
  }
  return Status::ok;
}

bool Client::derived_layout(std::vector<std::string>* manifests,
                            std::vector<std::string>* layouts) const {
  manifests->clear();
  layouts->clear();
  for (const auto& sh : shards_) {
    if (sh.device < 0) {
      manifests->emplace_back();
      layouts->emplace_back();
      continue;
    }
    if (!sh.holding || !sh.holding->reshard) return false;
    manifests->push_back(sh.holding->encoded);
    layouts->push_back(sh.holding->layout);
  }
  return true;
}

Result<std::string> Client::layout_bytes(std::uint32_t shard) const {
  if (shard >= num_shards_ || !shards_[shard].holding) return Status::not_found;
  return shards_[shard].holding->layout;
}

void Client::commit_publish(VersionId v, Status st) {
  if (!ok(st)) return;
  for (auto& sh : shards_) {
    if (sh.device < 0) continue;
    sh.partial_version.reset();
    serve(sh, v, true);
  }
  current_ = v;
  published_ = true;
  start_finalize(v);  // early publish: the background digests (no-op otherwise)
}

Status Client::publish(VersionId v) {
  if (!opened_) {
    if (Status s = open(); !ok(s)) return s;
  }
  if (published_) return Status::mutability_violation;
  std::vector<std::string> manifests, layouts;
  if (Status s = prepare_publish(v, &manifests, &layouts); !ok(s)) return s;
  PhaseClock pc;
  OpOutcome o;
  Status s = reg_->publish(model_, replica_, v, manifests, &o, layouts, publish_pending());
  if (ok(s)) s = o.status;
  pc.mark("publish: registry");
  commit_publish(v, s);
  pc.mark("publish: commit");
  return s;
}

Status Client::unpublish() {
  if (!opened_) return Status::invalid_state;
  // an early publish's digests still read the regions: finish them before
  // the caller may mutate the weights
  join_finalize();
  apply_releases();
  OpOutcome o;
  Status s = reg_->unpublish(model_, replica_, &o);
  if (!ok(s)) return s;
  if (Status so = settle_offload(&o, 600.0); !ok(so)) return so;
  if (!o.done) o = reg_->wait_op(model_, replica_, 600.0);
  if (!o.done) return Status::timeout;
  if (ok(o.status)) {
    published_ = false;
    stop_serving();
  }
  return o.status;
}

// ---- serve state ----------------------------------------------------------

void Client::serve(Shard& sh, VersionId v, bool complete) {
  if (!sh.serve) sh.serve = serves_->ensure(ServeRegistry::key(model_, replica_, sh.idx));
  const auto& p = *sh.holding;
  std::vector<std::uint64_t> ends;
  for (const auto& it : p.manifest.items()) ends.push_back(it.stream_offset + it.length);
  std::lock_guard lk(sh.serve->m);
  sh.serve->serving = true;
  sh.serve->imported = false;
  sh.serve->version = v;
  sh.serve->complete = complete;
  sh.serve->progress = complete ? p.manifest.items().size() : 0;
  sh.serve->device = sh.device;
  sh.serve->pid = static_cast<int>(getpid());
  sh.serve->item_ends = std::move(ends);
  sh.serve->item_ptrs = p.item_ptrs;
  sh.serve->cmap = p.cmap;
  sh.serve->digests = reinterpret_cast<std::uint64_t>(p.digests.p);
  sh.serve->flags = reinterpret_cast<std::uint64_t>(p.flags.p);
  sh.serve->epoch = p.epoch;
}

void Client::invalidate() {
  for (auto& sh : shards_) {
    if (sh.holding) {
      sh.holding->epoch = ++sh.epoch_ctr;
      sh.holding->landed_some = false;
    }
    sh.partial_version.reset();
  }
  current_.reset();
}

void Client::stop_serving() {
  for (auto& sh : shards_) {
    if (!sh.serve) continue;
    std::lock_guard lk(sh.serve->m);
    sh.serve->serving = false;
  }
}

// ---- receive --------------------------------------------------------------

Status Client::resolve_source(Shard& sh, const Assignment& a, VersionId v, SourceView* out,
                              double wait_s) {
  // An assigned upstream that is not serving yet is waited for, not
  // condemned (the reference's threaded race).
  auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(wait_s);
  const std::string k = ServeRegistry::key(model_, a.source_replica, sh.idx);
  for (;;) {
    auto st = serves_->is_silent(k) ? nullptr : serves_->find(k);
    if (st) {
      bool ready, same_gpu_filling;
      {
        std::lock_guard lk(st->m);
        ready = st->serving && st->version == v && !st->cmap.chunk0.empty();
        // A persistent pull kernel holds every SM of its GPU, so a chaser on
        // the upstream's own GPU could start first, spin, and starve the fill
        // it waits for: on one GPU the chase waits for the upstream instead.
        // A capped grid (rs_config.grid_sms) is the caller's promise that
        // the two fills co-reside, so the chase runs concurrently.
        same_gpu_filling = !st->imported && st->device == sh.device && !st->complete &&
                           cfg_.grid_sms == 0;
      }
      if (ready && !same_gpu_filling) return map_source(st, sh.device, out);
      if (ready) deadline = std::max(deadline, std::chrono::steady_clock::now() +
                                                   std::chrono::duration<double>(4 * wait_s));
    }
    if (std::chrono::steady_clock::now() > deadline) return Status::not_serving;
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

Status Client::bind(Shard& sh, const Assignment& a, VersionId v) {
  if (Status s = ensure_stream(sh); !ok(s)) return s;
  bool same = sh.holding && sh.holding->encoded == a.manifest;
  if (sh.holding && !same && (sh.holding->provisional || a.provisional) && sh.holding->deferred.empty()) {
    // an early publish's provisional bytes against its final ones (or the
    // reverse): the same version's payload when the structure agrees
    auto m = Manifest::decode(a.manifest);
    const bool vsame = (current_ && *current_ == v) || (sh.partial_version && *sh.partial_version == v);
    if (m && vsame && m->same_structure(sh.holding->manifest)) {
      if (!a.provisional) {
        sh.holding->manifest = std::move(*m);
        sh.holding->encoded = a.manifest;
        sh.holding->provisional = false;
      }
      same = true;
    }
  }
  if (same) {
    // Identical manifest: resume.  Keeping the fill epoch keeps every batch
    // already landed for this version (flag == epoch) out of the pull.
    bool resume = (current_ && *current_ == v) || (sh.partial_version && *sh.partial_version == v);
    if (!resume) {
      sh.holding->epoch = ++sh.epoch_ctr;
      sh.holding->landed_some = false;
    }
    sh.partial_version = v;
    sh.reported = 0;
    return Status::ok;
  }
  auto mr = Manifest::decode(a.manifest);
  if (!mr) return Status::protocol_error;
  if (mr->entries.size() != sh.regs.size()) return Status::invalid_argument;
  for (const auto& e : mr->entries) {
    auto it = sh.by_name.find(e.name);
    if (it == sh.by_name.end() || sh.regs[it->second].len != e.length)
      return Status::invalid_argument;
  }
  DeviceGuard g(sh.device);
  auto p = std::make_shared<Payload>();
  p->manifest = std::move(*mr);
  p->encoded = a.manifest;
  const auto& items = p->manifest.items();
  // Everything that can reject the assignment is checked before any buffer
  // is taken over from the payload being replaced.  The chunk map is a pure
  // function of (manifest, the publisher's chunk lengths), so a reader can
  // serve its own fill before its source is even reachable.
  if (!a.layout.empty()) {
    auto lay = ShardLayout::decode(a.layout);
    if (!lay || lay->chunk_len.size() != items.size()) return Status::protocol_error;
    p->cmap = ChunkMap::from_layout(p->manifest, *lay, cfg_.chunk_bytes, cfg_.reshard_align);
    p->layout = a.layout;
  } else {
    p->cmap = ChunkMap::uniform(p->manifest, cfg_.chunk_bytes);
  }
  // Buffers taken over from the drained payload go back to it if a later
  // step fails, so its serve state never points at freed memory.
  std::vector<std::size_t> taken;  // group indices whose staging came from sh.holding
  auto give_back = [&](Status st) {
    if (sh.holding) {
      for (std::size_t gi : taken)
        if (p->group_bufs[gi]) sh.holding->group_bufs[gi] = std::move(p->group_bufs[gi]);
      if (p->digests.p && !sh.holding->digests.p) sh.holding->digests = std::move(p->digests);
      if (p->flags.p && !sh.holding->flags.p) sh.holding->flags = std::move(p->flags);
    }
    return st;
  };
  for (std::size_t gi = 0; gi < p->manifest.groups.size(); ++gi) {
    // group staging of the drained payload being replaced is taken over
    // (no cudaFree / cudaMalloc on the update path; see alloc_tables)
    p->group_bufs.push_back(nullptr);
    if (sh.holding && gi < sh.holding->group_bufs.size() && sh.holding->group_bufs[gi] &&
        sh.holding->group_bufs[gi]->dev == sh.device) {
      p->group_bufs.back() = std::move(sh.holding->group_bufs[gi]);
      taken.push_back(gi);
    } else {
      p->group_bufs.back() = std::make_unique<DevBuf>();
    }
    if (Status s = p->group_bufs.back()->alloc(sh.device, p->manifest.groups[gi].packed_length); !ok(s))
      return give_back(s);
  }
  p->item_ptrs.resize(items.size());
  for (std::size_t i = 0; i < items.size(); ++i) {
    const auto& it = items[i];
    p->item_ptrs[i] =
        it.is_group ? reinterpret_cast<std::uint64_t>(p->group_bufs[it.index]->p)
                    : reinterpret_cast<std::uint64_t>(
                          sh.regs[sh.by_name.at(p->manifest.entries[it.index].name)].ptr);
  }
  if (Status s = alloc_tables(sh, *p, 0); !ok(s)) return give_back(s);
  if (cudaStreamSynchronize(sh.stream) != cudaSuccess) return give_back(Status::transfer_failed);
  p->epoch = ++sh.epoch_ctr;
  p->provisional = a.provisional;
  sh.holding = std::move(p);
  sh.partial_version = v;
  sh.reported = 0;
  return Status::ok;
}

Status Client::derive(const Shard& sh, Manifest* m, std::string* encoded, std::string* layout,
                      std::vector<std::uint32_t>* lens) const {
  std::vector<EntryInfo> infos;
  for (const auto& r : sh.regs) infos.push_back({r.name, r.len, 0});
  auto mr = assemble(infos, cfg_.limits);
  if (!mr) return mr.status();
  *m = std::move(*mr);
  m->alg = kAlgDerived;
  *encoded = m->encode();
  ShardLayout lay;
  for (const auto& r : sh.regs) lay.geo.push_back(r.geo);
  lay.chunk_len = item_chunk_lens(*m, lay.geo, cfg_.chunk_bytes, cfg_.reshard_align);
  *layout = lay.encode();
  if (lens) *lens = lay.chunk_len;
  return Status::ok;
}

Status Client::derived_blobs(std::vector<std::string>* manifests,
                             std::vector<std::string>* layouts) const {
  manifests->clear();
  layouts->clear();
  bool any_geo = false;
  for (std::uint32_t i = 0; i < num_shards_; ++i) any_geo |= shard_hash(i).geometry;
  if (!any_geo) return Status::ok;  // plain replica: nothing derived
  for (const auto& sh : shards_) {
    if (sh.device < 0) {  // a shard of this replica held by another process
      manifests->emplace_back();
      layouts->emplace_back();
      continue;
    }
    Manifest m;
    std::string enc, lay;
    if (Status s = derive(sh, &m, &enc, &lay, nullptr); !ok(s)) return s;
    manifests->push_back(std::move(enc));
    layouts->push_back(std::move(lay));
  }
  return Status::ok;
}

Status Client::bind_reshard(Shard& sh, const Assignment& a, VersionId v) {
  // K4 reshard: this shard's slicing differs from the source's.  Its own
  // manifest is derived (alg 2: same entries/groups as the reference would
  // assemble, digests not computed); its chunks follow the chunk rule on its
  // own geometry; the plan maps them onto the source shards' chunks.
  if (Status s = ensure_stream(sh); !ok(s)) return s;
  if (!a.all_manifests || !a.all_layouts) return Status::protocol_error;
  auto same = [](const Assignment::Blobs& x, const Assignment::Blobs& y) {
    return x == y || (x && y && *x == *y);  // shared snapshot, or equal bytes
  };
  if (sh.holding && sh.holding->reshard && same(sh.holding->reshard->src_manifests, a.all_manifests) &&
      same(sh.holding->reshard->src_layouts, a.all_layouts)) {
    // Same source slicing and bytes' manifests: keep the plan and the tables;
    // a new fill epoch unless this resumes the same version's fill.
    bool resume = (current_ && *current_ == v) || (sh.partial_version && *sh.partial_version == v);
    if (!resume) {
      sh.holding->epoch = ++sh.epoch_ctr;
      sh.holding->landed_some = false;
    }
    sh.holding->reshard->endpoints = a.all_endpoints;
    sh.partial_version = v;
    return Status::ok;
  }
  DeviceGuard g(sh.device);
  auto p = std::make_shared<Payload>();
  std::vector<std::uint32_t> lens;
  if (Status s = derive(sh, &p->manifest, &p->encoded, &p->layout, &lens); !ok(s)) return s;
  {
    auto own = ShardLayout::decode(p->layout);
    if (!own) return Status::protocol_error;
    p->cmap = ChunkMap::from_layout(p->manifest, *own, cfg_.chunk_bytes, cfg_.reshard_align);
  }
  for (const auto& grp : p->manifest.groups) {
    auto buf = std::make_unique<DevBuf>();
    if (Status s = buf->alloc(sh.device, grp.packed_length); !ok(s)) return s;
    p->group_bufs.push_back(std::move(buf));
  }
  const auto& items = p->manifest.items();
  p->item_ptrs.resize(items.size());
  for (std::size_t i = 0; i < items.size(); ++i)
    p->item_ptrs[i] = items[i].is_group
                          ? reinterpret_cast<std::uint64_t>(p->group_bufs[items[i].index]->p)
                          : reinterpret_cast<std::uint64_t>(sh.regs[items[i].index].ptr);
  // Source shards as the planner sees them.
  auto rs = std::make_unique<Reshard>();
  rs->endpoints = a.all_endpoints;
  rs->src_manifests = a.all_manifests;
  rs->src_layouts = a.all_layouts;
  const auto& all_man = *a.all_manifests;
  const auto& all_lay = *a.all_layouts;
  for (std::size_t s = 0; s < all_man.size(); ++s) {
    SourceShard ss;
    auto sm = Manifest::decode(all_man[s]);
    if (!sm) return Status::protocol_error;
    ss.manifest = std::move(*sm);
    if (s < all_lay.size() && !all_lay[s].empty()) {
      auto sl = ShardLayout::decode(all_lay[s]);
      if (!sl) return Status::protocol_error;
      ss.layout = std::move(*sl);
    } else {
      ss.layout.chunk_len.assign(ss.manifest.items().size(),
                                 static_cast<std::uint32_t>(cfg_.chunk_bytes));
    }
    {
      ChunkMap scm = ChunkMap::from_layout(ss.manifest, ss.layout, cfg_.chunk_bytes, cfg_.reshard_align);
      ss.chunk0 = std::move(scm.chunk0);
      ss.parts = std::move(scm.parts);
    }
    rs->srcs.push_back(std::move(ss));
  }
  std::vector<ReaderEntry> rd;
  for (std::uint32_t e = 0; e < sh.regs.size(); ++e) {
    ReaderEntry re;
    re.name = sh.regs[e].name;
    re.ptr = reinterpret_cast<std::uint64_t>(sh.regs[e].ptr);
    re.len = sh.regs[e].len;
    re.geo = sh.regs[e].geo;
    re.cast = sh.regs[e].cast;
    re.in_group = p->manifest.group_of(e) >= 0;
    if (!re.in_group) {
      for (std::uint32_t i = 0; i < items.size(); ++i)
        if (!items[i].is_group && items[i].index == e) {
          re.item = i;
          re.chunk0 = p->cmap.chunk0[i];
          re.chunk_len = p->cmap.chunk_len[i];
        }
    } else if (!re.cast) {
      // a member of a member-cut group of this reader: its place in the
      // group's staging and its own run of chunks
      const auto g = static_cast<std::uint32_t>(p->manifest.group_of(e));
      for (std::uint32_t i = 0; i < items.size(); ++i) {
        if (!items[i].is_group || items[i].index != g || !p->cmap.cut(i)) continue;
        for (const auto& mem : p->manifest.groups[g].members) {
          if (mem.entry != e) continue;
          for (const ChunkPart& run : p->cmap.parts[i])
            if (run.off == mem.offset) {
              re.stage_ptr = reinterpret_cast<std::uint64_t>(p->group_bufs[g]->p) + mem.offset;
              re.stage_chunk0 = p->cmap.chunk0[i] + run.first;
              re.stage_chunk_len = run.chunk_len;
              re.group_item = i;
            }
        }
      }
    }
    rd.push_back(std::move(re));
  }
  if (Status s = plan_reshard(rd, rs->srcs, &rs->plan); !ok(s)) return s;
  // Gathered source items land in library staging, behind the reader's own
  // chunk range (batch aligned), verified against the source chunk digests.
  rs->own_chunks = p->cmap.n_chunks();
  if (Status s = build_gathers(sh, *rs); !ok(s)) return s;
  const std::uint32_t extra = rs->gather_chunks_end - rs->own_chunks;
  if (Status s = alloc_tables(sh, *p, extra); !ok(s)) return s;
  RS_CUDA(cudaStreamSynchronize(sh.stream));
  p->reshard = std::move(rs);
  p->epoch = ++sh.epoch_ctr;
  sh.holding = std::move(p);
  sh.partial_version = v;
  return Status::ok;
}

Status Client::bind_all(const std::vector<Assignment>& as, VersionId v) {
  if (as.size() != num_shards_) return Status::protocol_error;
  for (std::uint32_t i = 0; i < num_shards_; ++i) {
    if (!is_local(i)) continue;
    if (as[i].version != v) return Status::protocol_error;
    Status s = as[i].reshard ? bind_reshard(shards_[i], as[i], v) : bind(shards_[i], as[i], v);
    if (!ok(s)) return s;
  }
  // The incoming version overwrites registered regions in place: until every
  // shard verifies, this replica holds no coherent version.
  current_.reset();
  published_ = false;
  for (auto& sh : shards_)
    if (sh.device >= 0) serve(sh, v, false);
  return Status::ok;
}

namespace {
using WriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteValue32Fn write_value32() {
  static WriteValue32Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<WriteValue32Fn>(nullptr);
    return reinterpret_cast<WriteValue32Fn>(f);
  }();
  return fn;
}
bool host_dma_enabled() {
  static const bool on = !(std::getenv("RSB_HOST_DMA") && std::getenv("RSB_HOST_DMA")[0] == '0');
  return on;
}
// watermark batches per copy-engine frame: 1 << shift (RSB_DMA_SHIFT)
std::uint32_t dma_frame_shift() {
  static const std::uint32_t v = [] {
    const char* e = std::getenv("RSB_DMA_SHIFT");
    return e ? static_cast<std::uint32_t>(std::atoi(e)) : 10u;  // 128 MiB at 4 KiB chunks: 54.9 GB/s (64: 52.1)
  }();
  return v;
}
}  // namespace

Status Client::launch_host_dma(Shard& sh, const SourceView& src, std::uint32_t* epoch) {
  // Land a complete host-memory source (a retention offload) with the copy
  // engine, frame by frame, straight into the landing regions; each frame
  // raises its flag (cuStreamWriteValue32, no SM needed while the pull
  // kernel holds them all).  The pull kernel then runs as a hash pass over
  // the landed bytes, chasing those flags: PCIe at the copy engine's rate
  // (55.6 GB/s H2D measured) instead of SM reads of host memory (51).
  const auto& p = *sh.holding;
  const ChunkMap& cm = p.cmap;
  const std::uint32_t frames = (cm.n_batches() + (1u << dma_frame_shift()) - 1) >> dma_frame_shift();
  if (!sh.dma) RS_CUDA(cudaStreamCreateWithFlags(&sh.dma, cudaStreamNonBlocking));
  if (!sh.dma_flags.p || sh.dma_flags.n < std::size_t(frames) * 4) {
    if (Status s = sh.dma_flags.alloc(sh.device, std::size_t(frames) * 4); !ok(s)) return s;
    RS_CUDA(cudaMemset(sh.dma_flags.p, 0, sh.dma_flags.n));  // before any fill reads it
    sh.dma_epoch = 0;
  }
  *epoch = ++sh.dma_epoch;
  RS_CUDA(cudaStreamWaitEvent(sh.dma, sh.ev0, 0));  // the fill's clock starts first
  auto* flags = static_cast<std::uint32_t*>(sh.dma_flags.p);
  auto wv = write_value32();
  std::uint32_t cur = 0;  // frames below `cur` are flagged
  auto flag_until = [&](std::uint32_t f) -> Status {
    for (; cur < f; ++cur)
      if (wv(reinterpret_cast<CUstream>(sh.dma), reinterpret_cast<CUdeviceptr>(flags + cur), *epoch, 0) !=
          CUDA_SUCCESS)
        return Status::transfer_failed;
    return Status::ok;
  };
  const auto& items = p.manifest.items();
  for (std::size_t i = 0; i < items.size(); ++i) {
    const std::uint64_t len = items[i].length;
    const std::uint64_t per_batch = std::uint64_t(dev::kBatchChunks) * cm.chunk_len[i];
    const std::uint32_t b0 = cm.chunk0[i] / dev::kBatchChunks;
    for (std::uint64_t off = 0; off < len;) {
      const std::uint32_t b = b0 + static_cast<std::uint32_t>(off / per_batch);
      const std::uint32_t f = b >> dma_frame_shift();
      if (Status s = flag_until(f); !ok(s)) return s;
      const std::uint64_t frame_end_b = std::uint64_t(f + 1) << dma_frame_shift();  // first batch of the next frame
      const std::uint64_t end = std::min<std::uint64_t>(len, (frame_end_b - b0) * per_batch);
      RS_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(p.item_ptrs[i] + off),
                              reinterpret_cast<const void*>(src.item_ptrs[i] + off), end - off,
                              cudaMemcpyHostToDevice, sh.dma));
      off = end;  // payload bytes: not in stats_.h2d_bytes (plans and tables), as on the SM path
    }
  }
  return flag_until(frames);
}

Status Client::launch_fill(Shard& sh, const SourceView& src, bool src_complete) {
  DeviceGuard g(sh.device);
  const auto& p = *sh.holding;
  const auto& items = p.manifest.items();
  std::vector<dev::ItemDesc> descs;
  bool any_cast = false;
  for (std::size_t i = 0; i < items.size(); ++i) {
    const std::size_t at = descs.size();
    append_identity(&descs, src.item_ptrs[i], p.item_ptrs[i], items[i].length, p.cmap, i);
    if (!items[i].is_group &&
        sh.regs[sh.by_name.at(p.manifest.entries[items[i].index].name)].cast) {
      descs[at].chunk_len |= dev::kCastE4M3;  // a big item: one run
      any_cast = true;
    }
  }
  dev::SrcDesc sdesc{reinterpret_cast<const std::uint64_t*>(src.digests),
                     src_complete ? nullptr : reinterpret_cast<const std::uint32_t*>(src.flags),
                     src.epoch, 0};
  const bool remote = src.device != sh.device;
  // A complete source in host memory lands through the copy engine (no cast:
  // the engine cannot convert); the kernel verifies the landed bytes in place.
  // A resumed epoch (landed_some: an earlier attempt verified some batches)
  // takes the SM path, which skips the landed batches: the engine would copy
  // every frame again, over bytes already verified, and nothing re-checks them.
  // (Copy-engine frames cut items at uniform chunk boundaries: a member-cut
  // group takes the SM path too.)
  const bool dma = src.device < 0 && src_complete && !any_cast && !p.landed_some &&
                   !p.cmap.any_cut() && host_dma_enabled() && write_value32();
  if (dma) {
    for (std::size_t i = 0; i < items.size(); ++i) {
      descs[i].src = p.item_ptrs[i];
      descs[i].dst = 0;  // hash-only over the landed bytes
    }
    sdesc.flags = static_cast<const std::uint32_t*>(nullptr);  // set below, after the copies are queued
    sdesc.flag_shift = dma_frame_shift();
  }
  // link class of the source (schedule order, kernel path): 0 local HBM,
  // 1 host memory, 2 + d peer device d
  const std::uint32_t link = dma || !remote ? 0u : src.device < 0 ? 1u : static_cast<std::uint32_t>(src.device + 2);
  for (auto& d : descs) d.pad = link;
  RS_CUDA(cudaEventRecord(sh.ev0, sh.stream));
  if (dma) {
    std::uint32_t epoch = 0;
    sh.dma_fill = true;  // wait_shards drains sh.dma before anything else touches the regions
    if (Status s = launch_host_dma(sh, src, &epoch); !ok(s)) {
      cudaStreamSynchronize(sh.dma);
      sh.dma_fill = false;
      return s;
    }
    sdesc.flags = static_cast<const std::uint32_t*>(sh.dma_flags.p);
    sdesc.epoch = epoch;
  }
  dev::PullParams pp{};
  RS_CUDA(dev::upload_pull_plan(sh.device, sh.stream, descs.data(),
                                static_cast<std::uint32_t>(descs.size()), &sdesc, 1,
                                p.cmap.n_chunks(), &sh.plan, &pp));
  stats_.h2d_bytes += sh.plan.h2d_bytes;
  pp.dst_digests = static_cast<std::uint64_t*>(p.digests.p);
  pp.dst_flags = static_cast<std::uint32_t*>(p.flags.p);
  pp.dst_epoch = p.epoch;
  pp.timeout_ns = static_cast<std::uint64_t>(cfg_.pull_timeout_s * 1e9);
  pp.resume = p.landed_some ? 1u : 0u;
  // 2: a plain peer pull (no cast, the chain's hops): the kernel shape that
  // releases every verified batch at once, so a chaser downstream sees it sooner
  pp.remote = dma || !remote ? 0u : (src.device >= 0 && !any_cast) ? 2u : 1u;
  sh.t_launch = std::chrono::steady_clock::now();
  int ctas = grid(sh);
  if (pp.remote == 2) {  // A/B knob: CTAs of a plain peer pull (chain hop)
    static const int peer_grid = [] {
      const char* e = std::getenv("RSB_PEER_GRID");
      return e ? std::atoi(e) : 0;
    }();
    if (peer_grid > 0) ctas = std::min(ctas, peer_grid);
  }
  RS_CUDA(dev::launch_pull(pp, ctas, sh.stream));
  stats_.kernel_launches += dev::pull_has_work(pp) ? 1 : 0;
  // A fill fed over TCP waits on progress that may need this GPU's copy
  // engines (a StreamServer in this process staging a frame D2H).  Nothing
  // is queued behind its kernel: an event record or copy waiting on the
  // kernel can hold a hardware work queue that the server's copy shares,
  // and that copy would then wait for the kernel that waits for it (seen
  // with 4 connections and reader + server on one GPU: the frame moved only
  // when the kernel timed out).  wait_shards times it on the host.
  if (!sh.tcp) RS_CUDA(cudaEventRecord(sh.ev1, sh.stream));
  sh.holding->landed_some = true;
  // the group unpack queued right behind the fill (skipped on the device
  // if the fill fails); a TCP-fed fill has nothing queued behind it
  sh.unpack_queued = false;
  if (!sh.tcp && !sh.holding->manifest.groups.empty()) {
    auto* code = &reinterpret_cast<dev::PullStatus*>(static_cast<std::uint8_t*>(sh.plan.scratch) + 64)->code;
    if (Status s = queue_unpack(sh, code); !ok(s)) return s;
    sh.unpack_queued = true;
  }
  return Status::ok;
}

std::vector<Client::FillOutcome> Client::fill_shards(const std::vector<Assignment>& as,
                                                     const std::vector<std::uint32_t>& which) {
  launch_shards(as, which);
  return wait_shards(which);
}

void Client::launch_shards(const std::vector<Assignment>& as,
                           const std::vector<std::uint32_t>& which) {
  launch_out_.assign(num_shards_, FillOutcome{});
  launched_.assign(num_shards_, false);
  auto& out = launch_out_;
  auto& launched = launched_;
  if (launch_as_.size() != num_shards_) launch_as_.resize(num_shards_);
  for (std::uint32_t i : which) {
    Shard& sh = shards_[i];
    const Assignment& a = as[i];
    launch_as_[i] = a;
    if (sh.holding && sh.holding->reshard) {
      Status s = a.reshard ? launch_reshard_fill(sh, a, a.source_complete)
                           : Status::protocol_error;
      if (!ok(s)) {
        out[i] = {s, 0, 0};
        continue;
      }
      launched[i] = true;
      continue;
    }
    SourceView view;
    Status s;
    const bool off_box = a.source_endpoint.rfind("tcp:", 0) == 0;
    if (off_box) {
      // off-box source: its stream lands in pinned host memory and the pull
      // kernel chases the host watermarks the receiver raises (stream.hpp)
      sh.tcp = std::make_shared<StreamSource>();
      s = sh.tcp->open(a.source_endpoint, ServeRegistry::key(model_, a.source_replica, sh.idx),
                       a.version, cfg_.pull_timeout_s, &host_pool_);
      if (ok(s)) view = sh.tcp->view();
    } else {
      s = resolve_source(sh, a, a.version, &view, cfg_.pull_timeout_s);
    }
    // Every replica of a cluster digests with the same chunk size; a source
    // cut differently cannot be verified chunk-by-chunk.
    if (ok(s) && !(view.cmap == sh.holding->cmap)) s = Status::protocol_error;
    if (!ok(s)) {
      if (sh.tcp) sh.tcp->release(&host_pool_);
      sh.tcp.reset();
      out[i] = {s, 0, 0};
      continue;
    }
    s = launch_fill(sh, view, off_box ? false : a.source_complete);
    if (!ok(s)) {
      out[i] = {s, 0, 0};
      continue;
    }
    launched[i] = true;
  }
}

void Client::report_progress(Shard& sh) {
  if (!sh.holding || sh.holding->reshard || !sh.holding->flags.p) return;
  const Payload& p = *sh.holding;
  const ChunkMap& cm = p.cmap;
  const std::uint32_t nb = cm.n_batches();
  if (sh.reported + 1 >= cm.chunk0.size()) return;
  DeviceGuard g(sh.device);
  if (!sh.poll && cudaStreamCreateWithFlags(&sh.poll, cudaStreamNonBlocking) != cudaSuccess) return;
  // a window of watermarks from the first item not reported yet (items are
  // verified front to back only as a prefix: the first item with a batch
  // below the epoch ends it), so a poll reads KBs, not the whole table
  const std::uint32_t w0 = cm.chunk0[sh.reported] / dev::kBatchChunks;
  const std::uint32_t first_nb = (cm.count[sh.reported] + dev::kBatchChunks - 1) / dev::kBatchChunks;
  const std::uint32_t wn = std::min<std::uint32_t>(nb - w0, std::max<std::uint32_t>(8192, first_nb));
  sh.flag_host.resize(wn);
  if (wn == 0 ||
      cudaMemcpyAsync(sh.flag_host.data(), static_cast<const std::uint32_t*>(p.flags.p) + w0,
                      std::size_t(wn) * 4, cudaMemcpyDeviceToHost, sh.poll) != cudaSuccess ||
      cudaStreamSynchronize(sh.poll) != cudaSuccess)
    return;
  stats_.d2h_bytes += std::size_t(wn) * 4;
  std::uint64_t items = sh.reported;
  for (std::size_t i = items; i + 1 < cm.chunk0.size(); ++i) {
    const std::uint32_t b0 = cm.chunk0[i] / dev::kBatchChunks;
    const std::uint32_t n = (cm.count[i] + dev::kBatchChunks - 1) / dev::kBatchChunks;
    if (b0 + n > w0 + wn) break;  // beyond the window: the next poll
    bool done = true;
    for (std::uint32_t b = b0; b < b0 + n && done; ++b) done = sh.flag_host[b - w0] == p.epoch;
    if (!done) break;
    items = i + 1;
  }
  if (items > sh.reported) {
    sh.reported = items;
    reg_->progress(model_, replica_, sh.idx, items);
  }
}

Status Client::progress(std::uint32_t shard, std::uint32_t* batches_done, std::uint32_t* n_batches) {
  if (shard >= num_shards_ || !is_local(shard)) return Status::invalid_argument;
  Shard& sh = shards_[shard];
  *batches_done = 0;
  *n_batches = sh.holding ? sh.holding->cmap.n_batches() : 0;
  if (!sh.plan.scratch || shard >= launched_.size() || !launched_[shard]) return Status::ok;
  DeviceGuard g(sh.device);
  if (!sh.poll) RS_CUDA(cudaStreamCreateWithFlags(&sh.poll, cudaStreamNonBlocking));
  // the running kernel's status word, read on a side stream (copy engine)
  auto* status = reinterpret_cast<dev::PullStatus*>(static_cast<std::uint8_t*>(sh.plan.scratch) + 64);
  std::uint32_t v = 0;
  RS_CUDA(cudaMemcpyAsync(&v, &status->batches_done, 4, cudaMemcpyDeviceToHost, sh.poll));
  RS_CUDA(cudaStreamSynchronize(sh.poll));
  *batches_done = v;
  report_progress(sh);
  return Status::ok;
}

std::vector<Client::FillOutcome> Client::wait_shards(const std::vector<std::uint32_t>& which) {
  std::vector<FillOutcome> out = launch_out_;
  if (out.size() != num_shards_) out.assign(num_shards_, FillOutcome{});
  std::vector<bool> launched = launched_;
  if (launched.size() != num_shards_) launched.assign(num_shards_, false);
  std::vector<dev::PullStatus> st(num_shards_);
  stats_.fill_max_ms = stats_.fill_sum_ms = 0;
  stats_.fill_bytes = 0;
  PhaseClock wc;
  for (std::uint32_t i : which) {
    if (!launched[i]) continue;
    Shard& sh = shards_[i];
    DeviceGuard g(sh.device);
    auto* status = reinterpret_cast<dev::PullStatus*>(static_cast<std::uint8_t*>(sh.plan.scratch) + 64);
    const bool tcp = sh.tcp != nullptr;
    float host_ms = 0;
    if (tcp) {  // nothing queued behind the kernel (launch_fill): wait, then read
      cudaStreamSynchronize(sh.stream);
      host_ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - sh.t_launch).count();
    } else if (!sh.holding->reshard) {
      // Spin on the fill's end event; a fill still running after 10 ms
      // reports its verified item prefix to the registry every 10 ms
      // (task_progress), so the replica's view advances while it lands.
      auto next = sh.t_launch + std::chrono::milliseconds(10);
      while (cudaEventQuery(sh.ev1) == cudaErrorNotReady) {
        const auto now = std::chrono::steady_clock::now();
        if (now >= next) {
          report_progress(sh);
          next = now + std::chrono::milliseconds(10);
        }
        std::this_thread::yield();
      }
    }
    cudaMemcpyAsync(&st[i], status, sizeof(dev::PullStatus), cudaMemcpyDeviceToHost, sh.stream);
    cudaError_t e = cudaStreamSynchronize(sh.stream);
    stats_.d2h_bytes += sizeof(dev::PullStatus);
    Status net = Status::ok;
    if (sh.tcp) {
      net = sh.tcp->finish(e == cudaSuccess && st[i].code == dev::kPullOk);
      if (std::getenv("RSB_DEBUG") && st[i].code != dev::kPullOk) {
        auto fs = sh.tcp->flag_summary();
        std::fprintf(stderr, "[rsb] tcp source: %u of %u watermarks set, first missing %u, %llu bytes\n",
                     fs.first, sh.tcp->view().cmap.n_batches(), fs.second,
                     static_cast<unsigned long long>(sh.tcp->bytes_received()));
      }
      sh.tcp->release(&host_pool_);
      sh.tcp.reset();
    }
    if (sh.dma_fill) {
      // Copy-engine frames of a host-fed fill: a kernel that stopped early
      // (bad chunk, timeout) leaves frames queued on sh.dma.  Drain them
      // before a retry lands anything (possibly from another source, on
      // sh.stream) and before the lane's pinned buffer can be released.
      if (cudaStreamSynchronize(sh.dma) != cudaSuccess && e == cudaSuccess) e = cudaErrorUnknown;
      sh.dma_fill = false;
    }
    if (e == cudaSuccess && !ok(net) && st[i].code == dev::kPullOk) st[i].code = dev::kPullNotServing;
    if (std::getenv("RSB_DEBUG") && (st[i].code != dev::kPullOk || e != cudaSuccess))
      std::fprintf(stderr, "[rsb] %s shard %u fill: code %u bad_chunk %u (source batch %u flag %u) net %d cuda %d\n",
                   replica_.c_str(), i, st[i].code, st[i].bad_chunk,
                   static_cast<unsigned>(st[i].pad >> 32), static_cast<unsigned>(st[i].pad & 0xffffffffu),
                   static_cast<int>(net), static_cast<int>(e));
    if (e != cudaSuccess) {
      out[i] = {Status::transfer_failed, 0, 0};
      continue;
    }
    float ms = host_ms;
    if (!tcp) cudaEventElapsedTime(&ms, sh.ev0, sh.ev1);
    stats_.last_pull_ms = ms;
    stats_.last_pull_bytes = st[i].bytes;
    stats_.fill_max_ms = std::max(stats_.fill_max_ms, ms);
    stats_.fill_sum_ms += ms;
    stats_.fill_bytes += st[i].bytes;
    stats_.last_pull_launches = 1;
    // Stats (client_core.hpp:44-52): a local seed consumption is a local
    // copy, not a pull; a pull over the cross-datacenter link counts twice
    const auto& la = i < launch_as_.size() ? launch_as_[i] : std::optional<Assignment>{};
    if (la && la->local_seed_consume) {
      stats_.bytes_copied_local += st[i].bytes;
    } else {
      stats_.bytes_pulled += st[i].bytes;
      if (la && la->cross_dc) stats_.bytes_pulled_cross_dc += st[i].bytes;
    }
    stats_.checksum_failures += st[i].retried_batches;
    switch (st[i].code) {
      case dev::kPullOk:
        out[i] = {Status::ok, 0, 0};
        break;
      case dev::kPullChecksum:
        stats_.checksum_failures += 1;
        out[i] = {Status::checksum_mismatch, 1, st[i].bad_chunk};
        break;
      case dev::kPullTimeout:
        out[i] = {Status::timeout, 0, st[i].bad_chunk};
        break;
      default:
        out[i] = {Status::not_serving, 0, st[i].bad_chunk};
        break;
    }
  }
  wc.mark("wait kernels");
  // Unpack verified groups into their members (K3, unpack_group); a reshard
  // fill instead slices the gathered items and packs its own groups.
  for (std::uint32_t i : which) {
    if (!ok(out[i].status)) continue;
    Shard& sh = shards_[i];
    if (sh.holding->reshard) continue;  // its follow-up ran behind the fill (launch_reshard_fill)
    if (sh.unpack_queued) continue;     // queued behind the fill; the status read synchronized it
    if (sh.holding->manifest.groups.empty()) continue;
    if (Status s = queue_unpack(sh, nullptr); !ok(s)) out[i] = {s, 0, 0};
    if (cudaStreamSynchronize(sh.stream) != cudaSuccess) out[i] = {Status::transfer_failed, 0, 0};
  }
  return out;
}

Status Client::copy_spans(Shard& sh, const std::vector<std::uint64_t>& srcs,
                          const std::vector<std::uint64_t>& dsts,
                          const std::vector<std::uint64_t>& lens,
                          const std::uint32_t* guard, DevBuf* table,
                          std::vector<std::uint64_t>* last) {
  // Stream-ordered: returns once the copy is queued on sh.stream (callers
  // synchronize).  The span tables live in sh.span_tables; a later call's
  // upload is ordered behind this call's kernel on the same stream.
  if (srcs.empty()) return Status::ok;
  DeviceGuard g(sh.device);
  DevBuf& t = table ? *table : sh.span_tables;
  const std::size_t n = srcs.size();
  std::vector<std::uint64_t> host(4 * n);
  std::uint64_t tiles = 0;
  for (std::size_t i = 0; i < n; ++i) {
    host[i] = srcs[i];
    host[n + i] = dsts[i];
    host[2 * n + i] = lens[i];
    host[3 * n + i] = tiles;
    tiles += dev::copy_span_tiles(lens[i]);
  }
  const bool same = last && *last == host && t.p && t.n >= 4 * n * 8;
  if (!same) {
    if (Status s = t.alloc(sh.device, 4 * n * 8); !ok(s)) return s;
    RS_CUDA(cudaMemcpyAsync(t.p, host.data(), 4 * n * 8, cudaMemcpyHostToDevice, sh.stream));
    stats_.h2d_bytes += 32 * n;
    if (last) *last = std::move(host);
  }
  auto* d = static_cast<std::uint64_t*>(t.p);
  RS_CUDA(dev::launch_copy_spans(d, d + n, d + 2 * n, d + 3 * n, static_cast<int>(n), tiles,
                                 sh.stream, guard));
  ++stats_.kernel_launches;
  return Status::ok;
}

Status Client::queue_unpack(Shard& sh, const std::uint32_t* guard) {
  const auto& p = *sh.holding;
  std::vector<std::uint64_t> srcs, dsts, ls;
  for (std::size_t gi = 0; gi < p.manifest.groups.size(); ++gi)
    for (const auto& mem : p.manifest.groups[gi].members) {
      srcs.push_back(reinterpret_cast<std::uint64_t>(p.group_bufs[gi]->p) + mem.offset);
      const Reg& r = sh.regs[sh.by_name.at(p.manifest.entries[mem.entry].name)];
      dsts.push_back(reinterpret_cast<std::uint64_t>(r.ptr));
      ls.push_back(p.manifest.entries[mem.entry].length | (r.cast ? dev::kSpanCastE4M3 : 0));
    }
  return copy_spans(sh, srcs, dsts, ls, guard, &sh.unpack_tables, &sh.unpack_last);
}

Status Client::resolve_shard(Shard& sh, const std::string& replica, std::uint32_t shard,
                             VersionId v, SourceView* out) {
  auto deadline =
      std::chrono::steady_clock::now() + std::chrono::duration<double>(cfg_.pull_timeout_s);
  const std::string k = ServeRegistry::key(model_, replica, shard);
  for (;;) {
    auto st = serves_->is_silent(k) ? nullptr : serves_->find(k);
    if (st) {
      bool ready;
      {
        std::lock_guard lk(st->m);
        ready = st->serving && st->version == v && !st->cmap.chunk0.empty();
      }
      if (ready) return map_source(st, sh.device, out);
    }
    if (std::chrono::steady_clock::now() > deadline) return Status::not_serving;
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

Status Client::build_gathers(Shard& sh, Reshard& rs) {
  // Gathered source items (groups, unaligned slices) land in staging, but
  // only the watermark batches that hold bytes some slice copy reads: a
  // reader shard that needs a few members of a packed group does not pull
  // (and verify) the rest of it.  Each range is whole batches of the item
  // (cut at chunk-run boundaries), and the staging holds only those ranges,
  // packed: a window per run of adjacent ranges (item offset -> staging
  // offset), so a 64 MiB group whose biases and norms are needed costs
  // their batches, not 64 MiB.  A function of the plan: built once per bind,
  // re-addressed onto the sources' mappings per launch.
  rs.gather_segs.clear();
  rs.gather_items.clear();
  rs.gather_windows.assign(rs.plan.gathers.size(), {});
  rs.gather_bufs.clear();
  std::map<std::pair<std::uint32_t, std::uint32_t>, std::vector<std::pair<std::uint64_t, std::uint64_t>>> need_bytes;
  for (const auto& c : rs.plan.copies)
    need_bytes[{c.src_shard, c.src_item}].emplace_back(c.src_off,
                                                      c.src_off + (c.rows - 1) * c.src_stride + c.nc);
  std::uint32_t next = rs.own_chunks;
  for (std::size_t gi = 0; gi < rs.plan.gathers.size(); ++gi) {
    const auto& gth = rs.plan.gathers[gi];
    const SourceShard& ss = rs.srcs[gth.src_shard];
    const auto& it = ss.manifest.items()[gth.src_item];
    // the item's chunk runs (one for a uniform item; one per member of a
    // member-cut group)
    std::vector<ChunkPart> runs;
    if (gth.src_item < ss.parts.size() && !ss.parts[gth.src_item].empty())
      runs = ss.parts[gth.src_item];
    else
      runs.push_back(ChunkPart{0, it.length, ss.layout.chunk_len[gth.src_item], 0});
    auto run_chunks = [](const ChunkPart& r) {
      return static_cast<std::uint32_t>((r.len + r.chunk_len - 1) / r.chunk_len);
    };
    const std::uint32_t n = runs.back().first + run_chunks(runs.back());
    const std::uint32_t nb = (n + dev::kBatchChunks - 1) / dev::kBatchChunks;
    auto chunk_at = [&](std::uint64_t x) {  // the chunk holding byte x of the item
      auto r = std::upper_bound(runs.begin(), runs.end(), x,
                                [](std::uint64_t v, const ChunkPart& p) { return v < p.off; });
      --r;
      return r->first + static_cast<std::uint32_t>((x - r->off) / r->chunk_len);
    };
    std::vector<char> want(nb, 0);
    auto nit = need_bytes.find({gth.src_shard, gth.src_item});
    if (nit == need_bytes.end()) {
      std::fill(want.begin(), want.end(), 1);
    } else {
      for (const auto& [lo, hi] : nit->second)
        for (std::uint32_t b = chunk_at(lo) / dev::kBatchChunks;
             b <= chunk_at(hi - 1) / dev::kBatchChunks && b < nb; ++b)
          want[b] = 1;
    }
    std::uint64_t packed = 0;  // staging bytes so far
    const std::size_t seg0 = rs.gather_segs.size();
    for (std::uint32_t b0 = 0; b0 < nb;) {
      if (!want[b0]) {
        ++b0;
        continue;
      }
      std::uint32_t b1 = b0;
      while (b1 < nb && want[b1]) ++b1;
      const std::uint32_t k0 = b0 * dev::kBatchChunks, k1 = std::min(n, b1 * dev::kBatchChunks);
      // one window per run of wanted batches: its ranges are adjacent in the item
      std::uint64_t win_lo = ~0ull, win_base = (packed + 255) / 256 * 256;
      for (const ChunkPart& r : runs) {  // whole batches, cut at run boundaries
        const std::uint32_t rk0 = std::max(k0, r.first), rk1 = std::min(k1, r.first + run_chunks(r));
        if (rk0 >= rk1) continue;
        const std::uint64_t off = r.off + std::uint64_t(rk0 - r.first) * r.chunk_len;
        const std::uint64_t end = std::min<std::uint64_t>(r.off + r.len,
                                                          r.off + std::uint64_t(rk1 - r.first) * r.chunk_len);
        if (win_lo == ~0ull) win_lo = off;
        dev::ItemDesc d{};
        d.src = off;                         // + the source item's address at launch
        d.dst = win_base + (off - win_lo);   // + the staging's address below
        d.len = end - off;
        d.chunk0 = next + rk0;
        d.chunk_len = r.chunk_len;
        d.src_chunk0 = ss.chunk0[gth.src_item] + rk0;
        d.q = d.m = 1;
        d.src_id = gth.src_shard;
        rs.gather_segs.push_back(d);
        rs.gather_items.push_back(gth.src_item);
        packed = win_base + (end - win_lo);
      }
      if (win_lo != ~0ull) rs.gather_windows[gi].push_back({win_lo, win_lo + (packed - win_base), win_base});
      b0 = b1;
    }
    auto buf = std::make_unique<DevBuf>();
    if (Status s = buf->alloc(sh.device, std::max<std::uint64_t>(packed, 256)); !ok(s)) return s;
    for (std::size_t k = seg0; k < rs.gather_segs.size(); ++k)
      rs.gather_segs[k].dst += reinterpret_cast<std::uint64_t>(buf->p);
    rs.gather_bufs.push_back(std::move(buf));
    next += nb * dev::kBatchChunks;
  }
  rs.gather_chunks_end = next;
  return Status::ok;
}

std::uint64_t Client::Reshard::staged(std::size_t gi, std::uint64_t item_off) const {
  // the staging address of byte item_off of gather gi's source item
  for (const auto& w : gather_windows[gi])
    if (item_off >= w[0] && item_off < w[1])
      return reinterpret_cast<std::uint64_t>(gather_bufs[gi]->p) + w[2] + (item_off - w[0]);
  return 0;  // not landed: the plan never reads it
}

Status Client::launch_reshard_fill(Shard& sh, const Assignment& a, bool src_complete) {
  DeviceGuard g(sh.device);
  PhaseClock pc;
  Payload& p = *sh.holding;
  Reshard& rs = *p.reshard;
  const auto nsrc = static_cast<std::uint32_t>(rs.srcs.size());
  std::vector<SourceView> views(nsrc);
  std::vector<dev::SrcDesc> sd(nsrc);
  std::vector<bool> need(nsrc, false);
  for (const auto& d : rs.plan.segs) need[d.src_id] = true;
  for (const auto& gth : rs.plan.gathers) need[gth.src_shard] = true;
  for (std::uint32_t s = 0; s < nsrc; ++s) {
    if (!need[s]) continue;
    if (Status st = resolve_shard(sh, a.source_replica, s, a.version, &views[s]); !ok(st))
      return st;
    if (views[s].cmap.chunk0 != rs.srcs[s].chunk0) return Status::protocol_error;
    sd[s] = {reinterpret_cast<const std::uint64_t*>(views[s].digests),
             src_complete ? nullptr : reinterpret_cast<const std::uint32_t*>(views[s].flags),
             views[s].epoch, 0};
  }
  pc.mark("reshard fill: resolve sources");
  std::vector<int> src_dev(nsrc, sh.device);
  for (std::uint32_t s = 0; s < nsrc; ++s)
    if (need[s]) src_dev[s] = views[s].device;
  auto link_class = [&](std::uint32_t s) {
    // 0: local HBM, 1: host memory (device -1), 2 + d: peer device d
    return src_dev[s] == sh.device ? 0u : static_cast<std::uint32_t>(src_dev[s] + 2);
  };
  std::vector<dev::ItemDesc> descs = rs.plan.segs;
  for (auto& d : descs) {
    d.src = views[d.src_id].item_ptrs[d.pad] + d.src;
    d.pad = link_class(d.src_id);
  }
  // the gather segments (built at bind, build_gathers) re-addressed onto
  // the sources' current mappings
  for (std::size_t k = 0; k < rs.gather_segs.size(); ++k) {
    dev::ItemDesc d = rs.gather_segs[k];
    d.src += views[d.src_id].item_ptrs[rs.gather_items[k]];
    d.pad = link_class(d.src_id);
    descs.push_back(d);
  }
  const std::uint32_t next = rs.gather_segs.empty() ? rs.own_chunks : rs.gather_chunks_end;
  bool remote = false;
  for (std::uint32_t s = 0; s < nsrc; ++s) remote |= need[s] && src_dev[s] != sh.device;
  dev::PullParams pp{};
  pc.mark("reshard fill: segments");
  RS_CUDA(dev::upload_pull_plan(sh.device, sh.stream, descs.data(),
                                static_cast<std::uint32_t>(descs.size()), sd.data(), nsrc, next,
                                &sh.plan, &pp));
  pc.mark("reshard fill: plan upload");
  stats_.h2d_bytes += sh.plan.h2d_bytes;
  pp.dst_digests = static_cast<std::uint64_t*>(p.digests.p);
  pp.dst_flags = static_cast<std::uint32_t*>(p.flags.p);
  pp.dst_epoch = p.epoch;
  pp.timeout_ns = static_cast<std::uint64_t>(cfg_.pull_timeout_s * 1e9);
  pp.resume = p.landed_some ? 1u : 0u;
  pp.remote = remote ? 1u : 0u;
  RS_CUDA(cudaEventRecord(sh.ev0, sh.stream));
  RS_CUDA(dev::launch_pull(pp, grid(sh), sh.stream));
  stats_.kernel_launches += dev::pull_has_work(pp) ? 1 : 0;
  RS_CUDA(cudaEventRecord(sh.ev1, sh.stream));
  pc.mark("reshard fill: launched");
  p.landed_some = true;
  // the follow-up (slice copies, packing, re-digests) queued right behind the
  // fill, skipped on the device if it fails: no host round trip in between
  auto* code = &reinterpret_cast<dev::PullStatus*>(static_cast<std::uint8_t*>(sh.plan.scratch) + 64)->code;
  Status fs = finish_reshard(sh, code);
  pc.mark("reshard fill: follow-up queued");
  return fs;
}

Status Client::finish_reshard(Shard& sh, const std::uint32_t* guard) {
  Payload& p = *sh.holding;
  Reshard& rs = *p.reshard;
  // 1) slices out of gathered source items (rows of nc bytes)
  std::map<std::pair<std::uint32_t, std::uint32_t>, std::size_t> gidx;
  for (std::size_t gi = 0; gi < rs.plan.gathers.size(); ++gi)
    gidx[{rs.plan.gathers[gi].src_shard, rs.plan.gathers[gi].src_item}] = gi;
  const auto& items = p.manifest.items();
  // A re-digested big item filled entirely by contiguous, chunk-aligned
  // copies is landed by one more pull pass instead (staging -> region,
  // digests computed on the way, watermarks released): one read and one
  // write of its bytes instead of a copy plus a hash pass re-reading them.
  std::vector<dev::ItemDesc> fused;
  std::set<std::uint32_t> fused_items;
  if (!terminal()) {
    std::map<std::uint64_t, std::uint32_t> by_ptr;  // region address -> reader big item
    for (std::uint32_t i : rs.plan.rehash) by_ptr[p.item_ptrs[i]] = i;
    std::map<std::uint32_t, std::vector<std::pair<std::uint64_t, std::uint64_t>>> cover;  // item -> [off, end)
    std::set<std::uint32_t> bad;
    for (const auto& c : rs.plan.copies) {
      auto it = by_ptr.upper_bound(c.dst);
      if (it == by_ptr.begin()) continue;
      --it;
      const std::uint32_t i = it->second;
      const std::uint64_t off = c.dst - it->first, len = c.rows * c.nc, cl = p.cmap.chunk_len[i];
      if (off >= items[i].length) continue;
      const bool contiguous = c.src_stride == c.nc && c.dst_stride == c.nc && !c.cast;
      if (!contiguous || off % cl || (len % cl && off + len != items[i].length)) bad.insert(i);
      cover[i].emplace_back(off, off + len);
    }
    for (auto& [i, v] : cover) {
      if (bad.count(i)) continue;
      std::sort(v.begin(), v.end());
      std::uint64_t at = 0;
      for (const auto& [a, b] : v) at = a == at ? b : ~0ull;
      if (at == items[i].length) fused_items.insert(i);  // copies cover the item exactly
    }
  }
  // region address of each of this reader's packed members -> (region end,
  // the member's address in its group staging)
  std::map<std::uint64_t, std::pair<std::uint64_t, std::uint64_t>> member_at;
  for (std::uint32_t i = 0; i < items.size(); ++i) {
    if (!items[i].is_group) continue;
    for (const auto& mem : p.manifest.groups[items[i].index].members) {
      const auto ptr = reinterpret_cast<std::uint64_t>(sh.regs[mem.entry].ptr);
      member_at[ptr] = {ptr + sh.regs[mem.entry].len,
                        reinterpret_cast<std::uint64_t>(p.group_bufs[items[i].index]->p) + mem.offset};
    }
  }
  std::vector<std::uint64_t> srcs, dsts, lens;
  for (const auto& c : rs.plan.copies) {
    const std::size_t gi = gidx.at({c.src_shard, c.src_item});
    const std::uint64_t at = rs.staged(gi, c.src_off);  // the copy's first byte in staging
    if (!at) return Status::protocol_error;
    const std::uint64_t base = at - c.src_off;  // item offsets inside this copy's window
    if (!fused_items.empty()) {
      auto it = std::find_if(fused_items.begin(), fused_items.end(), [&](std::uint32_t i) {
        return c.dst >= p.item_ptrs[i] && c.dst < p.item_ptrs[i] + items[i].length;
      });
      if (it != fused_items.end()) {
        const std::uint32_t i = *it;
        const std::uint64_t off = c.dst - p.item_ptrs[i], cl = p.cmap.chunk_len[i];
        dev::ItemDesc d{};
        d.src = base + c.src_off;
        d.dst = c.dst;
        d.len = c.rows * c.nc;
        d.chunk0 = p.cmap.chunk0[i] + static_cast<std::uint32_t>(off / cl);
        d.chunk_len = static_cast<std::uint32_t>(cl);
        d.q = d.m = 1;
        fused.push_back(d);
        continue;
      }
    }
    const std::uint64_t flag = c.cast ? dev::kSpanCastE4M3 : 0;
    // 2) a slice of one of this reader's own packed members lands in its
    //    group staging too (the group re-served by this copy), copied from
    //    the same source bytes in the same launch: members are only ever
    //    filled by copies (plan_reshard), so no separate packing pass
    std::uint64_t also = 0;  // staging address of c.dst, or 0
    if (!terminal()) {
      auto mt = member_at.upper_bound(c.dst);
      if (mt != member_at.begin() && c.dst < (--mt)->second.first)
        also = mt->second.second + (c.dst - mt->first);
    }
    auto add = [&](std::uint64_t src, std::uint64_t dst, std::uint64_t len) {
      srcs.push_back(src);
      dsts.push_back(dst);
      lens.push_back(len | flag);
      if (also) {
        srcs.push_back(src);
        dsts.push_back(also + (dst - c.dst));
        lens.push_back(len);
      }
    };
    if (c.src_stride == c.nc && c.dst_stride * (c.cast ? 2 : 1) == c.nc) {
      add(base + c.src_off, c.dst, c.rows * c.nc);  // whole rows on both sides: one contiguous span
      continue;
    }
    for (std::uint64_t r = 0; r < c.rows; ++r)
      add(base + c.src_off + r * c.src_stride, c.dst + r * c.dst_stride, c.nc);
  }
  // groups the fill landed straight into their staging: unpack to the regions
  const std::set<std::uint32_t> direct(rs.plan.direct_groups.begin(), rs.plan.direct_groups.end());
  for (std::uint32_t i : direct)
    for (const auto& mem : p.manifest.groups[items[i].index].members) {
      srcs.push_back(reinterpret_cast<std::uint64_t>(p.group_bufs[items[i].index]->p) + mem.offset);
      dsts.push_back(reinterpret_cast<std::uint64_t>(sh.regs[mem.entry].ptr));
      lens.push_back(sh.regs[mem.entry].len);
    }
  if (Status s = copy_spans(sh, srcs, dsts, lens, guard); !ok(s)) return s;
  if (terminal()) return Status::ok;  // a cast copy never re-serves: nothing to pack or digest
  std::vector<std::uint32_t> group_items;  // re-digested: filled by copies
  for (std::uint32_t i = 0; i < items.size(); ++i)
    if (items[i].is_group && !direct.count(i)) group_items.push_back(i);
  // 3) digest + release the items whose bytes arrived by copy: the groups and
  //    big items sliced out of gathered source items (own chunk table and
  //    watermarks)
  std::vector<std::uint32_t> rehash = group_items;
  for (std::uint32_t i : rs.plan.rehash)
    if (!fused_items.count(i)) rehash.push_back(i);
  std::sort(rehash.begin(), rehash.end());
  if (!fused.empty()) {
    std::sort(fused.begin(), fused.end(),
              [](const dev::ItemDesc& a, const dev::ItemDesc& b) { return a.chunk0 < b.chunk0; });
    DeviceGuard g(sh.device);
    const dev::SrcDesc staging{nullptr, nullptr, 0, 0};  // verified when gathered: compute only
    dev::PullParams pp{};
    RS_CUDA(dev::upload_pull_plan(sh.device, sh.stream, fused.data(), static_cast<std::uint32_t>(fused.size()),
                                  &staging, 1, p.cmap.n_chunks(), &sh.fuse_plan, &pp));
    stats_.h2d_bytes += sh.fuse_plan.h2d_bytes;
    pp.first_batch = fused.front().chunk0 / dev::kBatchChunks;
    pp.dst_digests = static_cast<std::uint64_t*>(p.digests.p);
    pp.dst_flags = static_cast<std::uint32_t*>(p.flags.p);
    pp.dst_epoch = p.epoch;
    pp.timeout_ns = static_cast<std::uint64_t>(cfg_.pull_timeout_s * 1e9);
    pp.guard = guard;
    RS_CUDA(dev::launch_pull(pp, grid(sh), sh.stream));
    stats_.kernel_launches += dev::pull_has_work(pp) ? 1 : 0;
  }
  if (std::getenv("RSB_TIMING")) {
    std::uint64_t gb = 0, cb = 0, rb = 0;
    for (const auto& gbuf : rs.gather_bufs) gb += gbuf->n;
    for (const auto& c : rs.plan.copies) cb += c.rows * c.nc;
    for (auto i : rehash) rb += items[i].length;
    std::fprintf(stderr, "[rsb] finish_reshard shard %u: %zu gathers (%llu B), %zu copies (%llu B), "
                 "%zu group spans, %zu rehash items (%llu B), %zu items landed by copy-hash segments\n",
                 sh.idx, rs.gather_bufs.size(), (unsigned long long)gb, rs.plan.copies.size(),
                 (unsigned long long)cb, srcs.size(), rehash.size(), (unsigned long long)rb, fused_items.size());
  }
  return hash_items(sh, p, rehash, guard);
}

void Client::finish_transfers(VersionId v, bool good) {
  if (good) {
    for (auto& sh : shards_) {
      if (sh.device < 0 || !sh.holding) continue;
      sh.partial_version.reset();
      {
        std::lock_guard lk(sh.serve->m);
        sh.serve->complete = true;
        sh.serve->progress = sh.holding->manifest.items().size();
      }
      stats_.items_verified += sh.holding->manifest.items().size();
    }
    current_ = v;
    published_ = true;
  } else {
    stop_serving();
    current_.reset();
    published_ = false;
  }
}

Status Client::run_replicate_loop(const OpOutcome& o, VersionId v) {
  std::vector<Assignment> as = o.assignments;
  PhaseClock pc;
  Status bs = bind_all(as, v);
  pc.mark("bind");
  if (Status s = bs; !ok(s)) {
    for (std::uint32_t i = 0; i < num_shards_; ++i) reg_->complete(model_, replica_, i, s);
    finish_transfers(v, false);
    return s;
  }
  std::vector<int> reports_left(num_shards_, cfg_.checksum_retries);
  std::vector<std::uint32_t> pending;
  for (std::uint32_t i = 0; i < num_shards_; ++i) pending.push_back(i);
  while (!pending.empty()) {
    launch_shards(as, pending);
    pc.mark("launch");
    auto res = wait_shards(pending);
    pc.mark("wait+finish");
    std::vector<std::uint32_t> next;
    for (std::uint32_t i : pending) {
      if (ok(res[i].status)) {
        reg_->progress(model_, replica_, i, shards_[i].holding->manifest.items().size());
        continue;
      }
      Status fail = res[i].status;
      if (res[i].reason == 1 && reports_left[i]-- <= 0) fail = Status::checksum_mismatch;
      else {
        stats_.failure_reports++;
        auto r = reg_->failure_report(model_, replica_, i, as[i].source_replica, res[i].reason);
        if (r) {
          as[i] = *r;
          next.push_back(i);
          continue;
        }
        fail = r.status();
      }
      for (std::uint32_t j = 0; j < num_shards_; ++j) reg_->complete(model_, replica_, j, fail);
      finish_transfers(v, false);
      return fail;
    }
    pending = std::move(next);
  }
  finish_transfers(v, true);
  for (std::uint32_t i = 0; i < num_shards_; ++i) reg_->complete(model_, replica_, i, Status::ok);
  pc.mark("complete");
  return Status::ok;
}

Status Client::replicate(const VersionSpec& spec, VersionId* out, double wait_s) {
  if (!opened_) {
    if (Status s = open(); !ok(s)) return s;
  }
  PhaseClock pc;
  apply_releases();
  OpOutcome o;
  Status s = reg_->replicate(model_, replica_, spec, &o);
  if (!ok(s)) return s;
  if (!o.done) o = reg_->wait_op(model_, replica_, wait_s);
  if (!o.done) return Status::timeout;
  if (!ok(o.status)) return o.status;
  pc.mark("replicate: registry");
  s = run_replicate_loop(o, *o.version);
  if (ok(s) && out) *out = *o.version;
  return s;
}

Status Client::update(const VersionSpec& spec, bool* changed, VersionId* out, double wait_s) {
  if (!opened_) {
    if (Status s = open(); !ok(s)) return s;
  }
  apply_releases();
  OpOutcome o;
  Status s = reg_->update(model_, replica_, spec, current_, &o);
  if (!ok(s)) return s;
  if (Status so = settle_offload(&o, wait_s); !ok(so)) return so;
  if (!o.done) o = reg_->wait_op(model_, replica_, wait_s);
  if (!o.done) return Status::timeout;
  if (!ok(o.status)) return o.status;
  if (changed) *changed = o.changed;
  if (!o.changed) {
    if (out && o.version) *out = *o.version;
    // still on what we hold; the reply may start a background seed fill
    // (client_core.cpp:1331-1337)
    if (o.seed) return start_seed(*o.seed);
    return Status::ok;
  }
  s = run_replicate_loop(o, *o.version);
  if (ok(s) && out) *out = *o.version;
  return s;
}

Status Client::close() {
  join_finalize();
  join_seed();
  closed_ = true;
  stop_serving();
  for (auto& sh : shards_) serves_->erase(ServeRegistry::key(model_, replica_, sh.idx));
  if (opened_) reg_->close(model_, replica_);
  opened_ = false;
  published_ = false;
  return Status::ok;
}

Result<std::string> Client::manifest_bytes(std::uint32_t shard) {
  if (shard >= num_shards_ || !shards_[shard].holding) return Status::not_found;
  // early publish: the reference-identical bytes, once their digests are in
  if (Status s = adopt_final(shards_[shard], 60.0); !ok(s)) return s;
  return shards_[shard].holding->encoded;
}

Result<std::string> Client::held_manifest(std::uint32_t shard) const {
  if (shard >= num_shards_ || !shards_[shard].holding) return Status::not_found;
  return shards_[shard].holding->encoded;
}

bool Client::publish_pending() const {
  for (const auto& sh : shards_)
    if (sh.device >= 0 && sh.holding && !sh.holding->deferred.empty()) return true;
  return false;
}

Status Client::chunk_digests(std::uint32_t shard, std::vector<std::uint64_t>* out) {
  if (shard >= num_shards_ || !shards_[shard].holding) return Status::not_found;
  Shard& sh = shards_[shard];
  DeviceGuard g(sh.device);
  const ChunkMap& cm = sh.holding->cmap;
  std::vector<std::uint64_t> raw(cm.n_chunks());
  out->clear();
  if (raw.empty()) return Status::ok;
  RS_CUDA(cudaMemcpy(raw.data(), sh.holding->digests.p, raw.size() * 8, cudaMemcpyDeviceToHost));
  // dense, in item order: the holes between batch-aligned items are skipped
  out->reserve(cm.n_real());
  for (std::size_t i = 0; i < cm.count.size(); ++i)
    out->insert(out->end(), raw.begin() + cm.chunk0[i], raw.begin() + cm.chunk0[i] + cm.count[i]);
  return Status::ok;
}

// ---- retention offload lanes ---------------------------------------------

Status Client::make_retention_lane(Shard& sh, VersionId v, std::string* endpoint) {
  auto it = sh.lanes.find(v);
  if (it != sh.lanes.end()) {  // re-confirm is idempotent
    *endpoint = it->second.endpoint;
    return Status::ok;
  }
  if (!sh.holding || !current_ || *current_ != v) return Status::invalid_state;
  const Payload& p = *sh.holding;
  const auto& items = p.manifest.items();
  // [items, 256-byte aligned][chunk-digest table]
  std::vector<std::uint64_t> off(items.size());
  std::uint64_t tot = 0, bytes = 0;
  for (std::size_t i = 0; i < items.size(); ++i) {
    off[i] = tot;
    tot += (items[i].length + 255) / 256 * 256;
    bytes += items[i].length;
  }
  const std::uint64_t dig_off = tot;
  tot += std::uint64_t(p.cmap.n_chunks()) * 8;
  std::unique_ptr<HostBuf> buf;
  for (auto it = host_pool_.begin(); it != host_pool_.end(); ++it)
    if ((*it)->n >= tot) {
      buf = std::move(*it);
      host_pool_.erase(it);
      break;
    }
  if (!buf) {
    buf = std::make_unique<HostBuf>();
    if (Status s = buf->alloc(tot); !ok(s)) return s;
  }
  auto* base = static_cast<std::uint8_t*>(buf->p);
  {
    DeviceGuard g(sh.device);
    for (std::size_t i = 0; i < items.size(); ++i)
      RS_CUDA(cudaMemcpyAsync(base + off[i], reinterpret_cast<const void*>(p.item_ptrs[i]),
                              items[i].length, cudaMemcpyDeviceToHost, sh.stream));
    if (p.cmap.n_chunks())
      RS_CUDA(cudaMemcpyAsync(base + dig_off, p.digests.p, std::size_t(p.cmap.n_chunks()) * 8,
                              cudaMemcpyDeviceToHost, sh.stream));
    RS_CUDA(cudaStreamSynchronize(sh.stream));
  }
  stats_.bytes_copied_local += bytes;
  Shard::Lane lane;
  lane.key = ServeRegistry::key(model_, replica_ + "+offload@" + std::to_string(v), sh.idx);
  lane.endpoint = "host:" + replica_ + ":" + std::to_string(sh.idx);
  lane.serve = serves_->ensure(lane.key);
  {
    std::vector<std::uint64_t> ends, ptrs;
    for (std::size_t i = 0; i < items.size(); ++i) {
      ends.push_back(items[i].stream_offset + items[i].length);
      ptrs.push_back(reinterpret_cast<std::uint64_t>(base + off[i]));
    }
    std::lock_guard lk(lane.serve->m);
    lane.serve->serving = true;
    lane.serve->imported = false;
    lane.serve->version = v;
    lane.serve->complete = true;
    lane.serve->progress = items.size();
    lane.serve->device = -1;
    lane.serve->pid = static_cast<int>(getpid());
    lane.serve->item_ends = std::move(ends);
    lane.serve->item_ptrs = std::move(ptrs);
    lane.serve->cmap = p.cmap;
    lane.serve->digests = reinterpret_cast<std::uint64_t>(base + dig_off);
    lane.serve->flags = 0;
    lane.serve->epoch = 1;
    lane.serve->host_name = buf->name;
    lane.serve->host_size = buf->n;
    lane.serve->host_base = reinterpret_cast<std::uint64_t>(base);
  }
  lane.buf = std::move(buf);
  *endpoint = lane.endpoint;
  sh.lanes.emplace(v, std::move(lane));
  return Status::ok;
}

Status Client::make_retention_lanes(VersionId v, std::vector<std::string>* endpoints) {
  endpoints->assign(num_shards_, "");
  for (auto& sh : shards_) {
    if (sh.device < 0) continue;
    if (Status s = make_retention_lane(sh, v, &(*endpoints)[sh.idx]); !ok(s)) return s;
  }
  return Status::ok;
}

Result<std::string> Client::export_lane(std::uint32_t shard, VersionId v) {
  if (shard >= num_shards_) return Status::invalid_argument;
  auto it = shards_[shard].lanes.find(v);
  if (it == shards_[shard].lanes.end()) return Status::not_found;
  return serves_->export_state(it->second.key);
}

void Client::release_lane(VersionId v) {
  for (auto& sh : shards_) {
    auto it = sh.lanes.find(v);
    if (it == sh.lanes.end()) continue;
    {
      std::lock_guard lk(it->second.serve->m);
      it->second.serve->serving = false;
    }
    serves_->erase(it->second.key);
    if (host_pool_.size() < 2) host_pool_.push_back(std::move(it->second.buf));
    sh.lanes.erase(it);  // a buffer not pooled is unregistered and unlinked
  }
}

void Client::apply_releases() {
  for (const auto& r : reg_->take_releases(model_, replica_)) {
    if (r.seed) release_seed_lane(r.version);
    else release_lane(r.version);
  }
}

std::vector<VersionId> Client::lanes() const {
  std::set<VersionId> vs;
  for (const auto& sh : shards_)
    for (const auto& [v, lane] : sh.lanes) vs.insert(v);
  return {vs.begin(), vs.end()};
}

// ---- cross-link seed buffers ----------------------------------------------

Status Client::launch_seed(Shard& sh, const Assignment& a) {
  // start_seed_fill (client_core.cpp:1720-1770): the lane is this replica's
  // serve state "<replica>+seed@<v>", items in pinned host memory (POSIX
  // shm, device-mapped) with its chunk-digest table beside them.  The pull
  // kernel lands the source's bytes there over PCIe, verifying every chunk
  // against the source's table and writing the lane's own.
  if (a.reshard) return Status::invalid_argument;  // seeds hold the source's slicing
  auto mr = Manifest::decode(a.manifest);
  if (!mr) return Status::protocol_error;
  const VersionId v = a.version;
  if (sh.seed_lanes.count(v)) return Status::ok;  // already seeded (start ignored)
  if (Status s = ensure_stream(sh); !ok(s)) return s;
  DeviceGuard g(sh.device);
  const auto& items = mr->items();
  ChunkMap cm = ChunkMap::uniform(*mr, cfg_.chunk_bytes);
  if (!a.layout.empty()) {
    auto lay = ShardLayout::decode(a.layout);
    if (!lay || lay->chunk_len.size() != items.size()) return Status::protocol_error;
    cm = ChunkMap::from_layout(*mr, *lay, cfg_.chunk_bytes, cfg_.reshard_align);
  }
  std::vector<std::uint64_t> off(items.size());
  std::uint64_t tot = 0, bytes = 0;
  for (std::size_t i = 0; i < items.size(); ++i) {
    off[i] = tot;
    tot += (items[i].length + 255) / 256 * 256;
    bytes += items[i].length;
  }
  const std::uint64_t dig_off = tot;
  tot += std::uint64_t(cm.n_chunks()) * 8;
  Shard::SeedLane lane;
  for (auto it = host_pool_.begin(); it != host_pool_.end(); ++it)
    if ((*it)->n >= tot) {
      lane.buf = std::move(*it);
      host_pool_.erase(it);
      break;
    }
  if (!lane.buf) {
    lane.buf = std::make_unique<HostBuf>();
    if (Status s = lane.buf->alloc(tot); !ok(s)) return s;
  }
  auto* base = static_cast<std::uint8_t*>(lane.buf->p);
  // the source: a serve state in this process (or imported), or off-box
  SourceView view;
  if (a.source_endpoint.rfind("tcp:", 0) == 0) {
    lane.tcp = std::make_shared<StreamSource>();
    Status s = lane.tcp->open(a.source_endpoint, ServeRegistry::key(model_, a.source_replica, sh.idx),
                              v, cfg_.pull_timeout_s, &host_pool_);
    if (!ok(s)) {
      lane.tcp->release(&host_pool_);
      return s;
    }
    view = lane.tcp->view();
  } else if (Status s = resolve_source(sh, a, v, &view, cfg_.pull_timeout_s); !ok(s)) {
    return s;
  }
  if (!(view.cmap == cm)) {
    if (lane.tcp) lane.tcp->release(&host_pool_);
    return Status::protocol_error;
  }
  std::vector<dev::ItemDesc> descs;
  for (std::size_t i = 0; i < items.size(); ++i)
    append_identity(&descs, view.item_ptrs[i], reinterpret_cast<std::uint64_t>(base + off[i]),
                    items[i].length, cm, i);
  for (auto& d : descs) d.pad = 1;  // host-memory landing: no tensor maps (generic bulk stores)
  const bool src_complete = a.source_complete && !lane.tcp;
  dev::SrcDesc sdesc{reinterpret_cast<const std::uint64_t*>(view.digests),
                     src_complete ? nullptr : reinterpret_cast<const std::uint32_t*>(view.flags),
                     view.epoch, 0};
  if (!sh.seed_stream) RS_CUDA(cudaStreamCreateWithFlags(&sh.seed_stream, cudaStreamNonBlocking));
  if (!sh.seed_ev) RS_CUDA(cudaEventCreateWithFlags(&sh.seed_ev, cudaEventDisableTiming));
  dev::PullParams pp{};
  RS_CUDA(dev::upload_pull_plan(sh.device, sh.seed_stream, descs.data(),
                                static_cast<std::uint32_t>(descs.size()), &sdesc, 1, cm.n_chunks(),
                                &sh.seed_plan, &pp));
  stats_.h2d_bytes += sh.seed_plan.h2d_bytes;
  pp.dst_digests = reinterpret_cast<std::uint64_t*>(base + dig_off);
  pp.dst_flags = nullptr;  // not served while it fills (seeding copies are never chased)
  pp.dst_epoch = 1;
  pp.timeout_ns = static_cast<std::uint64_t>(cfg_.pull_timeout_s * 1e9);
  pp.remote = view.device >= 0 && view.device != sh.device ? 1u : 0u;
  // A PCIe-bound background fill: a few SMs, beside whatever else runs.
  RS_CUDA(dev::launch_pull(pp, std::min(grid(sh), 16), sh.seed_stream));
  stats_.kernel_launches += dev::pull_has_work(pp) ? 1 : 0;
  RS_CUDA(cudaEventRecord(sh.seed_ev, sh.seed_stream));
  lane.key = ServeRegistry::key(model_, replica_ + "+seed@" + std::to_string(v), sh.idx);
  lane.serve = serves_->ensure(lane.key);
  {
    std::vector<std::uint64_t> ends, ptrs;
    for (std::size_t i = 0; i < items.size(); ++i) {
      ends.push_back(items[i].stream_offset + items[i].length);
      ptrs.push_back(reinterpret_cast<std::uint64_t>(base + off[i]));
    }
    std::lock_guard lk(lane.serve->m);
    lane.serve->serving = false;  // until the fill verified every chunk
    lane.serve->imported = false;
    lane.serve->version = v;
    lane.serve->complete = false;
    lane.serve->progress = 0;
    lane.serve->device = -1;
    lane.serve->pid = static_cast<int>(getpid());
    lane.serve->item_ends = std::move(ends);
    lane.serve->item_ptrs = std::move(ptrs);
    lane.serve->cmap = cm;
    lane.serve->digests = reinterpret_cast<std::uint64_t>(base + dig_off);
    lane.serve->flags = 0;
    lane.serve->epoch = 1;
    lane.serve->host_name = lane.buf->name;
    lane.serve->host_size = lane.buf->n;
    lane.serve->host_base = reinterpret_cast<std::uint64_t>(base);
  }
  sh.seed_lanes.emplace(v, std::move(lane));
  (void)bytes;
  return Status::ok;
}

Status Client::start_seed(const SeedStart& ss) {
  join_seed();  // a fill of a stale target ends first (its report is ignored)
  seed_status_.assign(num_shards_, Status::not_found);
  struct Job {
    std::uint32_t shard;
    int device;
    cudaEvent_t ev;
    const dev::PullStatus* status;
    std::shared_ptr<ServeState> serve;
    std::shared_ptr<StreamSource> tcp;
    std::uint64_t bytes, items;
  };
  std::vector<Job> jobs;
  for (auto& sh : shards_) {
    if (sh.device < 0 || sh.idx >= ss.assignments.size()) continue;
    const bool had = sh.seed_lanes.count(ss.version) != 0;
    Status s = launch_seed(sh, ss.assignments[sh.idx]);
    if (!ok(s)) {
      seed_status_[sh.idx] = s;
      if (seed_report_) reg_->complete(model_, replica_, sh.idx, s, true, ss.version);
      continue;
    }
    auto& lane = sh.seed_lanes.at(ss.version);
    if (had) {  // filled by an earlier start (join_seed above: not running)
      std::lock_guard lk(lane.serve->m);
      seed_status_[sh.idx] = lane.serve->complete ? Status::ok : Status::transfer_failed;
      continue;
    }
    std::uint64_t bytes = 0;
    for (std::size_t i = 0; i < lane.serve->item_ends.size(); ++i)
      bytes += lane.serve->item_ends[i] - (i ? lane.serve->item_ends[i - 1] : 0);
    jobs.push_back({sh.idx, sh.device, sh.seed_ev,
                    reinterpret_cast<const dev::PullStatus*>(
                        static_cast<std::uint8_t*>(sh.seed_plan.scratch) + 64),
                    lane.serve, lane.tcp, bytes, lane.serve->item_ends.size()});
  }
  if (jobs.empty()) return Status::ok;
  // The waiter touches only what it was handed (events, status words, the
  // lanes' serve states), its own status slots and the registry (its own lock).
  seed_thread_ = std::thread([this, jobs = std::move(jobs), v = ss.version, report = seed_report_] {
    for (const auto& j : jobs) {
      DeviceGuard g(j.device);
      cudaError_t e = cudaEventSynchronize(j.ev);
      dev::PullStatus st{};
      if (e == cudaSuccess) e = cudaMemcpy(&st, j.status, sizeof(st), cudaMemcpyDeviceToHost);
      bool good = e == cudaSuccess && st.code == dev::kPullOk;
      if (j.tcp) good = ok(j.tcp->finish(good)) && good;
      if (good) {
        std::lock_guard lk(j.serve->m);
        j.serve->serving = true;
        j.serve->complete = true;
        j.serve->progress = j.items;
        seed_cross_dc_ += j.bytes;
      }
      const Status out = good ? Status::ok
                         : e != cudaSuccess ? Status::transfer_failed
                         : st.code == dev::kPullChecksum ? Status::checksum_mismatch
                         : Status::timeout;
      seed_status_[j.shard] = out;
      if (!report) continue;  // the caller reports through its operation log
      if (good) reg_->progress(model_, replica_, j.shard, j.items, true, v);
      reg_->complete(model_, replica_, j.shard, out, true, v);
    }
  });
  return Status::ok;
}

Status Client::seed_status(std::uint32_t shard) {
  join_seed();
  return shard < seed_status_.size() ? seed_status_[shard] : Status::not_found;
}

Result<std::string> Client::export_seed(std::uint32_t shard, VersionId v) {
  if (shard >= num_shards_) return Status::invalid_argument;
  join_seed();
  auto it = shards_[shard].seed_lanes.find(v);
  if (it == shards_[shard].seed_lanes.end()) return Status::not_found;
  return serves_->export_state(it->second.key);
}

void Client::join_seed() {
  if (seed_thread_.joinable()) seed_thread_.join();
  for (auto& sh : shards_)  // off-box sources' pinned buffers back to the pool
    for (auto& [v, lane] : sh.seed_lanes)
      if (lane.tcp) {
        lane.tcp->release(&host_pool_);
        lane.tcp.reset();
      }
}

void Client::release_seed_lane(VersionId v) {
  // DirectiveKind::offload_release, purpose seed (client_core.cpp:1773-1794)
  join_seed();
  for (auto& sh : shards_) {
    auto it = sh.seed_lanes.find(v);
    if (it == sh.seed_lanes.end()) continue;
    {
      std::lock_guard lk(it->second.serve->m);
      it->second.serve->serving = false;
    }
    serves_->erase(it->second.key);
    if (host_pool_.size() < 2) host_pool_.push_back(std::move(it->second.buf));
    sh.seed_lanes.erase(it);
  }
}

std::vector<VersionId> Client::seed_lanes() const {
  std::set<VersionId> vs;
  for (const auto& sh : shards_)
    for (const auto& [v, lane] : sh.seed_lanes) vs.insert(v);
  return {vs.begin(), vs.end()};
}

Status Client::settle_offload(OpOutcome* o, double wait_s) {
  // ResponseKind::offload_first (client_core.cpp:1237-1253): park the named
  // version in host memory, confirm every shard, then the op proceeds.
  if (o->done || !o->offload_first) return Status::ok;
  const VersionId v = *o->offload_first;
  std::vector<std::string> eps;
  const bool ok_lane = ok(make_retention_lanes(v, &eps));
  for (std::uint32_t i = 0; i < num_shards_; ++i)
    if (Status s = reg_->offload_confirm(model_, replica_, i, v, ok_lane, eps[i]); !ok(s)) return s;
  *o = reg_->op_result(model_, replica_);
  if (!o->done) *o = reg_->wait_op(model_, replica_, wait_s);
  return Status::ok;
}

Status Client::serve_tables(std::uint32_t shard, std::uint64_t* digests, std::uint64_t* flags,
                            std::uint32_t* epoch, std::uint32_t* n_batches) const {
  if (shard >= num_shards_ || !shards_[shard].holding) return Status::not_found;
  const Payload& p = *shards_[shard].holding;
  *digests = reinterpret_cast<std::uint64_t>(p.digests.p);
  *flags = reinterpret_cast<std::uint64_t>(p.flags.p);
  *epoch = p.epoch;
  *n_batches = p.cmap.n_batches();
  return Status::ok;
}

Result<std::string> Client::export_serve(std::uint32_t shard) {
  if (shard >= num_shards_) return Status::invalid_argument;
  return serves_->export_state(ServeRegistry::key(model_, replica_, shard));
}

}  // namespace rsb
