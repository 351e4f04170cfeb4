// The reference's own client scenarios, run through the two integration
// levels of INTEGRATION.md on a GPU.  Compiled against the UNMODIFIED
// reference headers (/root/reference/proj/include) and linked with the
// reference library built from its sources (oracle/_ref) plus libros_b200.so.
//
//   level A  B200Client (refstore_b200/b200_client.hpp) over the C ABI,
//            device-resident regions;
//   level B  the reference ClientCore + ServerCore + SimExecutor, with
//            B200Transport (refstore_b200/b200_transport.hpp) as the
//            DataTransport -- the reference's own pull loop and item
//            verification, the B200 kernel moving the bytes.
//
// Scenarios (tests/unit/test_client_core.cpp):
//   replicate pulls bytes that verify against the manifest  :163-202
//   corrupt source: quiet retry, report, re-pick             :346-377
//   cross-link update fills a host seed, consumes it locally :460-503
//
// Prints one "PASS <level> <scenario> k=v ..." or "FAIL ..." line per
// scenario; exit status 0 iff every scenario passed.  --list prints the
// scenario names without touching a GPU.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include <future>

#include "refstore/client_core.hpp"
#include "refstore/digest.hpp"
#include "refstore/manifest.hpp"
#include "refstore/transport_stream.hpp"
#include "refstore/server_core.hpp"
#include "refstore/trace.hpp"
#include "refstore/transport_mem.hpp"
#include "refstore_b200/b200_client.hpp"
#include "refstore_b200/b200_transport.hpp"

using namespace refstore;

namespace {

int failures = 0;

void report(bool ok, const char* level, const char* scenario, const std::string& kv) {
  std::printf("%s %s %s %s\n", ok ? "PASS" : "FAIL", level, scenario, kv.c_str());
  std::fflush(stdout);
  if (!ok) ++failures;
}

// fill pattern of the reference ClusterFix (test_client_core.cpp:76-81)
std::vector<std::byte> pattern(std::size_t len, std::uint64_t salt) {
  std::vector<std::byte> v(len);
  for (std::size_t i = 0; i < len; ++i) v[i] = std::byte((salt * 1315423911u + i * 131u) & 0xff);
  return v;
}

struct Tensor {
  std::uint32_t shard;
  std::string name;
  std::size_t len;
  std::uint64_t salt;
};
const std::vector<Tensor> kT = {{0, "big", 3u << 20, 7}, {0, "t1", 1000, 8}, {0, "t2", 2000, 9},
                                {1, "u1", 4096, 10}};
const std::uint64_t kBytes = (3u << 20) + 1000 + 2000 + 4096;

std::string counters(const ClientCore::Stats& s) {
  return "items_verified=" + std::to_string(s.items_verified) +
         " bytes_pulled=" + std::to_string(s.bytes_pulled) +
         " checksum_failures=" + std::to_string(s.checksum_failures) +
         " failure_reports=" + std::to_string(s.failure_reports);
}

// ------------------------------------------------------------------ level A
struct DevBufs {
  std::map<std::pair<std::uint32_t, std::string>, std::byte*> p;
  ~DevBufs() {
    for (auto& [k, v] : p) cudaFree(v);
  }
  std::span<std::byte> make(const Tensor& t, std::uint64_t salt) {
    std::byte* d = nullptr;
    cudaMalloc(&d, t.len);
    auto h = pattern(t.len, salt);
    cudaMemcpy(d, h.data(), t.len, cudaMemcpyHostToDevice);
    p[{t.shard, t.name}] = d;
    return {d, t.len};
  }
  std::vector<std::byte> host(const Tensor& t) const {
    std::vector<std::byte> h(t.len);
    cudaMemcpy(h.data(), p.at({t.shard, t.name}), t.len, cudaMemcpyDeviceToHost);
    return h;
  }
};

void level_a_replicate() {
  B200Cluster cl;
  DevBufs tb, rb;
  B200Client t(cl, "m", "T", 2);
  for (const auto& x : kT) t.register_tensor(x.shard, x.name, tb.make(x, x.salt));
  std::optional<ClientCore::OpResult> pr;
  t.publish(1, [&](ClientCore::OpResult r) { pr = r; });
  B200Client w(cl, "m", "R", 2);
  for (const auto& x : kT) w.register_tensor(x.shard, x.name, rb.make(x, 100));
  std::optional<ClientCore::OpResult> rr;
  w.replicate(VersionSpec::latest(), [&](ClientCore::OpResult r) { rr = r; });
  bool ok = pr && pr->status == Status::ok && rr && rr->status == Status::ok && rr->version == VersionId{1};
  ok &= w.is_published() && w.current_version() == VersionId{1};
  for (const auto& x : kT) ok &= rb.host(x) == pattern(x.len, x.salt);
  const auto s = w.stats();
  ok &= s.items_verified == 3 && s.bytes_pulled == kBytes && s.checksum_failures == 0;
  auto view = cl.replica_view("m", "R");
  ok &= view && view->lifecycle == "published" && view->version == VersionId{1};
  auto lm = cl.listing("m");
  ok &= lm.count(1) && lm[1].count("T") && lm[1].count("R");
  report(ok, "A", "replicate_pulls_bytes_that_verify", counters(s));
}

// ------------------------------------------------------------------ level B
// ClusterFix (test_client_core.cpp:23-117) with B200Transport as the data
// plane and managed memory regions.
struct RefFix {
  SimExecutor exec;
  TraceLog log;
  MemNetwork net;
  B200Transport b200{&net, 0};
  ServerCore srv;
  struct Node {
    ServeRegistry serves;
    std::map<std::pair<std::uint32_t, std::string>, std::byte*> bufs;
    std::unique_ptr<ClientCore> core;
    ~Node() {
      core.reset();
      for (auto& [k, v] : bufs) cudaFree(v);
    }
  };
  std::map<std::string, std::unique_ptr<Node>> nodes;

  bool use_b200 = true;  // false: the reference MemNetwork moves the bytes (equivalence runs)
  RefFix() : srv("A", ServerConfig{}, &exec, &log, net.sender()) {
    net.register_server("A", &srv, &exec);
    srv.start();
  }
  ~RefFix() {
    nodes.clear();
    srv.stop();
  }
  ClientCore& make(const std::string& replica, std::uint32_t shards) {
    auto n = std::make_unique<Node>();
    ClientConfig cfg;
    cfg.servers = {"A"};
    cfg.data_endpoint = "ep:" + replica;
    b200.register_data(cfg.data_endpoint, &n->serves);
    DataTransport* data = use_b200 ? static_cast<DataTransport*>(&b200) : static_cast<DataTransport*>(&net);
    n->core = std::make_unique<ClientCore>("m", replica, shards, cfg, &exec, &log, &net, data, &n->serves);
    ClientCore& r = *n->core;
    nodes[replica] = std::move(n);
    return r;
  }
  void reg(const std::string& replica, const Tensor& t, std::uint64_t salt) {
    Node& n = *nodes.at(replica);
    std::byte* p = nullptr;
    cudaMallocManaged(&p, t.len);
    n.bufs[{t.shard, t.name}] = p;
    fill(replica, t, salt);
    n.core->register_tensor(t.shard, t.name, {p, t.len});
  }
  void fill(const std::string& replica, const Tensor& t, std::uint64_t salt) {
    cudaDeviceSynchronize();
    auto h = pattern(t.len, salt);
    std::memcpy(nodes.at(replica)->bufs.at({t.shard, t.name}), h.data(), t.len);
  }
  std::vector<std::byte> bytes(const std::string& replica, const Tensor& t) {
    cudaDeviceSynchronize();
    const std::byte* p = nodes.at(replica)->bufs.at({t.shard, t.name});
    return {p, p + t.len};
  }
  bool same(const std::string& a, const std::string& b, const Tensor& t) {
    cudaDeviceSynchronize();
    return std::memcmp(nodes.at(a)->bufs.at({t.shard, t.name}), nodes.at(b)->bufs.at({t.shard, t.name}),
                       t.len) == 0;
  }
  ClientCore::OpResult run(std::function<void(ClientCore::OpFn)> op) {
    std::optional<ClientCore::OpResult> out;
    op([&](ClientCore::OpResult r) { out = std::move(r); });
    Time h = exec.now() + std::chrono::seconds(60);
    while (!out && exec.step(h)) {
    }
    if (!out) {
      ClientCore::OpResult r;
      r.status = Status::timeout;
      return r;
    }
    return std::move(*out);
  }
  void settle() {
    Time h = exec.now() + std::chrono::seconds(5);
    while (exec.step(h)) {
    }
  }
};

void level_b_replicate() {
  RefFix fx;
  ClientCore& t = fx.make("T", 2);
  for (const auto& x : kT) fx.reg("T", x, x.salt);
  bool ok = fx.run([&](auto cb) { t.publish(1, cb); }).status == Status::ok;
  ClientCore& w = fx.make("R", 2);
  for (const auto& x : kT) fx.reg("R", x, 100);
  auto r = fx.run([&](auto cb) { w.replicate(VersionSpec::latest(), cb); });
  ok &= r.status == Status::ok && r.version == VersionId{1};
  ok &= w.is_published() && w.current_version() == VersionId{1};
  for (const auto& x : kT) ok &= fx.same("T", "R", x);
  const auto s = w.stats();
  ok &= s.items_verified == 3 && s.bytes_pulled == kBytes && s.checksum_failures == 0;
  fx.settle();
  auto view = fx.srv.replica_view("m", "R");
  ok &= view && view->lifecycle == "published" && view->version == VersionId{1};
  // the bytes moved on the GPU, through the B200 kernel
  // the registered regions' bytes moved on the GPU, through the B200 kernel;
  // the packed groups (host-heap staging in the reference client) on the host
  ok &= fx.b200.device_pulls() > 0 && fx.b200.device_bytes() == (3u << 20) &&
        fx.b200.device_bytes() + fx.b200.host_bytes() == kBytes;
  report(ok, "B", "replicate_pulls_bytes_that_verify",
         counters(s) + " device_pulls=" + std::to_string(fx.b200.device_pulls()) +
             " device_bytes=" + std::to_string(fx.b200.device_bytes()) +
             " host_bytes=" + std::to_string(fx.b200.host_bytes()) +
             " last_error=" + std::to_string(fx.b200.last_error()) +
             " status=" + std::to_string(static_cast<int>(r.status)));
}

void level_b_corrupt_source() {
  // test_client_core.cpp:346-377: T2's copy is corrupted in place; the
  // reader's item check fails, retries quietly, reports, and re-picks T1.
  RefFix fx;
  const std::vector<Tensor> ts = {{0, "big", 3u << 20, 11}, {0, "tiny", 5000, 12}};
  ClientCore& t1 = fx.make("T1", 1);
  for (const auto& x : ts) fx.reg("T1", x, x.salt);
  bool ok = fx.run([&](auto cb) { t1.publish(1, cb); }).status == Status::ok;
  ClientCore& t2 = fx.make("T2", 1);
  fx.reg("T2", ts[0], 20);
  fx.reg("T2", ts[1], 21);
  ok &= fx.run([&](auto cb) { t2.replicate(VersionSpec::latest(), cb); }).status == Status::ok;
  cudaDeviceSynchronize();
  fx.nodes.at("T2")->bufs.at({0, "big"})[17] ^= std::byte{0xFF};
  ClientCore& w = fx.make("R", 1);
  fx.reg("R", ts[0], 30);
  fx.reg("R", ts[1], 31);
  auto r = fx.run([&](auto cb) { w.replicate(VersionSpec::latest(), cb); });
  ok &= r.status == Status::ok;
  const auto s = w.stats();
  ok &= s.checksum_failures == 2 && s.failure_reports == 1;
  for (const auto& x : ts) ok &= fx.same("T1", "R", x);
  ok &= fx.srv.listing("m")[1].count("T2") == 1;  // corruption does not condemn
  report(ok, "B", "corrupt_source_quiet_retry_report_repick", counters(s));
}

void level_a_update() {
  // test_client_core.cpp:204-231: update reports no change, then pulls v2
  B200Cluster cl;
  DevBufs tb, rb;
  const Tensor w{0, "w", 200000, 1};
  B200Client t(cl, "m", "T", 1);
  t.register_tensor(0, w.name, tb.make(w, 1));
  std::optional<ClientCore::OpResult> r;
  t.publish(1, [&](ClientCore::OpResult x) { r = x; });
  bool ok = r && r->status == Status::ok;
  B200Client rd(cl, "m", "R", 1);
  rd.register_tensor(0, w.name, rb.make(w, 50));
  rd.replicate(VersionSpec::latest(), [&](ClientCore::OpResult x) { r = x; });
  ok &= r->status == Status::ok;
  rd.update(VersionSpec::latest(), [&](ClientCore::OpResult x) { r = x; });
  ok &= r->status == Status::ok && !r->changed && r->version == VersionId{1};
  t.unpublish([&](ClientCore::OpResult x) { r = x; });
  ok &= r->status == Status::ok;
  auto h2 = pattern(w.len, 2);
  cudaMemcpy(tb.p.at({0, "w"}), h2.data(), w.len, cudaMemcpyHostToDevice);
  t.publish(2, [&](ClientCore::OpResult x) { r = x; });
  ok &= r->status == Status::ok;
  rd.update(VersionSpec::latest(), [&](ClientCore::OpResult x) { r = x; });
  ok &= r->status == Status::ok && r->changed && r->version == VersionId{2};
  ok &= rd.current_version() == VersionId{2} && rb.host(w) == h2;
  report(ok, "A", "update_no_change_then_newer", counters(rd.stats()));
}

void level_a_seed() {
  // test_client_core.cpp:460-503: a cross-link update fills a host seed,
  // then consumes it locally (ClientConfig.datacenter / offload_seed)
  B200Cluster cl;
  DevBufs tb, fb;
  const Tensor w{0, "w", 200000, 44}, x{1, "x", 100000, 45};
  ClientConfig c1;
  c1.datacenter = "dc1";
  B200Client t(cl, "m", "T", 2, c1);
  t.register_tensor(0, w.name, tb.make(w, w.salt));
  t.register_tensor(1, x.name, tb.make(x, x.salt));
  std::optional<ClientCore::OpResult> r;
  t.publish(1, [&](ClientCore::OpResult o) { r = o; });
  bool ok = r && r->status == Status::ok;
  ClientConfig c2;
  c2.datacenter = "dc2";
  c2.offload_seed = true;
  B200Client f(cl, "m", "F", 2, c2);
  f.register_tensor(0, w.name, fb.make(w, 46));
  f.register_tensor(1, x.name, fb.make(x, 47));
  // first poll: the version is masked for dc2, a background fill starts
  f.update(VersionSpec::latest(), [&](ClientCore::OpResult o) { r = o; });
  ok &= r->status == Status::ok && !r->changed && !r->version.has_value();
  f.poll();  // the fill's report is in
  auto sv = cl.replica_view("m", "F+seed@1");
  ok &= sv && sv->lifecycle == "published";
  ok &= f.stats().bytes_pulled_cross_dc == 200000 + 100000;
  // second poll: the change lands by consuming the local seed buffer
  f.update(VersionSpec::latest(), [&](ClientCore::OpResult o) { r = o; });
  ok &= r->status == Status::ok && r->changed && r->version == VersionId{1};
  ok &= f.current_version() == VersionId{1};
  ok &= fb.host(w) == pattern(w.len, w.salt) && fb.host(x) == pattern(x.len, x.salt);
  const auto s = f.stats();
  ok &= s.bytes_copied_local == 200000 + 100000 && s.bytes_pulled_cross_dc == 200000 + 100000;
  // consumed and drained: handed back, the lane vanishes
  f.poll();
  ok &= !cl.replica_view("m", "F+seed@1").has_value();
  report(ok, "A", "cross_link_update_fills_a_host_seed_then_consumes_it",
         "bytes_pulled_cross_dc=" + std::to_string(s.bytes_pulled_cross_dc) +
             " bytes_copied_local=" + std::to_string(s.bytes_copied_local));
}

void level_b_update() {
  RefFix fx;
  const Tensor w{0, "w", 200000, 1};
  ClientCore& t = fx.make("T", 1);
  fx.reg("T", w, 1);
  bool ok = fx.run([&](auto cb) { t.publish(1, cb); }).status == Status::ok;
  ClientCore& rd = fx.make("R", 1);
  fx.reg("R", w, 50);
  ok &= fx.run([&](auto cb) { rd.replicate(VersionSpec::latest(), cb); }).status == Status::ok;
  auto r = fx.run([&](auto cb) { rd.update(VersionSpec::latest(), cb); });
  ok &= r.status == Status::ok && !r.changed && r.version == VersionId{1};
  ok &= fx.run([&](auto cb) { t.unpublish(cb); }).status == Status::ok;
  fx.fill("T", w, 2);
  ok &= fx.run([&](auto cb) { t.publish(2, cb); }).status == Status::ok;
  r = fx.run([&](auto cb) { rd.update(VersionSpec::latest(), cb); });
  ok &= r.status == Status::ok && r.changed && r.version == VersionId{2};
  ok &= rd.current_version() == VersionId{2} && fx.same("T", "R", w);
  report(ok, "B", "update_no_change_then_newer", counters(rd.stats()));
}

void level_b_silent_source() {
  // test_client_core.cpp:317-344: a silent source is reported (timeout) and
  // the pull moves to a sibling; the report condemns the silent copy
  RefFix fx;
  const Tensor w{0, "w", 150000, 6};
  ClientCore& t1 = fx.make("T1", 1);
  fx.reg("T1", w, 6);
  bool ok = fx.run([&](auto cb) { t1.publish(1, cb); }).status == Status::ok;
  ClientCore& t2 = fx.make("T2", 1);
  fx.reg("T2", w, 60);
  ok &= fx.run([&](auto cb) { t2.replicate(VersionSpec::latest(), cb); }).status == Status::ok;
  fx.b200.set_data_silent("ep:T2", true);
  ClientCore& rd = fx.make("R", 1);
  fx.reg("R", w, 70);
  auto r = fx.run([&](auto cb) { rd.replicate(VersionSpec::latest(), cb); });
  ok &= r.status == Status::ok && rd.stats().failure_reports >= 1 && fx.same("T1", "R", w);
  auto lm = fx.srv.listing("m");
  ok &= lm.count(1) && !lm[1].count("T2") && lm[1].count("T1");
  report(ok, "B", "silent_source_reported_and_pull_moves", counters(rd.stats()));
}

void level_b_equivalence() {
  // test_transport.cpp:573-587: the same replicate through the reference
  // MemNetwork and through B200Transport lands identical bytes, equal to the
  // publisher's pattern
  std::map<std::pair<std::uint32_t, std::string>, std::vector<std::byte>> got[2];
  std::uint64_t device_bytes = 0;
  for (int k = 0; k < 2; ++k) {
    RefFix fx;
    fx.use_b200 = k == 1;
    ClientCore& t = fx.make("T", 2);
    for (const auto& x : kT) fx.reg("T", x, x.salt);
    fx.run([&](auto cb) { t.publish(1, cb); });
    ClientCore& rd = fx.make("R", 2);
    for (const auto& x : kT) fx.reg("R", x, 100);
    fx.run([&](auto cb) { rd.replicate(VersionSpec::latest(), cb); });
    for (const auto& x : kT) got[k][{x.shard, x.name}] = fx.bytes("R", x);
    if (k == 1) device_bytes = fx.b200.device_bytes();
  }
  bool ok = device_bytes > 0;
  for (const auto& x : kT) ok &= got[0][{x.shard, x.name}] == got[1][{x.shard, x.name}] &&
                                 got[1][{x.shard, x.name}] == pattern(x.len, x.salt);
  report(ok, "B", "transport_equivalence_mem_vs_b200", "device_bytes=" + std::to_string(device_bytes));
}

// ------------------------------------------------------------------ level C
// The reference's own data-plane dialer (StreamData, transport_stream.cpp)
// against the B200 process's TCP server, which answers the reference wire
// (RSDP, transport_stream.hpp:36-76) from device-resident serve states.  The
// reference decodes the B200 manifest and verifies every item it pulled with
// its own digest64.
void level_c_rsdp_reader() {
  B200Cluster cl;
  DevBufs tb;
  B200Client t(cl, "m", "T", 2);
  for (const auto& x : kT) t.register_tensor(x.shard, x.name, tb.make(x, x.salt));
  std::optional<ClientCore::OpResult> pr;
  t.publish(1, [&](ClientCore::OpResult r) { pr = r; });
  int port = 0;
  bool ok = pr && pr->status == Status::ok && rs_cluster_listen(cl.get(), "127.0.0.1", 0, &port) == 0;
  const std::string ep = "127.0.0.1:" + std::to_string(port);
  StreamData sd;
  ThreadExecutor exec;
  std::uint64_t items_verified = 0, bytes = 0;
  for (std::uint32_t shard = 0; ok && shard < 2; ++shard) {
    std::size_t n = 0;
    rs_manifest(t.handle(), shard, nullptr, 0, &n);
    std::string enc(n, '\0');
    rs_manifest(t.handle(), shard, enc.data(), enc.size(), &n);
    auto man = TensorManifest::decode(enc);  // the reference decoder
    if (!man) {
      ok = false;
      break;
    }
    const auto& items = man->items();
    std::uint64_t total = 0;
    for (const auto& it : items) total += it.length;
    // long-poll query: the version is complete, every item readable
    QuerySpec q{"m", "T", 1, shard, items.size()};
    std::promise<QueryResult> qp;
    sd.async_query(ep, q, &exec, [&](QueryResult r) { qp.set_value(r); });
    const QueryResult qr = qp.get_future().get();
    ok &= qr.status == Status::ok && qr.progress == items.size() && qr.complete;
    // pull the whole item stream (responses may be short: loop)
    std::vector<std::byte> stream(total);
    for (std::uint64_t off = 0; ok && off < total;) {
      PullSpec ps;
      ps.model = "m";
      ps.replica = "T";
      ps.version = 1;
      ps.shard = shard;
      ps.offset = off;
      ps.max_bytes = total - off;
      std::promise<PullResult> pp;
      sd.async_pull(ep, ps, PullDest{{stream.data() + off, total - off}}, &exec,
                    [&](PullResult r) { pp.set_value(r); });
      const PullResult r = pp.get_future().get();
      ok &= r.status == Status::ok && r.bytes > 0 && r.source_complete;
      off += r.bytes;
      bytes += r.bytes;
    }
    // digest64 of every item against the manifest (TransferTask::verify_ready)
    std::uint64_t at = 0;
    for (const auto& it : items) {
      ok &= digest64(stream.data() + at, it.length) == it.digest;
      at += it.length;
      ++items_verified;
    }
    // a wrong version is refused (compute_slice: not_serving)
    PullSpec bad;
    bad.model = "m";
    bad.replica = "T";
    bad.version = 2;
    bad.shard = shard;
    bad.max_bytes = 16;
    std::byte tmp[16];
    std::promise<PullResult> bp;
    sd.async_pull(ep, bad, PullDest{{tmp, 16}}, &exec, [&](PullResult r) { bp.set_value(r); });
    ok &= bp.get_future().get().status == Status::not_serving;
  }
  report(ok, "C", "rsdp_reference_reader_pulls_and_verifies",
         "items_verified=" + std::to_string(items_verified) + " bytes_pulled=" + std::to_string(bytes));
}

}  // namespace

int main(int argc, char** argv) {
  const std::vector<std::pair<const char*, void (*)()>> scenarios = {
      {"A replicate_pulls_bytes_that_verify", level_a_replicate},
      {"B replicate_pulls_bytes_that_verify", level_b_replicate},
      {"B corrupt_source_quiet_retry_report_repick", level_b_corrupt_source},
      {"A update_no_change_then_newer", level_a_update},
      {"B update_no_change_then_newer", level_b_update},
      {"B silent_source_reported_and_pull_moves", level_b_silent_source},
      {"B transport_equivalence_mem_vs_b200", level_b_equivalence},
      {"C rsdp_reference_reader_pulls_and_verifies", level_c_rsdp_reader},
      {"A cross_link_update_fills_a_host_seed_then_consumes_it", level_a_seed},
  };
  if (argc > 1 && std::strcmp(argv[1], "--list") == 0) {
    for (const auto& [name, fn] : scenarios) std::printf("%s\n", name);
    return 0;
  }
  if (argc > 1 && std::strcmp(argv[1], "--probe") == 0) {
    // one managed-memory copy through rs_pull_spans (diagnostic)
    const std::size_t len = 8u << 20;
    std::byte *a = nullptr, *b = nullptr;
    cudaMallocManaged(&a, len);
    cudaMallocManaged(&b, len);
    auto h = pattern(len, 5);
    std::memcpy(a, h.data(), len);
    std::uint64_t src = reinterpret_cast<std::uint64_t>(a), dst = reinterpret_cast<std::uint64_t>(b), n = len;
    int code = -1;
    float ms = 0;
    int rc = rs_pull_spans(&src, &dst, &n, 1, 4096, nullptr, nullptr, 0, nullptr, &code, &ms);
    cudaDeviceSynchronize();
    std::printf("probe rc=%d code=%d equal=%d err=%s\n", rc, code, std::memcmp(a, b, len) == 0,
                cudaGetErrorString(cudaGetLastError()));
    return rc;
  }
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    std::printf("FAIL no CUDA device\n");
    return 2;
  }
  for (const auto& [name, fn] : scenarios) {
    if (argc > 1 && std::strstr(name, argv[1]) == nullptr) continue;  // a filter
    std::fprintf(stderr, "[scenario] %s\n", name);
    fn();
    std::fprintf(stderr, "[scenario] %s done\n", name);
  }
  return failures ? 1 : 0;
}
