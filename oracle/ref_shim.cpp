// TEST INFRASTRUCTURE ONLY -- a C ABI over the UNMODIFIED reference refstore
// library (compiled from /root/reference/proj/src by oracle/Makefile).
//
// Used by tests/ (parity checker), tests/golden/make_golden.py (fixture
// generator) and bench.py's cpu_baseline / --impl reference legs. Never
// linked into or called by the product library.
//
// The cluster driver mirrors the reference's own ClusterFix fixture
// (tests/unit/test_client_core.cpp:23-117): one ServerCore plus N ClientCores
// wired through MemNetwork (transport_mem.cpp), driven either by one
// deterministic SimExecutor (parity mode) or one ThreadExecutor per
// participant (throughput mode).

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <future>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <set>
#include <span>
#include <thread>
#include <functional>
#include <string>
#include <vector>

#include "refstore/client_core.hpp"
#include "refstore/digest.hpp"
#include "refstore/manifest.hpp"
#include "refstore/server_core.hpp"
#include "refstore/transport_mem.hpp"

using namespace refstore;

namespace {

long copy_out(const std::string& s, char* out, std::size_t cap) {
  if (out && cap >= s.size()) std::memcpy(out, s.data(), s.size());
  return static_cast<long>(s.size());
}

struct Node {
  ServeRegistry serves;
  std::unique_ptr<ThreadExecutor> texec;  // threaded mode only
  std::unique_ptr<ClientCore> core;
};

struct Cluster {
  bool threaded = false;
  SimExecutor sim;
  std::unique_ptr<ThreadExecutor> server_exec;
  TraceLog log;
  MemNetwork net;
  std::unique_ptr<ServerCore> srv;
  ClientConfig base_cfg;
  std::map<std::string, std::unique_ptr<Node>> nodes;

  Executor* sexec() {
    return threaded ? static_cast<Executor*>(server_exec.get()) : &sim;
  }

  // Runs a set of asynchronous ops to completion; returns results in order.
  std::vector<ClientCore::OpResult> run_many(
      std::vector<std::function<void(ClientCore::OpFn)>> ops, double* secs) {
    std::vector<std::optional<ClientCore::OpResult>> out(ops.size());
    auto t0 = std::chrono::steady_clock::now();
    if (!threaded) {
      for (std::size_t i = 0; i < ops.size(); ++i)
        ops[i]([&out, i](ClientCore::OpResult r) { out[i] = std::move(r); });
      auto all = [&] {
        for (auto& o : out)
          if (!o) return false;
        return true;
      };
      Time horizon = sim.now() + std::chrono::seconds(600);
      while (!all() && sim.step(horizon)) {
      }
    } else {
      std::mutex m;
      std::condition_variable cv;
      std::size_t left = ops.size();
      for (std::size_t i = 0; i < ops.size(); ++i)
        ops[i]([&, i](ClientCore::OpResult r) {
          std::lock_guard lk(m);
          out[i] = std::move(r);
          left--;
          cv.notify_all();
        });
      std::unique_lock lk(m);
      cv.wait_for(lk, std::chrono::seconds(600), [&] { return left == 0; });
    }
    if (secs)
      *secs = std::chrono::duration<double>(std::chrono::steady_clock::now() -
                                            t0)
                  .count();
    std::vector<ClientCore::OpResult> res;
    for (auto& o : out) {
      ClientCore::OpResult r;
      if (o) r = std::move(*o);
      else r.status = Status::timeout;
      res.push_back(std::move(r));
    }
    return res;
  }
};

}  // namespace

extern "C" {

std::uint64_t ref_digest64(const void* p, std::size_t n) {
  return digest64(p, n);
}

// build_publish_payload (client_core.cpp:1547-1579) for one shard of real
// regions: digest every entry, assemble, pack+digest every group, encode.
long ref_build_manifest(int n, const char** names, const void** ptrs,
                        const std::uint64_t* lens, std::uint64_t tiny,
                        std::uint64_t target, char* out, std::size_t cap) {
  std::vector<EntryDesc> descs;
  std::vector<std::span<const std::byte>> regions;
  for (int i = 0; i < n; ++i) {
    auto* b = static_cast<const std::byte*>(ptrs[i]);
    regions.emplace_back(b, lens[i]);
    descs.push_back({names[i], lens[i], digest64(ptrs[i], lens[i])});
  }
  auto m = assemble_manifest(descs, ManifestLimits{tiny, target});
  if (!m) return -static_cast<long>(m.status());
  for (std::uint32_t g = 0; g < m->groups.size(); ++g) {
    std::vector<std::byte> staging(m->groups[g].packed_length);
    pack_group(*m, g, regions, staging);
  }
  return copy_out(m->encode(), out, cap);
}

// build_publish_payload (client_core.cpp:1547-1579) with the entry digests
// supplied by the caller -- each one the reference digest64 of that entry,
// computed elsewhere (in parallel, tensor by tensor) -- so a 16-65 GB
// synthetic model need not sit in memory at once.  Only group members need
// a pointer: pack_group stages them and digests the staging, exactly as the
// reference does.
long ref_build_manifest_pre(int n, const char** names, const void** ptrs,
                            const std::uint64_t* lens, const std::uint64_t* digests,
                            std::uint64_t tiny, std::uint64_t target, char* out,
                            std::size_t cap) {
  std::vector<EntryDesc> descs;
  std::vector<std::span<const std::byte>> regions;
  for (int i = 0; i < n; ++i) {
    regions.emplace_back(static_cast<const std::byte*>(ptrs[i]), ptrs[i] ? lens[i] : 0);
    descs.push_back({names[i], lens[i], digests[i]});
  }
  auto m = assemble_manifest(descs, ManifestLimits{tiny, target});
  if (!m) return -static_cast<long>(m.status());
  for (std::uint32_t g = 0; g < m->groups.size(); ++g) {
    for (const auto& mem : m->groups[g].members)
      if (!ptrs[mem.entry_idx]) return -1;  // a group member without its bytes
    std::vector<std::byte> staging(m->groups[g].packed_length);
    pack_group(*m, g, regions, staging);
  }
  return copy_out(m->encode(), out, cap);
}

// assemble_manifest over explicit (name, length, digest) descriptors, groups
// sealed with seal_groups_modeled when `seal` (modeled payloads).
long ref_assemble_manifest(int n, const char** names, const std::uint64_t* lens,
                           const std::uint64_t* digests, std::uint64_t tiny,
                           std::uint64_t target, int seal, char* out,
                           std::size_t cap) {
  std::vector<EntryDesc> descs;
  for (int i = 0; i < n; ++i) descs.push_back({names[i], lens[i], digests[i]});
  auto m = assemble_manifest(descs, ManifestLimits{tiny, target});
  if (!m) return -static_cast<long>(m.status());
  if (seal) seal_groups_modeled(*m);
  return copy_out(m->encode(), out, cap);
}

std::uint64_t ref_modeled_entry_digest(const char* name, std::uint64_t version,
                                       std::uint64_t length) {
  return modeled_entry_digest(name, version, length);
}

// Decodes a manifest and writes its items as 5 u64 per item
// (is_group, index, length, digest, stream_offset). Returns item count or
// -status.
long ref_manifest_items(const char* data, std::size_t len, std::uint64_t* out,
                        std::size_t cap_items) {
  auto m = TensorManifest::decode(std::string_view(data, len));
  if (!m) return -static_cast<long>(m.status());
  const auto& items = m->items();
  if (out && cap_items >= items.size()) {
    for (std::size_t i = 0; i < items.size(); ++i) {
      out[5 * i + 0] = items[i].is_group;
      out[5 * i + 1] = items[i].index;
      out[5 * i + 2] = items[i].length;
      out[5 * i + 3] = items[i].digest;
      out[5 * i + 4] = items[i].stream_offset;
    }
  }
  return static_cast<long>(items.size());
}

int ref_version_resolve(const char* spec, const std::uint64_t* avail, int n,
                        std::uint64_t* out) {
  auto s = VersionSpec::parse(spec);
  if (!s) return static_cast<int>(s.status());
  std::set<VersionId> a(avail, avail + n);
  auto r = resolve_version(*s, a);
  if (!r) return static_cast<int>(Status::not_found);
  *out = *r;
  return 0;
}

// ---------------------------------------------------------------- clusters

void* ref_cluster_new(int threaded, int server_pipeline, int client_pipeline,
                      std::uint64_t chunk_bytes) {
  auto* c = new Cluster();
  c->threaded = threaded != 0;
  if (c->threaded) c->server_exec = std::make_unique<ThreadExecutor>();
  ServerConfig scfg;
  scfg.pipeline = server_pipeline != 0;
  c->srv = std::make_unique<ServerCore>("A", scfg, c->sexec(), &c->log,
                                        c->net.sender());
  c->net.register_server("A", c->srv.get(), c->sexec());
  if (c->threaded) {
    std::promise<void> p;
    c->server_exec->post([&] {
      c->srv->start();
      p.set_value();
    });
    p.get_future().wait();
  } else {
    c->srv->start();
  }
  c->base_cfg.servers = {"A"};
  c->base_cfg.pipeline = client_pipeline != 0;
  if (chunk_bytes) c->base_cfg.chunk_bytes = chunk_bytes;
  return c;
}

int ref_cluster_add(void* h, const char* replica, std::uint32_t shards,
                    std::uint64_t tiny, std::uint64_t target) {
  auto* c = static_cast<Cluster*>(h);
  auto n = std::make_unique<Node>();
  ClientConfig cfg = c->base_cfg;
  cfg.data_endpoint = std::string("ep:") + replica;
  if (tiny) cfg.manifest.tiny_threshold = tiny;
  if (target) cfg.manifest.group_target = target;
  c->net.register_data(cfg.data_endpoint, &n->serves);
  Executor* ex = &c->sim;
  if (c->threaded) {
    n->texec = std::make_unique<ThreadExecutor>();
    ex = n->texec.get();
  }
  n->core = std::make_unique<ClientCore>("m", replica, shards, cfg, ex,
                                         &c->log, &c->net, &c->net,
                                         &n->serves);
  c->nodes[replica] = std::move(n);
  return 0;
}

// ref_cluster_add with ClientConfig.datacenter and ClientConfig.offload_seed
// (the cross-link seeding scenario, test_client_core.cpp:460-503).
int ref_cluster_add_dc(void* h, const char* replica, std::uint32_t shards, const char* dc,
                       int offload_seed) {
  auto* c = static_cast<Cluster*>(h);
  ref_cluster_add(h, replica, shards, 0, 0);
  auto& n = *c->nodes.at(replica);
  ClientConfig cfg = c->base_cfg;
  cfg.data_endpoint = std::string("ep:") + replica;
  cfg.datacenter = dc;
  cfg.offload_seed = offload_seed != 0;
  Executor* ex = &c->sim;
  if (c->threaded) ex = n.texec.get();
  n.core = std::make_unique<ClientCore>("m", replica, shards, cfg, ex, &c->log, &c->net, &c->net,
                                        &n.serves);
  return 0;
}

int ref_cluster_register(void* h, const char* replica, std::uint32_t shard,
                         const char* name, void* ptr, std::uint64_t len) {
  auto* c = static_cast<Cluster*>(h);
  auto& n = *c->nodes.at(replica);
  return static_cast<int>(n.core->register_tensor(
      shard, name, {static_cast<std::byte*>(ptr), len}));
}

int ref_cluster_register_modeled(void* h, const char* replica,
                                 std::uint32_t shard, const char* name,
                                 std::uint64_t len) {
  auto* c = static_cast<Cluster*>(h);
  auto& n = *c->nodes.at(replica);
  return static_cast<int>(n.core->register_tensor_modeled(shard, name, len));
}

int ref_cluster_publish(void* h, const char* replica, std::uint64_t v,
                        double* secs) {
  auto* c = static_cast<Cluster*>(h);
  auto* core = c->nodes.at(replica)->core.get();
  auto r = c->run_many({[&](ClientCore::OpFn cb) { core->publish(v, cb); }},
                       secs);
  return static_cast<int>(r[0].status);
}

// ClientCore::set_retention (client_core.cpp:528): sent with the handle's
// open (OpenReq.retain), so call before the replica's first operation.
int ref_cluster_set_retention(void* h, const char* replica, const std::uint64_t* lags, int n) {
  auto* c = static_cast<Cluster*>(h);
  auto it = c->nodes.find(replica);
  if (it == c->nodes.end()) return -1;
  RetentionRule rule;
  for (int i = 0; i < n; ++i) rule.lags.insert(lags[i]);
  it->second->core->set_retention(rule);
  return 0;
}

int ref_cluster_open(void* h, const char* replica) {
  auto* c = static_cast<Cluster*>(h);
  auto* core = c->nodes.at(replica)->core.get();
  auto r = c->run_many({[&](ClientCore::OpFn cb) { core->open(cb); }}, nullptr);
  return static_cast<int>(r[0].status);
}

// ClientCore::close (client_core.hpp:93): the replica leaves the cluster
// and stops serving its regions, which the caller may then reuse.
int ref_cluster_close(void* h, const char* replica) {
  auto* c = static_cast<Cluster*>(h);
  auto* core = c->nodes.at(replica)->core.get();
  auto r = c->run_many({[&](ClientCore::OpFn cb) { core->close(cb); }}, nullptr);
  return static_cast<int>(r[0].status);
}

int ref_cluster_unpublish(void* h, const char* replica) {
  auto* c = static_cast<Cluster*>(h);
  auto* core = c->nodes.at(replica)->core.get();
  auto r = c->run_many({[&](ClientCore::OpFn cb) { core->unpublish(cb); }},
                       nullptr);
  return static_cast<int>(r[0].status);
}

// Issues replicate(spec) (update when `update`) on every listed replica at
// the same instant and runs them all to completion. Per replica: status,
// resolved version, changed flag. `secs` = wall time of the whole fan-out.
int ref_cluster_pull_many(void* h, int n, const char** replicas,
                          const char* spec, int update, int* statuses,
                          std::uint64_t* versions, int* changed, double* secs) {
  auto* c = static_cast<Cluster*>(h);
  auto s = VersionSpec::parse(spec);
  if (!s) return static_cast<int>(s.status());
  std::vector<std::function<void(ClientCore::OpFn)>> ops;
  for (int i = 0; i < n; ++i) {
    auto* core = c->nodes.at(replicas[i])->core.get();
    VersionSpec vs = *s;
    if (update)
      ops.push_back([core, vs](ClientCore::OpFn cb) { core->update(vs, cb); });
    else
      ops.push_back(
          [core, vs](ClientCore::OpFn cb) { core->replicate(vs, cb); });
  }
  auto res = c->run_many(std::move(ops), secs);
  for (int i = 0; i < n; ++i) {
    statuses[i] = static_cast<int>(res[i].status);
    versions[i] = res[i].version ? *res[i].version : 0;
    if (changed) changed[i] = res[i].changed ? 1 : 0;
  }
  return 0;
}

// Issues replicate("latest") on the readers first (they park: no version
// exists), then publish(v) on `src`, and runs everything to completion
// (test_server_core.cpp:317-340 scenario through the full client stack).
int ref_cluster_publish_during(void* h, int n, const char** readers, const char* src,
                               std::uint64_t v, int* statuses) {
  auto* c = static_cast<Cluster*>(h);
  std::vector<std::function<void(ClientCore::OpFn)>> ops;
  for (int i = 0; i < n; ++i) {
    auto* core = c->nodes.at(readers[i])->core.get();
    ops.push_back([core](ClientCore::OpFn cb) { core->replicate(VersionSpec::latest(), cb); });
  }
  auto* pub = c->nodes.at(src)->core.get();
  ops.push_back([pub, v](ClientCore::OpFn cb) { pub->publish(v, cb); });
  auto res = c->run_many(std::move(ops), nullptr);
  for (int i = 0; i < n; ++i) statuses[i] = static_cast<int>(res[i].status);
  return static_cast<int>(res[n].status);
}

// Lets queued one-way notices (CompleteMsg, progress) land.
void ref_cluster_settle(void* h) {
  auto* c = static_cast<Cluster*>(h);
  if (!c->threaded) {
    Time horizon = c->sim.now() + std::chrono::milliseconds(50);
    while (c->sim.step(horizon)) {
    }
  } else {
    std::this_thread::sleep_for(std::chrono::milliseconds(50));
  }
}

long ref_cluster_trace(void* h, char* out, std::size_t cap) {
  auto* c = static_cast<Cluster*>(h);
  return copy_out(c->log.render(), out, cap);
}

// Stats (client_core.hpp:44-52): bytes_pulled, bytes_pulled_cross_dc,
// bytes_copied_local, items_verified, checksum_failures, failure_reports,
// failovers.
int ref_cluster_stats(void* h, const char* replica, std::uint64_t* out) {
  auto* c = static_cast<Cluster*>(h);
  auto& n = *c->nodes.at(replica);
  std::promise<ClientCore::Stats> p;
  if (c->threaded) {
    n.texec->post([&] { p.set_value(n.core->stats()); });
  } else {
    p.set_value(n.core->stats());
  }
  auto s = p.get_future().get();
  out[0] = s.bytes_pulled;
  out[1] = s.bytes_pulled_cross_dc;
  out[2] = s.bytes_copied_local;
  out[3] = s.items_verified;
  out[4] = s.checksum_failures;
  out[5] = s.failure_reports;
  out[6] = s.failovers;
  return 0;
}

// Replica view (server_core.hpp:42-50): lifecycle string, version, serving.
long ref_cluster_view(void* h, const char* replica, std::uint64_t* version,
                      std::uint32_t* serving, char* lifecycle, std::size_t cap) {
  auto* c = static_cast<Cluster*>(h);
  std::optional<ServerCore::ReplicaView> v;
  if (c->threaded) {
    std::promise<void> p;
    c->server_exec->post([&] {
      v = c->srv->replica_view("m", replica);
      p.set_value();
    });
    p.get_future().wait();
  } else {
    v = c->srv->replica_view("m", replica);
  }
  if (!v) return -1;
  *version = v->version ? *v->version : 0;
  *serving = v->serving;
  return copy_out(v->lifecycle, lifecycle, cap);
}

void ref_cluster_free(void* h) {
  auto* c = static_cast<Cluster*>(h);
  if (c->threaded) {
    for (auto& [k, n] : c->nodes) n->texec->stop();
    c->server_exec->stop();
  }
  c->nodes.clear();
  if (!c->threaded) c->srv->stop();
  c->srv.reset();
  delete c;
}

}  // extern "C"
