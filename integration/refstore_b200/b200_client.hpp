// refstore/b200_client.hpp -- level A integration: a
// ClientCore-shaped handle for device-resident weights, backed by the B200
// read path's C ABI (include/ros_b200.h).
//
// This is the reference-side binding a maintainer would add next to
// /root/reference/proj/include/refstore/client_core.hpp.  It compiles against
// the reference's own headers (Status, VersionSpec, ClientCore::OpResult,
// ListingMap) and mirrors ClientCore's operation surface
// (client_core.hpp:82-93: open/publish/unpublish/replicate/update/list/close)
// and Stats (client_core.hpp:44-52).  The C ABI is blocking, so every
// callback completes inline on the caller's thread.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <chrono>
#include <cstdio>
#include <string>

#include "refstore/client_core.hpp"
#include "refstore/messages.hpp"
#include "refstore/types.hpp"
#include "ros_b200.h"

namespace refstore {

// ServerCore + ServeRegistry of this process (one per process).
class B200Cluster {
 public:
  explicit B200Cluster(bool pipeline = true, bool smart_skipping = true) {
    check(rs_cluster_create(pipeline, smart_skipping, &c_));
  }
  ~B200Cluster() {
    if (c_) rs_cluster_destroy(c_);
  }
  B200Cluster(const B200Cluster&) = delete;
  B200Cluster& operator=(const B200Cluster&) = delete;
  rs_cluster* get() const { return c_; }

  // ServerCore::listing (server_core.hpp:52), parsed from "v:rep,rep;...".
  ListingMap listing(const std::string& model) const {
    std::size_t n = 0;
    rs_cluster_listing(c_, model.c_str(), nullptr, 0, &n);
    std::string s(n, '\0');
    rs_cluster_listing(c_, model.c_str(), s.data(), s.size(), &n);
    ListingMap out;
    std::size_t p = 0;
    while (p < s.size()) {
      std::size_t e = s.find(';', p);
      if (e == std::string::npos) e = s.size();
      std::string part = s.substr(p, e - p);
      std::size_t colon = part.find(':');
      if (colon != std::string::npos) {
        auto& reps = out[std::stoull(part.substr(0, colon))];
        std::size_t q = colon + 1;
        while (q < part.size()) {
          std::size_t c = part.find(',', q);
          if (c == std::string::npos) c = part.size();
          if (c > q) reps.insert(part.substr(q, c - q));
          q = c + 1;
        }
      }
      p = e + 1;
    }
    return out;
  }

  // ServerCore::replica_view (server_core.hpp:41-51): lifecycle + version.
  std::optional<ServerCore::ReplicaView> replica_view(const std::string& model,
                                                      const std::string& replica) const {
    char life[16] = {};
    std::uint64_t v = 0;
    std::uint32_t serving = 0;
    int visible = 0;
    if (rs_cluster_view(c_, model.c_str(), replica.c_str(), life, &v, &serving, &visible) != 0)
      return std::nullopt;
    ServerCore::ReplicaView out;
    out.lifecycle = life;
    out.kind = "worker";
    if (v) out.version = v;
    out.serving = serving;
    out.visible = visible != 0;
    return out;
  }

  static void check(int s) {
    if (s) throw std::runtime_error(rs_status_name(s));
  }

 private:
  rs_cluster* c_ = nullptr;
};

class B200Client {
 public:
  using OpResult = ClientCore::OpResult;
  using OpFn = ClientCore::OpFn;

  B200Client(B200Cluster& cluster, std::string model, std::string replica,
             std::uint32_t num_shards)
      : B200Client(cluster, std::move(model), std::move(replica), num_shards, ClientConfig{}) {}
  // The ClientCore constructor's ClientConfig (config.hpp:23-47): the knobs
  // that shape the read path carry over; chunk_bytes (the reference's pull
  // window) does not -- the device path digests 4 KiB chunks.
  B200Client(B200Cluster& cluster, std::string model, std::string replica,
             std::uint32_t num_shards, const ClientConfig& rc)
      : cluster_(cluster), model_(std::move(model)), replica_(std::move(replica)) {
    rs_config cfg;
    rs_config_default(&cfg);
    cfg.tiny_threshold = rc.manifest.tiny_threshold;
    cfg.group_target = rc.manifest.group_target;
    cfg.pipeline = rc.pipeline ? 1 : 0;
    cfg.checksum_retries = rc.checksum_retries;
    cfg.pull_timeout_s = std::chrono::duration<double>(rc.pull_timeout).count();
    std::snprintf(cfg.datacenter, sizeof(cfg.datacenter), "%s", rc.datacenter.c_str());
    cfg.offload_seed = rc.offload_seed ? 1 : 0;
    B200Cluster::check(rs_open(cluster.get(), model_.c_str(), replica_.c_str(), num_shards, &cfg, &h_));
  }
  ~B200Client() {
    if (h_) rs_close(h_);
  }
  B200Client(const B200Client&) = delete;
  B200Client& operator=(const B200Client&) = delete;

  // register_tensor (client_core.hpp:72-73): `region` is device memory,
  // caller-owned, and must outlive the handle (weights live in place).
  Status register_tensor(std::uint32_t shard, const std::string& name, std::span<std::byte> region) {
    return Status(rs_register(h_, shard, name.c_str(), region.data(), region.size()));
  }

  void open(OpFn done) { done(result(rs_connect(h_))); }
  void publish(VersionId v, OpFn done) {
    OpResult r = result(rs_publish(h_, v));
    if (r.status == Status::ok) r.version = v;
    done(std::move(r));
  }
  void unpublish(OpFn done) { done(result(rs_unpublish(h_))); }
  void replicate(VersionSpec spec, OpFn done, double wait_s = 60.0) {
    std::uint64_t v = 0;
    OpResult r = result(rs_replicate(h_, spec.to_string().c_str(), wait_s, &v));
    if (r.status == Status::ok) r.version = v;
    done(std::move(r));
  }
  void update(VersionSpec spec, OpFn done, double wait_s = 60.0) {
    std::uint64_t v = 0;
    int changed = 0;
    OpResult r = result(rs_update(h_, spec.to_string().c_str(), wait_s, &changed, &v));
    if (r.status == Status::ok && v) r.version = v;
    r.changed = changed != 0;
    done(std::move(r));
  }
  void list(OpFn done) {
    OpResult r;
    r.listing = cluster_.listing(model_);
    done(std::move(r));
  }
  void close(OpFn done) {
    OpResult r = result(h_ ? rs_close(h_) : static_cast<int>(Status::closed));
    h_ = nullptr;
    done(std::move(r));
  }

  std::optional<VersionId> current_version() const {
    std::uint64_t v = 0;
    if (!h_ || rs_current_version(h_, &v) != 0) return std::nullopt;
    return v;
  }
  bool is_published() const { return h_ && rs_is_published(h_); }
  // ClientCore::Stats (client_core.hpp:44-52): the same seven counters.
  ClientCore::Stats stats() const {
    rs_stats s{};
    ClientCore::Stats out;
    if (!h_ || rs_stats_get(h_, &s) != 0) return out;
    out.bytes_pulled = s.bytes_pulled;
    out.bytes_pulled_cross_dc = s.bytes_pulled_cross_dc;
    out.bytes_copied_local = s.bytes_copied_local;
    out.items_verified = s.items_verified;
    out.checksum_failures = s.checksum_failures;
    out.failure_reports = s.failure_reports;
    out.failovers = s.failovers;
    return out;
  }
  rs_handle* handle() const { return h_; }
  // The reference client reacts to offload_release directives on its
  // executor; a blocking handle applies them here (and waits for a running
  // seed fill's report first).
  void poll() {
    if (!h_) return;
    rs_seed_wait(h_);
    rs_poll(h_);
  }

 private:
  static OpResult result(int st) {
    OpResult r;
    r.status = Status(st);
    return r;
  }
  B200Cluster& cluster_;
  std::string model_, replica_;
  rs_handle* h_ = nullptr;
};

}  // namespace refstore
