// Version registry + transfer planner: the metadata half of ROS.
//
// This is the subset of the reference ServerCore
// (/root/reference/proj/src/server_core.cpp) that decides WHERE a reader
// pulls from: replica lifecycle, version availability with smart skipping
// (available_versions 1487-1515), source choice (pick_source 1517-1543),
// settle-time re-validation (settle_source 1007-1037), assignment building
// (make_assignment 1545-1557), parked-replicate wake order (wake_blocked
// 1565-1587), completion/drain (on_complete 1142-1175, finish_replication
// 1177-1204, release_source 1206-1216, check_drain 1218-1226) and failure
// reassignment (on_failure_report 1291-1382, fail_replica 1682-1711).
//
// Differences by design (B200 in-box path):
//  * Group transactions arrive whole: one call carries every shard of a
//    replica, so there is no straggler assembly / txn timeout machinery.
//  * Calls are synchronous and deterministic.  A caller whose op parks
//    (replicate before a version exists, unpublish/update waiting for readers
//    to drain) gets Status::ok with `pending` set and later reads the outcome
//    with op_result(); with several threads it may block in wait_op().  The
//    same call sequence applied on every rank (replicated state machine,
//    paper_2604_09107_b200/ros.py Cluster) yields the same plan everywhere.
//  * Retention offloads follow the reference (unpublish_needs_offload
//    1606-1618, on_offload_confirm 1387-1437, create_offload_replica
//    1439-1485, eval_offload_releases 1620-1645), and so do cross-link seed
//    buffers (update's seed start 915-970, role-seed progress/complete
//    1124-1175, consumption and release 1177-1204; find_seed_replica 88-99):
//    a replica opened with offload_seed whose update source sits in another
//    datacenter fills "<replica>+seed@<v>" in host memory in the background,
//    stays on its version, and consumes the seed locally on a later update.
//  * pick_source's key gains a topology cost between dc and serving; on a
//    uniform NVSwitch box every cost is equal and the order is exactly the
//    reference's (own_seed, same_dc, serving, last_assigned, name).
#pragma once

#include <condition_variable>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <set>
#include <string>
#include <vector>

#include "common.hpp"

namespace rsb {

// Layout keys: "" is the reference's single slicing, "L<hash>" another
// slicing (layout.hpp).  A leading '!' marks a terminal replica -- one whose
// regions receive a cast of the version (K5, bf16 -> e4m3): it pulls like a
// replica of the slicing after the '!', but never serves or publishes.
inline bool terminal_layout(const std::string& k) { return !k.empty() && k[0] == '!'; }
inline std::string slicing(const std::string& k) { return terminal_layout(k) ? k.substr(1) : k; }

// messages.hpp:40-52, plus the layout fields of the B200 path.
struct Assignment {
  VersionId version = 0;
  std::string source_replica;
  std::string source_endpoint;
  bool source_complete = false;
  bool cross_dc = false;
  bool seeding = false;
  bool local_seed_consume = false;
  std::string manifest;  // encoded Manifest of this shard ("" on a reshard)
  std::string layout;    // encoded ShardLayout of this shard (chunk lengths)
  // Early publish: the manifest's big-entry digests are not computed yet (0);
  // the publisher commits them later (Registry::finalize_manifests).
  bool provisional = false;
  // Reshard (the source's slicing differs from the reader's): every source
  // shard's manifest, layout and endpoint.  The blobs are shared with the
  // registry (tens of KB per shard: an outcome is copied several times on its
  // way to the client, and a rebind compares them).
  bool reshard = false;
  using Blobs = std::shared_ptr<const std::vector<std::string>>;
  Blobs all_manifests, all_layouts;
  std::vector<std::string> all_endpoints;
};

enum class OpKind : std::uint8_t { none, publish, unpublish, replicate, update };

// SeedStart (messages.hpp): a background host-memory fill the client starts
// for every shard while its update reports no change.
struct SeedStart {
  VersionId version = 0;
  std::string source;
  std::vector<Assignment> assignments;  // per shard, seeding = true
};

struct OpOutcome {
  bool done = false;
  Status status = Status::ok;
  std::optional<VersionId> version;
  bool changed = false;                 // update
  std::vector<Assignment> assignments;  // replicate/update(change): per shard
  // Set while an unpublish/update waits for the client to park this version
  // in host memory first (ResponseKind::offload_first, server_core.cpp:428-440):
  // the client answers with offload_confirm for every shard.
  std::optional<VersionId> offload_first;
  // update without change: the seed fill to start (server_core.cpp:483-494)
  std::optional<SeedStart> seed;
};

// A retention offload the owner may now free (DirectiveKind::offload_release).
struct OffloadRelease {
  std::string owner;
  VersionId version = 0;
  bool seed = false;  // OffloadPurpose::seed (else retention)
};

struct ReplicaView {
  std::string kind = "worker";  // worker|offload
  std::string lifecycle;  // registered|replicating|published|failed
  std::optional<VersionId> version;
  std::uint32_t serving = 0;
  bool visible = false;
  bool seeding = false;
  std::uint64_t min_progress = 0;
  std::string source;
};

struct TraceLine {
  std::uint64_t seq = 0;
  std::string kind;
  std::vector<std::pair<std::string, std::string>> kv;
  std::string format() const;
};

class Registry {
 public:
  struct Config {
    bool pipeline = true;
    bool smart_skipping = true;
  };
  // Returns a topology cost (lower = closer) between two data endpoints;
  // default: every pair costs 0.
  using TopoFn = std::function<int(const std::string& reader_ep,
                                   const std::string& source_ep)>;

  explicit Registry(Config cfg);

  void set_topology(TopoFn fn);

  // `layout` keys the replica's slicing ("" = plain, the reference's only
  // kind).  Replicas with equal keys pull item-for-item (and may chase each
  // other); a reader with a different non-empty key reshards from complete
  // copies.
  // A reshard-capable replica also hands over its derived per-shard
  // manifests/layouts (they depend only on its registrations); they become a
  // layout of version v the moment it is assigned a differently sliced
  // source, so same-slicing readers can chase it in the same round.
  Status open(const std::string& model, const std::string& replica,
              std::uint32_t num_shards, const std::string& dc,
              const std::vector<std::string>& endpoints, const std::string& layout = "",
              const std::vector<std::string>& derived_manifests = {},
              const std::vector<std::string>& derived_layouts = {});
  Status close(const std::string& model, const std::string& replica);
  // RetentionRule (types.hpp:119-123): versions at these lags behind the
  // newest published one stay reachable -- the last durable copy of such a
  // version is parked in host memory (an offload replica) before it goes.
  Status set_retention(const std::string& model, const std::string& replica,
                       const std::set<std::uint64_t>& lags);
  // ClientConfig.offload_seed (OpenReq.offload_seed, server_core.cpp:230).
  Status set_offload_seed(const std::string& model, const std::string& replica, bool on);
  // OffloadConfirmMsg (server_core.cpp:1387-1437): the shard parked
  // `version` in host memory (ok) and serves it at `endpoint`.
  Status offload_confirm(const std::string& model, const std::string& replica,
                         std::uint32_t shard, VersionId version, bool ok,
                         const std::string& endpoint);
  // Offload buffers of `owner` the registry no longer needs (drained).
  std::vector<OffloadRelease> take_releases(const std::string& model, const std::string& owner);

  // Each returns the immediate status; if ok and the op is parked,
  // *pending = true and the outcome arrives through op_result().
  // provisional: an early publish (ClientConfig.early_publish) -- the
  // manifests' big-entry digests are still being computed; readers may bind
  // and pull (they verify chunk by chunk), and finalize_manifests commits
  // the reference-identical bytes later.
  Status publish(const std::string& model, const std::string& replica,
                 VersionId v, const std::vector<std::string>& manifests,
                 OpOutcome* out, const std::vector<std::string>& layouts = {},
                 bool provisional = false);
  // Commits the final manifests of an early publish: same structure as the
  // provisional ones (entries, packing), digests filled in.  A final version
  // accepts only identical bytes.
  Status finalize_manifests(const std::string& model, const std::string& replica, VersionId v,
                            const std::vector<std::string>& manifests);
  // The manifest bytes of version v for a slicing key's shard, and whether
  // they are final (not an early publish still digesting).
  Status current_manifest(const std::string& model, VersionId v, const std::string& layout_key,
                          std::uint32_t shard, std::string* bytes, bool* final_bytes);
  // The same, for the slicing `replica` was opened with (a replica whose
  // shards live in several processes has its key only in the registry).
  Status replica_manifest(const std::string& model, const std::string& replica, VersionId v,
                          std::uint32_t shard, std::string* bytes, bool* final_bytes);
  // A resharding reader registers the derived manifests/layouts of its own
  // slicing so readers of the same slicing can later pull from it.
  Status add_layout(const std::string& model, VersionId v, const std::string& layout_key,
                    const std::vector<std::string>& manifests,
                    const std::vector<std::string>& layouts);
  Status unpublish(const std::string& model, const std::string& replica,
                   OpOutcome* out);
  Status replicate(const std::string& model, const std::string& replica,
                   const VersionSpec& spec, OpOutcome* out);
  Status update(const std::string& model, const std::string& replica,
                const VersionSpec& spec, std::optional<VersionId> current,
                OpOutcome* out);

  // Transfer lifecycle reports from the reader (ProgressMsg / CompleteMsg).
  // seed = TransferRole::seed: the report is about the replica's seed fill
  // of `seed_version` (ignored when its seed moved on to another version).
  void progress(const std::string& model, const std::string& replica,
                std::uint32_t shard, std::uint64_t items, bool seed = false,
                VersionId seed_version = 0);
  void complete(const std::string& model, const std::string& replica,
                std::uint32_t shard, Status outcome, bool seed = false,
                VersionId seed_version = 0);
  // FailureReportMsg: reason 0 = timeout, 1 = checksum.  On success returns
  // the replacement assignment for `shard`.
  Result<Assignment> failure_report(const std::string& model,
                                    const std::string& replica,
                                    std::uint32_t shard,
                                    const std::string& failed_replica,
                                    int reason);

  // Dry-run plan view: which source `replica` would be assigned for `spec`
  // right now (no counters move).
  Result<Assignment> locate(const std::string& model, const std::string& replica,
                            const VersionSpec& spec, std::uint32_t shard);
  // The replicating replica's current assignment for `shard` (after
  // failure_report retargets it).
  Result<Assignment> current_assignment(const std::string& model,
                                        const std::string& replica, std::uint32_t shard);

  // Outcome of the replica's most recent op (done=false while parked).
  OpOutcome op_result(const std::string& model, const std::string& replica);
  // Blocks until that op is done or `timeout_s` passes (multi-threaded use).
  OpOutcome wait_op(const std::string& model, const std::string& replica,
                    double timeout_s);

  std::map<VersionId, std::set<std::string>> listing(const std::string& model);
  std::optional<ReplicaView> view(const std::string& model,
                                  const std::string& replica);
  std::vector<TraceLine> trace();
  std::string trace_text();

 private:
  enum class Life { registered, replicating, published, failed };
  enum class Kind { worker, offload };
  struct Txn {
    OpKind kind = OpKind::none;
    std::uint64_t order = 0;
    VersionSpec spec;
    std::optional<VersionId> current;  // update: caller's held version
    bool blocked = false, resolved = false, settled = false, changed = false;
    bool was_visible = false;
    std::optional<VersionId> target;
    std::string source;
    // retention offload of the held version before the op settles
    bool offload_needed = false, offload_done = false;
    VersionId offload_v = 0;
    std::set<std::uint32_t> offload_confirmed;
    std::vector<std::string> offload_endpoints;
  };
  struct ShardState {
    std::uint64_t progress = 0;
    bool complete = false;
  };
  struct Rep {
    Kind kind = Kind::worker;
    std::string owner;        // offload: the worker whose buffer this is
    bool releasing = false;   // offload: released, draining its readers
    bool seed = false;        // offload: OffloadPurpose::seed (else retention)
    VersionId offload_v = 0;  // offload: the version the buffer holds
    bool offload_seed = false;  // worker: ClientConfig.offload_seed
    std::set<std::uint64_t> retain;  // retention lags requested by this replica
    std::string model, name, dc;
    std::string layout;  // slicing key ("" plain)
    std::vector<std::string> derived_manifests, derived_layouts;  // reshard readers
    std::uint32_t num_shards = 1;
    std::vector<std::string> endpoints;
    Life life = Life::registered;
    bool visible = false, seeding = false;
    std::optional<VersionId> version, last_published;
    std::string source;
    std::uint32_t serving = 0;
    std::uint64_t last_assigned = 0;
    std::vector<ShardState> shards;
    std::optional<Txn> txn;  // in-flight op (one per replica)
    OpOutcome last;          // outcome of the latest op
    bool complete_all() const {
      for (const auto& s : shards)
        if (!s.complete) return false;
      return true;
    }
  };
  struct LayoutInfo {
    std::uint32_t num_shards = 0;
    std::vector<std::string> manifests;
    std::vector<std::string> layouts;
    bool provisional = false;  // early publish: big-entry digests still pending
    // shared snapshots handed to reshard assignments (reset when the
    // manifests change)
    Assignment::Blobs man_sp, lay_sp;
  };
  struct VersionInfo {
    std::map<std::string, LayoutInfo> by_layout;  // slicing key -> per-shard metadata
  };
  struct ModelState {
    std::map<std::string, std::unique_ptr<Rep>> reps;
    std::map<VersionId, VersionInfo> versions;
    std::optional<VersionId> max_published;
  };

  ModelState& ms(const std::string& model) { return models_[model]; }
  Rep* find(const std::string& model, const std::string& replica);
  void trace(std::string kind,
             std::vector<std::pair<std::string, std::string>> kv);
  static const char* life_name(Life l);

  std::set<VersionId> available(ModelState& m, const std::string& dc);
  Rep* pick_source(ModelState& m, VersionId v, const Rep& reader);
  bool still_good(const Rep& cand, const Rep& reader, VersionId v) const;
  Rep* settle_source(Rep& r, Txn& t);
  Assignment make_assignment(ModelState& m, Rep& src, VersionId v,
                             std::uint32_t shard, const Rep& reader);
  bool servable(ModelState& m, VersionId v, const Rep& reader);
  void start_replicate(Rep& r);
  void start_update(Rep& r);
  void try_settle(Rep& r);
  void apply_settle(Rep& r);
  void finish_op(Rep& r, Status st);
  void settle_ok(Rep& r);
  void wake_blocked(const std::string& model);
  void release_source(Rep& r);
  void check_drain(Rep& src);
  void finish_replication(Rep& r);
  void void_replication(Rep& r, const std::string& reason);
  void fail_replica(Rep& r, const std::string& reason);
  void prune_version(ModelState& m, VersionId v);
  std::set<VersionId> retained_versions(ModelState& m);
  bool needs_offload(ModelState& m, const Rep& r, VersionId v);
  void request_offload(Rep& r, Txn& t, VersionId v);
  void create_offload_replica(Rep& owner, VersionId v, const std::vector<std::string>& endpoints);
  void eval_offload_releases(const std::string& model);
  void release_offload(Rep& off);
  void finish_offload_release(Rep& off);
  Rep* find_seed(const Rep& owner);

  std::map<std::string, std::vector<OffloadRelease>> releases_;  // model -> pending directives
  Config cfg_;
  TopoFn topo_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::map<std::string, ModelState> models_;
  std::vector<TraceLine> trace_;
  std::uint64_t tick_ = 0;   // assign tick (last_assigned)
  std::uint64_t order_ = 0;  // op arrival order (wake_blocked)
};

}  // namespace rsb
