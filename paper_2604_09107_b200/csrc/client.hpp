// Reader/publisher side of the B200 ROS read path: one replica's shard
// handles, their registered device regions, the serve state peers chase, and
// the device transfer loop.
//
// Mirrors the data-path parts of the reference ClientCore
// (/root/reference/proj/include/refstore/client_core.hpp:35-104):
//   register_tensor            client_core.hpp:72-73
//   build_publish_payload      client_core.cpp:1547-1579  -> prepare_publish
//   bind_receive_payload       client_core.cpp:1581-1622  -> bind()
//   serve_payload/payload_spans client_core.cpp:1624-1670 -> serve()
//   TransferTask (step/issue_pull/verify_ready/item_failed/retarget)
//                              client_core.cpp:47-492     -> fill_shards()
//   task_progress / task_done  client_core.cpp:1414-1542
// and of the transport boundary (transport.hpp:53-156): ServeRegistry,
// PeerServeState, compute_slice / copy_slice_locked (the latter two become
// the device pull kernel over peer-mapped source spans).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "common.hpp"
#include "device.hpp"
#include "manifest.hpp"
#include "layout.hpp"
#include "registry.hpp"

namespace rsb {

class StreamSource;  // stream.hpp: a source reached over TCP

struct ClientConfig {
  std::uint64_t chunk_bytes = 4096;  // digest + watermark unit (multiple of 16)
  PackLimits limits;                 // tiny-tensor packing (config.hpp:46)
  bool pipeline = true;              // serve partially landed fills
  int checksum_retries = 3;          // failure reports per fill (config.hpp:42)
  double pull_timeout_s = 4.0;       // upstream silence before reporting
  std::string dc = "dc0";
  std::uint32_t reshard_align = 2;   // chunk rule: TP splits up to this stay chunk aligned
  std::uint32_t grid_sms = 0;        // SMs a fill's persistent kernel may occupy (0: all)
  // Early publish: commit the chunk-digest table and the manifest structure
  // at once (readers bind and pull, verifying chunk by chunk) and the
  // big-entry XXH64 digests -- a serial chain per entry, ~0.43 s for the
  // 1.05 GB Llama-3-8B embedding -- when they are done.  The committed
  // manifest is the reference's, byte for byte; only its arrival is later.
  bool early_publish = false;
  // Host-memory seeding (ClientConfig.offload_seed, config.hpp): an update
  // whose source is in another datacenter fills "<replica>+seed@<v>" in
  // pinned host memory in the background and stays on its version; a later
  // update consumes the seed locally (PCIe, no cross-link traffic).
  bool offload_seed = false;
};

// Owned device allocation.
struct DevBuf {
  void* p = nullptr;
  std::size_t n = 0;
  int dev = -1;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), dev(o.dev) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      this->~DevBuf();
      p = o.p;
      n = o.n;
      dev = o.dev;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf();
  Status alloc(int device, std::size_t bytes);
};

// Item -> digest chunks.  Chunks are item-relative; chunk j of item i covers
// [j*len_i, min((j+1)*len_i, item_len)).  Batches of 32 chunks carry one
// watermark flag.  Every item starts a new batch (its first chunk index is a
// multiple of 32), so a batch never spans items; the unused indices between
// items are holes (no bytes, no digest).
struct ChunkMap {
  std::vector<std::uint32_t> chunk0;     // n_items + 1 prefix (batch aligned)
  std::vector<std::uint32_t> chunk_len;  // per item (0: member-cut, see parts)
  std::vector<std::uint32_t> count;      // real chunks per item
  // Per item: its runs when member-cut (layout.hpp member rule), else empty.
  // Derived from the manifest and the layout, so not compared.
  std::vector<std::vector<ChunkPart>> parts;
  std::uint32_t n_chunks() const { return chunk0.empty() ? 0 : chunk0.back(); }
  std::uint32_t n_batches() const {
    return (n_chunks() + dev::kBatchChunks - 1) / dev::kBatchChunks;
  }
  std::uint64_t n_real() const {
    std::uint64_t n = 0;
    for (auto c : count) n += c;
    return n;
  }
  static ChunkMap uniform(const Manifest& m, std::uint64_t chunk_bytes);
  // lens: per item (0: member-cut, with member_lens per entry).
  static ChunkMap from_lens(const Manifest& m, const std::vector<std::uint32_t>& lens,
                            const std::vector<std::uint32_t>& member_lens = {});
  static ChunkMap from_layout(const Manifest& m, const ShardLayout& lay, std::uint64_t chunk_bytes,
                              std::uint32_t align);
  bool cut(std::size_t i) const { return i < parts.size() && !parts[i].empty(); }
  bool any_cut() const {
    for (const auto& p : parts)
      if (!p.empty()) return true;
    return false;
  }
  // The runs of item i (a single run for a uniform item).
  std::vector<ChunkPart> runs(std::size_t i, std::uint64_t item_len) const {
    if (cut(i)) return parts[i];
    return {ChunkPart{0, item_len, chunk_len[i], 0}};
  }
  bool operator==(const ChunkMap& o) const {
    return chunk0 == o.chunk0 && chunk_len == o.chunk_len && count == o.count;
  }
};

// PeerServeState (transport.hpp:53-69) with device-resident watermarks.
// Host fields are guarded by `m`; the device watermark words are the
// authoritative progress for chasing readers.
struct ServeState {
  std::mutex m;
  bool serving = false;
  VersionId version = 0;
  std::uint64_t progress = 0;  // verified items (host view)
  bool complete = false;
  int device = -1;
  int pid = 0;
  std::vector<std::uint64_t> item_ends;  // stream end offset per item
  std::vector<std::uint64_t> item_ptrs;  // device address per item (owner VA)
  ChunkMap cmap;
  std::uint64_t digests = 0;  // device u64[n_chunks]
  std::uint64_t flags = 0;    // device u32[n_batches]
  std::uint32_t epoch = 0;    // current fill epoch (flags == epoch: landed)
  // Imported (other process) state: IPC handles per allocation.
  bool imported = false;
  struct Alloc {
    cudaIpcMemHandle_t handle;
    std::uint64_t size = 0;
  };
  std::vector<Alloc> allocs;
  std::vector<std::pair<std::uint32_t, std::uint64_t>> item_loc;  // (alloc, offset)
  std::pair<std::uint32_t, std::uint64_t> digests_loc{0, 0}, flags_loc{0, 0};
  // A retention offload in pinned host memory (device < 0): a POSIX shared
  // memory segment registered with CUDA, so other processes map it by name.
  std::string host_name;
  std::uint64_t host_size = 0;
  std::uint64_t host_base = 0;  // owner's mapping (offsets in the blob are from here)
};

// Owned pinned host buffer backed by POSIX shared memory (mapped into the
// device address space with cudaHostRegister).
struct HostBuf {
  std::string name;
  void* p = nullptr;
  std::size_t n = 0;
  HostBuf() = default;
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  ~HostBuf();
  Status alloc(std::size_t bytes);
};

// (model, replica, shard) -> serve state, process-wide (transport.hpp:72-85).
class ServeRegistry {
 public:
  static std::string key(const std::string& model, const std::string& replica,
                         std::uint32_t shard);
  std::shared_ptr<ServeState> ensure(const std::string& k);
  std::shared_ptr<ServeState> find(const std::string& k) const;
  void erase(const std::string& k);
  // Cross-process: serialize a local state / install a remote one.
  Result<std::string> export_state(const std::string& k);
  Status import_state(const std::string& blob);
  // Fault hook: a silent replica's serve states never answer
  // (MemNetwork::set_data_silent, transport_mem.hpp:33-46).
  void set_silent(const std::string& model, const std::string& replica, bool on);
  bool is_silent(const std::string& k) const;

 private:
  mutable std::mutex m_;
  std::map<std::string, std::shared_ptr<ServeState>> map_;
  std::set<std::string> silent_;  // "model|replica|" prefixes
};

// Source addresses as the reader's device sees them.
struct SourceView {
  int device = -1;  // GPU holding the source (-1: host memory)
  std::vector<std::uint64_t> item_ptrs;
  std::uint64_t digests = 0;
  std::uint64_t flags = 0;
  std::uint32_t epoch = 0;
  ChunkMap cmap;
  std::uint64_t total = 0;
};

struct ClientStats {
  std::uint64_t bytes_pulled = 0;
  std::uint64_t bytes_pulled_cross_dc = 0;
  std::uint64_t bytes_copied_local = 0;
  std::uint64_t items_verified = 0;
  std::uint64_t checksum_failures = 0;
  std::uint64_t failure_reports = 0;
  std::uint64_t failovers = 0;
  // device timing of the most recent fill / publish (CUDA events)
  float last_pull_ms = 0;
  float last_publish_ms = 0;
  std::uint64_t last_pull_bytes = 0;
  std::uint32_t last_pull_launches = 0;
  std::uint64_t h2d_bytes = 0;  // descriptor uploads (cumulative)
  std::uint64_t d2h_bytes = 0;  // status / digest read-backs (cumulative)
  // the last fill round over every local shard
  float fill_max_ms = 0, fill_sum_ms = 0;
  std::uint64_t fill_bytes = 0;
  std::uint64_t kernel_launches = 0;  // every kernel this client launched
};

class Client {
 public:
  Client(Registry* reg, ServeRegistry* serves, std::string model, std::string replica,
         std::uint32_t num_shards, ClientConfig cfg);
  ~Client();

  // cast: the region receives the version's bf16 bytes (len of them) as
  // e4m3 (len/2 bytes at ptr, K5); the replica becomes terminal (never serves
  // or publishes; layout key "!" + its slicing).
  Status register_tensor(std::uint32_t shard, const std::string& name, void* ptr,
                         std::uint64_t len, const Geometry& geo = {}, bool cast = false);
  // RetentionRule: versions at these lags behind the newest stay reachable
  // (sent with open; the split phase sends it as its own registry op).
  void set_retention(std::set<std::uint64_t> lags) { retain_ = std::move(lags); }
  const std::set<std::uint64_t>& retention() const { return retain_; }
  void set_shard_endpoint(std::uint32_t shard, std::string ep);
  // Slicing key of the replica ("" when no region carries a geometry;
  // "!" prefix when some region lands as a cast).  combine_layout_key of
  // every shard's shard_hash: a replica whose shards live in several
  // processes gets the same key from the gathered per-shard hashes.
  std::string layout_key() const;
  struct ShardHash {
    std::uint64_t hash = 0;
    bool geometry = false;  // some region of the shard carries a geometry
    bool cast = false;      // some region of the shard lands as e4m3
  };
  ShardHash shard_hash(std::uint32_t shard) const;
  static std::string combine_layout_key(const std::vector<ShardHash>& shards);
  bool terminal() const;  // some local region lands as a cast
  // A shard is local when this process registered its regions.  A replica
  // whose shards live in several processes (one process per GPU) has a
  // Client in each, every one driving only its local shards; the split-phase
  // calls then skip the others.
  bool is_local(std::uint32_t shard) const {
    return shard < num_shards_ && shards_[shard].device >= 0;
  }
  void set_stream(std::uint32_t shard, cudaStream_t s);

  // --- blocking ops (in-process registry) ---------------------------------
  Status open();
  Status publish(VersionId v);
  Status unpublish();
  Status replicate(const VersionSpec& spec, VersionId* out, double wait_s);
  Status update(const VersionSpec& spec, bool* changed, VersionId* out, double wait_s);
  Status close();

  // --- split phase (caller drives the registry, e.g. replicated across
  //     processes) -----------------------------------------------------------
  Status prepare_publish(VersionId v, std::vector<std::string>* manifests,
                         std::vector<std::string>* layouts = nullptr);
  // After bind_all on a reshard: the derived manifests/layouts of this
  // replica's slicing (to register with Registry::add_layout).
  bool derived_layout(std::vector<std::string>* manifests, std::vector<std::string>* layouts) const;
  // The derived manifests/layouts of this replica's own slicing (empty for a
  // plain replica), computed from its registrations; sent with open.
  Status derived_blobs(std::vector<std::string>* manifests,
                       std::vector<std::string>* layouts) const;
  Result<std::string> layout_bytes(std::uint32_t shard) const;
  void commit_publish(VersionId v, Status st);
  // Binds every shard to its assignment and starts serving the (empty)
  // fill so downstream readers can chase it.
  Status bind_all(const std::vector<Assignment>& a, VersionId v);
  // One attempt of every shard's fill.  Per-shard status; reason: 0 timeout
  // / not serving, 1 checksum.
  struct FillOutcome {
    Status status = Status::ok;
    int reason = 0;
    std::uint32_t bad_chunk = 0;
  };
  std::vector<FillOutcome> fill_shards(const std::vector<Assignment>& a,
                                       const std::vector<std::uint32_t>& which);
  // fill_shards in two halves: launch the shards' pull kernels (returns at
  // once), then wait for them and unpack.  Between the two, progress() reads
  // a running fill's verified-batch count (elastic joins key off it).
  void launch_shards(const std::vector<Assignment>& a, const std::vector<std::uint32_t>& which);
  std::vector<FillOutcome> wait_shards(const std::vector<std::uint32_t>& which);
  Status progress(std::uint32_t shard, std::uint32_t* batches_done, std::uint32_t* n_batches);
  // The assignment the shard's latest fill was launched on (null: none yet).
  const Assignment* launched_assignment(std::uint32_t shard) const {
    return shard < launch_as_.size() && launch_as_[shard] ? &*launch_as_[shard] : nullptr;
  }
  void finish_transfers(VersionId v, bool ok);
  void stop_serving();
  // Forget held bytes: the next fill of any version re-pulls everything
  // (a new fill epoch invalidates every landed watermark).
  void invalidate();

  std::optional<VersionId> current_version() const { return current_; }
  bool is_published() const { return published_; }
  ClientStats stats() const {
    ClientStats s = stats_;
    const std::uint64_t seeded = seed_cross_dc_.load();  // background seed fills
    s.bytes_pulled += seeded;
    s.bytes_pulled_cross_dc += seeded;
    return s;
  }
  const std::string& model() const { return model_; }
  const std::string& replica() const { return replica_; }
  std::uint32_t num_shards() const { return num_shards_; }
  Result<std::string> manifest_bytes(std::uint32_t shard);
  Result<std::string> held_manifest(std::uint32_t shard) const;  // no wait (provisional bytes)
  // Early publish: wait for this publisher's big-entry digests and commit
  // the final manifests (rs_publish_finalize); the final bytes per local
  // shard when manifests != null.
  Status finalize_publish(double wait_s, std::vector<std::string>* manifests = nullptr);
  // The last publish still digests its big entries in the background.
  bool publish_pending() const;
  void set_early_publish(bool on) { cfg_.early_publish = on; }
  Status chunk_digests(std::uint32_t shard, std::vector<std::uint64_t>* out);
  Result<std::string> export_serve(std::uint32_t shard);
  // The shard's device serve tables (rs_serve_state).
  Status serve_tables(std::uint32_t shard, std::uint64_t* digests, std::uint64_t* flags,
                      std::uint32_t* epoch, std::uint32_t* n_batches) const;

  // --- retention offload lanes (client_core.cpp:1675-1717) ------------------
  // Park version v of every local shard in pinned host memory and serve it as
  // replica "<replica>+offload@<v>"; the endpoints go to offload_confirm.
  Status make_retention_lanes(VersionId v, std::vector<std::string>* endpoints);
  Result<std::string> export_lane(std::uint32_t shard, VersionId v);
  void release_lane(VersionId v);
  // Free the lanes the registry released (DirectiveKind::offload_release).
  void apply_releases();
  std::vector<VersionId> lanes() const;
  // --- cross-link seed buffers (client_core.cpp:1720-1812) ---------------
  // Starts the background fill of every local shard's seed lane (an update's
  // SeedStart); its completion is reported to the registry by a waiter
  // thread (role seed).  The split phase calls it with the outcome of
  // Registry::update.
  Status start_seed(const SeedStart& ss);
  // Waits for a running seed fill (its registry report included).
  void join_seed();
  std::vector<VersionId> seed_lanes() const;
  // Split phase (a registry replicated through an operation log): the
  // waiter records each shard's outcome instead of reporting it, and the
  // caller appends the role-seed completions to the log.
  void set_seed_report(bool on) { seed_report_ = on; }
  Status seed_status(std::uint32_t shard);  // after join_seed
  Result<std::string> export_seed(std::uint32_t shard, VersionId v);
  std::string endpoint(std::uint32_t shard) const { return shards_[shard].endpoint; }

 private:
  struct Reg {
    std::string name;
    std::uint8_t* ptr = nullptr;
    std::uint64_t len = 0;  // bytes of the version's entry (bf16 bytes for a cast region)
    Geometry geo;
    bool cast = false;      // lands as e4m3: len/2 bytes at ptr
  };
  // Reshard state of a bound payload (Assignment.reshard).
  struct Reshard {
    std::vector<SourceShard> srcs;           // manifests/layouts/chunk0 of the source shards
    std::vector<std::string> endpoints;      // per source shard
    Assignment::Blobs src_manifests, src_layouts;  // what the plan was built from
    ReshardPlan plan;                        // segments (source offsets) / gathers / copies
    std::vector<std::unique_ptr<DevBuf>> gather_bufs;  // per plan.gathers entry
    std::uint32_t own_chunks = 0;            // landing chunks of the reader's own items
    // The gathers' landing segments (the batches slice copies read), built
    // on the first launch: src = offset in the source item, src_id = source
    // shard; gather_items[k] = the source item of segment k.
    std::vector<dev::ItemDesc> gather_segs;
    std::vector<std::uint32_t> gather_items;
    std::uint32_t gather_chunks_end = 0;
    // per gather: the staging windows (item offset lo, hi, staging offset)
    std::vector<std::vector<std::array<std::uint64_t, 3>>> gather_windows;
    std::uint64_t staged(std::size_t gi, std::uint64_t item_off) const;
  };
  struct Payload {
    Manifest manifest;
    std::string encoded;
    std::string layout;  // encoded ShardLayout of this payload
    std::vector<std::unique_ptr<DevBuf>> group_bufs;
    ChunkMap cmap;
    DevBuf digests;
    DevBuf flags;
    std::uint32_t epoch = 0;
    bool landed_some = false;  // a fill ran in this epoch: flags may be set
    std::vector<std::uint64_t> item_ptrs;  // own landing/serving address per item
    std::unique_ptr<Reshard> reshard;      // set when pulling from another slicing
    // early publish: the manifest's big-entry digests are not in yet
    bool provisional = false;
    std::vector<std::uint32_t> deferred;   // publisher: entries K6 digests in the background
  };
  struct Shard {
    std::uint32_t idx = 0;
    int device = -1;
    std::string endpoint;
    std::vector<Reg> regs;
    std::map<std::string, std::uint32_t> by_name;
    std::shared_ptr<Payload> holding;
    std::optional<VersionId> partial_version;
    std::shared_ptr<ServeState> serve;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    dev::PlanUpload plan;       // fill: item table + tensor maps + work/status words
    dev::PlanUpload hash_plan;  // hash-only passes (publish, reshard groups): kept apart so
                                // the fill plan stays resident between fills
    dev::PlanUpload fuse_plan;  // reshard: staging -> region copy-hash pass
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::chrono::steady_clock::time_point t_launch;  // host clock of the fill's launch
    cudaStream_t poll = nullptr;  // progress reads while a fill runs
    std::vector<std::uint32_t> flag_host;  // report_progress: the fill's watermarks
    std::uint64_t reported = 0;            // items last reported to the registry
    DevBuf span_tables;           // copy_spans' span tables (grow-only: no per-call malloc/free)
    DevBuf unpack_tables;         // the group unpack's span table (re-uploaded only on change)
    std::vector<std::uint64_t> unpack_last;
    bool unpack_queued = false;   // the launched fill's group unpack is queued behind it
    DevBuf dig_tables, group_tables;  // publish: K6 span tables (grow-only)
    // Copy-engine landing from host memory (launch_fill): frames copied on
    // `dma`, each raising dma_flags[frame] = dma_epoch for the hash pass
    cudaStream_t dma = nullptr;
    DevBuf dma_flags;
    std::uint32_t dma_epoch = 0;
    bool dma_fill = false;  // the launched fill is fed by frames on `dma`
    std::uint32_t epoch_ctr = 0;
    struct Lane {
      std::string key;
      std::shared_ptr<ServeState> serve;
      std::unique_ptr<HostBuf> buf;
      std::string endpoint;
    };
    std::map<VersionId, Lane> lanes;  // retention offloads held for the registry
    struct SeedLane {
      std::string key;
      std::shared_ptr<ServeState> serve;
      std::unique_ptr<HostBuf> buf;
      std::shared_ptr<StreamSource> tcp;  // the fill's off-box source
    };
    std::map<VersionId, SeedLane> seed_lanes;  // seed buffers (filling or complete)
    cudaStream_t seed_stream = nullptr;
    cudaEvent_t seed_ev = nullptr;
    dev::PlanUpload seed_plan;
    std::shared_ptr<StreamSource> tcp;  // the fill's source when it is off-box (tcp:)
    // early publish: K6 over the big entries on its own stream
    cudaStream_t k6 = nullptr;
    DevBuf k6_tables;
  };
  Status make_retention_lane(Shard& sh, VersionId v, std::string* endpoint);
  Status launch_seed(Shard& sh, const Assignment& a);
  void release_seed_lane(VersionId v);
  Status settle_offload(OpOutcome* o, double wait_s);

  Status ensure_stream(Shard& sh);
  // Early publish: the background digests of the last publish are committed
  // (registry + own manifests) once done; join_finalize waits for them.
  void start_finalize(VersionId v);
  Status join_finalize();
  // A payload holding provisional manifest bytes adopts the final ones from
  // the registry (waiting up to wait_s for them).
  Status adopt_final(Shard& sh, double wait_s);
  int grid(const Shard& sh) const;  // SMs this handle's persistent kernels occupy
  Status build_payload(Shard& sh, VersionId v, std::shared_ptr<Payload>* out);
  Status bind(Shard& sh, const Assignment& a, VersionId v);
  Status bind_reshard(Shard& sh, const Assignment& a, VersionId v);
  Status derive(const Shard& sh, Manifest* m, std::string* encoded, std::string* layout,
                std::vector<std::uint32_t>* lens) const;
  Status alloc_tables(Shard& sh, Payload& p, std::uint32_t extra_chunks);
  Status launch_reshard_fill(Shard& sh, const Assignment& a, bool src_complete);
  Status build_gathers(Shard& sh, Reshard& rs);
  // Queues the reshard's follow-up work behind its pull kernel on sh.stream
  // (slice copies, group packing, re-digests), skipped on the device when the
  // fill failed (guard = the fill's status code word).
  Status finish_reshard(Shard& sh, const std::uint32_t* guard);
  Status hash_items(Shard& sh, Payload& p, const std::vector<std::uint32_t>& items,
                    const std::uint32_t* guard = nullptr);
  // table/last (optional): a dedicated span table whose upload is skipped
  // when the spans equal the previous call's (the steady-state group unpack).
  Status copy_spans(Shard& sh, const std::vector<std::uint64_t>& srcs,
                    const std::vector<std::uint64_t>& dsts, const std::vector<std::uint64_t>& lens,
                    const std::uint32_t* guard = nullptr, DevBuf* table = nullptr,
                    std::vector<std::uint64_t>* last = nullptr);
  // unpack_group (manifest.cpp:217-225) of every packed group, queued on
  // sh.stream (behind the fill, skipped on the device if it failed).
  Status queue_unpack(Shard& sh, const std::uint32_t* guard);
  Status resolve_shard(Shard& sh, const std::string& replica, std::uint32_t shard, VersionId v,
                       SourceView* out);
  void serve(Shard& sh, VersionId v, bool complete);
  Status resolve_source(Shard& sh, const Assignment& a, VersionId v, SourceView* out,
                        double wait_s);
  Status launch_fill(Shard& sh, const SourceView& src, bool src_complete);
  // task_progress (client_core.cpp:1414-1439): the verified item prefix of a
  // running plain fill, read from its watermarks, to the registry.
  void report_progress(Shard& sh);
  Status launch_host_dma(Shard& sh, const SourceView& src, std::uint32_t* epoch);
  Status run_replicate_loop(const OpOutcome& o, VersionId v);

  Registry* reg_;
  ServeRegistry* serves_;
  std::string model_, replica_;
  std::uint32_t num_shards_;
  ClientConfig cfg_;
  std::vector<Shard> shards_;
  std::optional<VersionId> current_;
  std::set<std::uint64_t> retain_;
  // Released lanes' pinned host buffers, reused by the next offload: pinning
  // fresh host memory runs at ~2 GB/s, a D2H copy into pinned memory at ~50.
  std::vector<std::unique_ptr<HostBuf>> host_pool_;
  std::vector<FillOutcome> launch_out_;  // launch_shards -> wait_shards
  // early publish finalizer (background thread; results adopted on the
  // caller's thread)
  std::thread fin_thread_;
  std::mutex fin_m_;
  bool fin_running_ = false;
  Status fin_status_ = Status::ok;
  VersionId fin_v_ = 0;
  std::vector<std::string> fin_manifests_;  // per shard ("" for a non-local shard)
  std::vector<bool> launched_;
  // seed fill waiter (reports role-seed completion to the registry)
  std::thread seed_thread_;
  std::atomic<std::uint64_t> seed_cross_dc_{0};
  bool seed_report_ = true;
  std::vector<Status> seed_status_;  // per shard, the last seed fill's outcome
  std::vector<std::optional<Assignment>> launch_as_;  // per shard: the latest launch's assignment
  bool published_ = false;
  bool opened_ = false;
  bool closed_ = false;
  ClientStats stats_;
};

// A whole item copied as-is (q == m == 1), source and landing chunk indices
// equal.
dev::ItemDesc identity_segment(std::uint64_t src, std::uint64_t dst, std::uint64_t len,
                               const ChunkMap& cm, std::size_t item);

// Peer / IPC address translation for the reader's device.
Status map_source(const std::shared_ptr<ServeState>& st, int reader_device, SourceView* out);
Status enable_peer(int reader_device, int owner_device);
int ptr_device(std::uint64_t p);  // device holding a (possibly IPC-mapped) address, -1: none

}  // namespace rsb
