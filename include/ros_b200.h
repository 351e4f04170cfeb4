/* ros_b200.h -- C ABI of the B200-native ROS (Reference-Oriented Storage)
 * read path.  Plain pointers and sizes; no torch or C++ types.
 *
 * Every entry point returns an int status whose values are exactly the
 * reference's refstore::Status codes
 * (/root/reference/proj/include/refstore/types.hpp:22-41): 0 = ok,
 * 1 invalid_argument, 2 invalid_state, 3 already_exists, 4 not_found,
 * 5 version_regression, 6 manifest_conflict, 7 mutability_violation,
 * 8 version_unavailable, 9 group_aborted, 10 server_unavailable,
 * 11 transfer_failed, 12 checksum_mismatch, 13 not_serving, 14 timeout,
 * 15 offload_failed, 16 protocol_error, 17 closed.
 *
 * Which reference interface each group replaces is cited per function; the
 * bindings a maintainer would add on the reference side are in
 * INTEGRATION.md.  Threading: one caller per rs_handle; a
 * rs_cluster may be shared by handles on different threads.
 */
#ifndef ROS_B200_H
#define ROS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 3

typedef struct rs_cluster rs_cluster; /* ServerCore + ServeRegistry of this process */
typedef struct rs_handle rs_handle;   /* ClientCore: one replica's shard handles   */

/* ClientConfig (reference config.hpp:23-47) restricted to the knobs that shape
 * the read path, plus the digest chunk size of the device path. */
typedef struct {
  uint64_t chunk_bytes;    /* digest/watermark unit, multiple of 16 (default 4096)   */
  uint64_t tiny_threshold; /* ManifestLimits.tiny_threshold (default 2 MiB)          */
  uint64_t group_target;   /* ManifestLimits.group_target (default 64 MiB)           */
  int pipeline;            /* serve partially landed fills (default 1)               */
  int checksum_retries;    /* failure reports per fill before giving up (default 3) */
  double pull_timeout_s;   /* upstream silence before a failure report (default 4)  */
  char datacenter[32];     /* ClientConfig.datacenter (default "dc0")                */
  uint32_t reshard_align;  /* chunk rule: TP splits up to this stay chunk aligned (2) */
  uint32_t grid_sms;       /* SMs a fill's persistent pull kernel may occupy (0: all).
                            * Fills whose caps sum to <= the SM count co-reside on one
                            * GPU, so a reader may chase an upstream filling on its own
                            * GPU instead of waiting for it to complete.              */
  int early_publish;       /* 1: rs_publish commits the chunk-digest table and the
                            * manifest structure at once and the big-entry XXH64
                            * digests when their serial chains finish (background);
                            * readers pull meanwhile.  The committed manifest is the
                            * reference's, byte for byte (rs_publish_finalize waits
                            * for it).  Default 0: the reference order.            */
  int offload_seed;        /* ClientConfig.offload_seed (config.hpp): an update whose
                            * source is in another datacenter fills the version into
                            * pinned host memory in the background (replica
                            * "<replica>+seed@<v>") and reports no change; a later
                            * update consumes that seed locally.  Default 0.       */
} rs_config;

/* Assignment (reference messages.hpp:40-52) minus the manifest bytes, which
 * are read with rs_assignment_manifest / rs_manifest. */
typedef struct {
  uint64_t version;
  char source_replica[128];
  char source_endpoint[128];
  int source_complete;
  int cross_dc;
  int seeding;
  int local_seed_consume;
} rs_assignment;

/* ClientCore::Stats (client_core.hpp:44-52) + device-path timing. */
typedef struct {
  uint64_t bytes_pulled;
  uint64_t bytes_pulled_cross_dc;
  uint64_t bytes_copied_local;
  uint64_t items_verified;
  uint64_t checksum_failures;
  uint64_t failure_reports;
  uint64_t failovers;
  float last_pull_ms;       /* CUDA-event time of the last fill's pull kernel     */
  float last_publish_ms;    /* CUDA-event time of the last publish (digests+pack) */
  uint64_t last_pull_bytes; /* bytes landed+verified by that kernel               */
  uint32_t last_pull_launches;
  uint64_t h2d_bytes;       /* descriptor uploads, cumulative                     */
  uint64_t d2h_bytes;       /* status / digest read-backs, cumulative             */
  float fill_max_ms;        /* last fill round: the slowest local shard's kernel   */
  float fill_sum_ms;        /* last fill round: all local shards' kernels, summed  */
  uint64_t fill_bytes;      /* last fill round: bytes landed by all local shards   */
  uint64_t kernel_launches; /* this handle's kernels launched, cumulative          */
} rs_stats;

/* ---- process-level objects ------------------------------------------------ */
int rs_abi_version(void);
const char* rs_status_name(int status);                     /* types.cpp:7-29  */
void rs_config_default(rs_config* cfg);

/* ServerCore (server_core.hpp:30-52) + ServeRegistry (transport.hpp:72-85).
 * ServerConfig.pipeline / smart_skipping (config.hpp:15-21). */
int rs_cluster_create(int pipeline, int smart_skipping, rs_cluster** out);
void rs_cluster_destroy(rs_cluster* c);
/* Planner trace: one event per line "<seq> <kind> k=v ..." (kinds as the
 * reference's trace: assign, replicate_resolved, reassign, ...). */
int rs_cluster_trace(rs_cluster* c, char* buf, size_t cap, size_t* len);
/* ServerCore::listing (server_core.cpp:1276-1286) as "v:rep,rep;v:rep". */
int rs_cluster_listing(rs_cluster* c, const char* model, char* buf, size_t cap, size_t* len);
/* ServerCore::replica_view (server_core.hpp:42-50). lifecycle buffer >= 16. */
int rs_cluster_view(rs_cluster* c, const char* model, const char* replica, char* lifecycle,
                    uint64_t* version, uint32_t* serving, int* visible);
/* ReplicaView.min_progress (server_core.hpp:48): the fewest verified items
 * over the replica's shards, as its fills report them (ProgressMsg,
 * client_core.cpp:1414-1439) -- it advances while a fill runs. */
/* ReplicaView.seeding: the replica fills from another datacenter */
int rs_cluster_seeding(rs_cluster* c, const char* model, const char* replica, int* seeding);
int rs_cluster_progress(rs_cluster* c, const char* model, const char* replica,
                        uint64_t* min_progress);
/* The source replica a replicating replica currently pulls from ("" if none). */
int rs_cluster_source(rs_cluster* c, const char* model, const char* replica, char* buf,
                      size_t cap, size_t* len);
/* The box's measured topology, as the planner's source cost (pick_source,
 * server_core.cpp:1517-1543, gains the term between same_dc and serving):
 * cost[i * n + j] is the cost for a reader whose first data endpoint is
 * endpoints[i] to pull from a source whose first endpoint is endpoints[j]
 * (lower is nearer; pairs not listed cost 0).  A uniform matrix (every GPU
 * pair one NVSwitch hop) leaves every plan exactly the reference's. */
int rs_cluster_set_topology(rs_cluster* c, uint32_t n, const char* const* endpoints,
                            const int32_t* cost);
/* Fault hook (MemNetwork::set_data_silent, transport_mem.hpp:33-46): a
 * silent replica's data plane never answers, so its readers time out. */
int rs_cluster_set_silent(rs_cluster* c, const char* model, const char* replica, int silent);

/* ---- ClientCore API (paper Table 2; client_core.hpp:63-93) -------------- */
int rs_open(rs_cluster* c, const char* model, const char* replica, uint32_t num_shards,
            const rs_config* cfg, rs_handle** out);
/* register_tensor (client_core.hpp:72-73): dev_ptr is caller-owned device
 * memory that must outlive the handle (weights live in place). */
int rs_register(rs_handle* h, uint32_t shard, const char* name, void* dev_ptr, uint64_t bytes);
/* NEW (no reference counterpart): register a region that holds the slice
 * [r0, r0+nr) x [c0, c0+nc) (byte columns) of the logical tensor `name` of
 * shape [rows x row_bytes], densely (bytes == nr * nc).  Replicas whose
 * slicing differs reshard on pull (TP/FSDP gather and split). */
int rs_register_slice(rs_handle* h, uint32_t shard, const char* name, void* dev_ptr,
                      uint64_t bytes, uint64_t rows, uint64_t row_bytes, uint64_t r0, uint64_t nr,
                      uint64_t c0, uint64_t nc);
/* NEW (K5, no reference counterpart): register a region that receives the
 * version's bf16 entry `name` (`bytes` bf16 bytes; the slice geometry as in
 * rs_register_slice, rows == 0 for none) as fp8 e4m3: dev_ptr holds bytes/2
 * bytes, each element the saturating round-to-nearest-even cast of its bf16
 * source (NaN -> 0x7F).  Checksums are verified on the bf16 bytes before the
 * cast.  A replica with any cast region is terminal: it pulls, never serves
 * or publishes (rs_publish returns the invalid_state status). */
int rs_register_cast(rs_handle* h, uint32_t shard, const char* name, void* dev_ptr,
                     uint64_t bytes, uint64_t rows, uint64_t row_bytes, uint64_t r0, uint64_t nr,
                     uint64_t c0, uint64_t nc);
/* Replicas whose shards live in several processes (one process per GPU).
 * A shard is local to a handle once a region of it is registered there; the
 * split-phase calls (rs_prepare_publish, rs_transfer_*) act on local shards
 * only.  The replica's slicing key (rs_layout_key) is rs_combine_layout_key
 * of every shard's rs_shard_hash, gathered from the processes holding them. */
int rs_shard_local(rs_handle* h, uint32_t shard);
int rs_shard_hash(rs_handle* h, uint32_t shard, uint64_t* hash, int* geometry, int* cast);
int rs_combine_layout_key(uint32_t n, const uint64_t* hashes, const int* geometry, const int* cast,
                          char* buf, size_t cap, size_t* len);
/* The chunk length a region of geometry (row_bytes, slice width nc) is cut
 * into: the largest multiple of 128 <= chunk_bytes dividing
 * gcd(nc, row_bytes / align) (chunk_bytes when none). */
uint32_t rs_chunk_len_for(uint64_t row_bytes, uint64_t nc, uint64_t chunk_bytes, uint32_t align);
/* Slicing key of the replica ("" when no region has a geometry). */
int rs_layout_key(rs_handle* h, char* buf, size_t cap, size_t* len);
int rs_set_endpoint(rs_handle* h, uint32_t shard, const char* endpoint);
/* Launch the shard's device work on this cudaStream_t (default: a private
 * non-blocking stream). */
int rs_set_stream(rs_handle* h, uint32_t shard, void* cuda_stream);
int rs_publish(rs_handle* h, uint64_t version);              /* publish()   */
int rs_unpublish(rs_handle* h);                              /* unpublish() */
/* replicate(spec) / update(spec) -- spec "17" | "latest" | "latest-k".
 * Blocking; a parked replicate waits up to wait_s for a version to appear. */
int rs_replicate(rs_handle* h, const char* spec, double wait_s, uint64_t* out_version);
int rs_update(rs_handle* h, const char* spec, double wait_s, int* changed, uint64_t* out_version);
/* The names SURVEY.md §8b recommends for this boundary: rs_pull = replicate;
 * rs_release = drop a retention offload this handle holds for `version`;
 * rs_serve_state exposes a shard's device serve tables (chunk digests,
 * per-batch watermarks, current fill epoch: a batch is landed and verified
 * when its watermark == epoch) so a caller can chain on them. */
int rs_pull(rs_handle* h, const char* spec, double wait_s, uint64_t* out_version);
int rs_release(rs_handle* h, uint64_t version);
int rs_serve_state(rs_handle* h, uint32_t shard, uint64_t** digests, uint32_t** watermarks,
                   uint32_t* epoch, uint32_t* n_batches);
int rs_close(rs_handle* h);                                  /* close(); frees h */
/* Early publish (rs_config.early_publish): 1 while the handle's last publish
 * still digests its big entries; rs_publish_finalize waits for them and
 * commits the final manifests (to the in-process registry when this handle
 * holds every shard; rs_manifest then returns the final bytes). */
int rs_publish_pending(rs_handle* h);
/* Switch rs_config.early_publish for the handle's next publish. */
int rs_set_early_publish(rs_handle* h, int on);
int rs_publish_finalize(rs_handle* h, double wait_s);
/* Plan view without side effects: the source `replica` would pull `shard`
 * of `spec` from right now. */
int rs_locate(rs_cluster* c, const char* model, const char* replica, const char* spec,
              uint32_t shard, rs_assignment* out);
int rs_current_version(rs_handle* h, uint64_t* out); /* not_found if none held */
int rs_is_published(rs_handle* h);
int rs_stats_get(rs_handle* h, rs_stats* out);
/* Canonical manifest bytes of the shard's held version
 * (TensorManifest::encode, manifest.cpp:103-139). */
int rs_manifest(rs_handle* h, uint32_t shard, char* buf, size_t cap, size_t* len);
/* The manifest bytes the shard holds right now, without waiting: during an
 * early publish (rs_publish_pending) its provisional bytes, big-entry digests
 * 0 -- what a split-phase caller registers with rs_server_publish_provisional.
 * rs_manifest returns the final bytes, waiting for them if needed. */
int rs_manifest_now(rs_handle* h, uint32_t shard, char* buf, size_t cap, size_t* len);
/* The shard's per-chunk XXH64 table (device path integrity metadata). */
int rs_chunk_digests(rs_handle* h, uint32_t shard, uint64_t* out, size_t cap, size_t* n);
/* The shard's layout blob (entry geometries + per-item chunk lengths). */
int rs_layout(rs_handle* h, uint32_t shard, char* buf, size_t cap, size_t* len);
/* 1 if the bound fill reshards (its manifest/layout are derived), else 0. */
int rs_transfer_derived(rs_handle* h);
/* The replica's own-slicing derived manifest (what=0) or layout (what=1) of
 * `shard`, computed from its registrations; len 0 for a plain replica. */
int rs_derived(rs_handle* h, uint32_t shard, int what, char* buf, size_t cap, size_t* len);
/* Drop the landed watermark so the next fill re-pulls every byte. */
int rs_invalidate(rs_handle* h);

/* ---- split phase: the caller drives the registry (replicated across
 *      processes: every rank applies the same rs_server_* sequence) ------- */
/* derived_*: the replica's own-slicing manifests/layouts (rs_derived; NULL
 * for a plain replica). */
int rs_server_open(rs_cluster* c, const char* model, const char* replica, uint32_t num_shards,
                   const char* datacenter, const char* const* endpoints, const char* layout_key,
                   const char* const* derived_manifests, const size_t* dm_lens,
                   const char* const* derived_layouts, const size_t* dl_lens);
int rs_server_publish(rs_cluster* c, const char* model, const char* replica, uint64_t version,
                      uint32_t num_shards, const char* const* manifests, const size_t* lens,
                      const char* const* layouts, const size_t* layout_lens);
int rs_server_add_layout(rs_cluster* c, const char* model, uint64_t version, const char* layout_key,
                         uint32_t num_shards, const char* const* manifests, const size_t* lens,
                         const char* const* layouts, const size_t* layout_lens);
/* rs_server_publish of an early publish's provisional manifests, and the
 * later commit of their final bytes (same structure, digests filled). */
int rs_server_publish_provisional(rs_cluster* c, const char* model, const char* replica,
                                  uint64_t version, uint32_t num_shards,
                                  const char* const* manifests, const size_t* lens,
                                  const char* const* layouts, const size_t* layout_lens);
int rs_server_finalize(rs_cluster* c, const char* model, const char* replica, uint64_t version,
                       uint32_t num_shards, const char* const* manifests, const size_t* lens);
int rs_server_unpublish(rs_cluster* c, const char* model, const char* replica);
int rs_server_replicate(rs_cluster* c, const char* model, const char* replica, const char* spec);
int rs_server_update(rs_cluster* c, const char* model, const char* replica, const char* spec,
                     int has_current, uint64_t current);
/* Outcome of the replica's latest op: done=0 while parked. */
int rs_server_result(rs_cluster* c, const char* model, const char* replica, int* done,
                     int* status, uint64_t* version, int* changed);
int rs_server_complete(rs_cluster* c, const char* model, const char* replica, uint32_t shard,
                       int outcome);
int rs_server_failure_report(rs_cluster* c, const char* model, const char* replica,
                             uint32_t shard, const char* failed_replica, int reason);
int rs_server_close(rs_cluster* c, const char* model, const char* replica);
/* Client half. */
int rs_prepare_publish(rs_handle* h, uint64_t version);  /* digests+pack+manifest */
int rs_commit_publish(rs_handle* h, uint64_t version, int status);
/* Bind every shard to the registry's current assignment and start serving
 * the empty fill (so downstream readers can chase it). */
int rs_transfer_bind(rs_handle* h, uint64_t version);
/* One fill attempt of every shard still pending; statuses/reasons per shard
 * (reason 0 timeout/not serving, 1 checksum). */
int rs_transfer_fill(rs_handle* h, int* statuses, int* reasons);
/* rs_transfer_fill in two halves: launch the pending shards' pull kernels
 * (returns at once), then wait for them.  In between, rs_transfer_progress
 * reads a running fill's verified-batch count (32-chunk batches) -- the
 * watermark a late joiner chases. */
int rs_transfer_launch(rs_handle* h);
int rs_transfer_progress(rs_handle* h, uint32_t shard, uint32_t* batches_done, uint32_t* n_batches);
int rs_transfer_wait(rs_handle* h, int* statuses, int* reasons);
/* The assignment the shard's latest fill was launched on (Assignment,
 * messages.hpp:40-52): its source, and whether that source was complete or
 * a pipeline copy still filling (source_complete == 0: the fill chased the
 * source's watermarks).  not_found before any launch. */
int rs_transfer_assignment(rs_handle* h, uint32_t shard, rs_assignment* out);
int rs_transfer_finish(rs_handle* h, uint64_t version, int ok);
/* Cross-process serve state (CUDA IPC handles + watermarks). */
int rs_serve_export(rs_handle* h, uint32_t shard, void* buf, size_t cap, size_t* len);
int rs_serve_import(rs_cluster* c, const void* blob, size_t len);

/* ---- retention offload (RetentionRule types.hpp:119-123; client_core.cpp
 * 1675-1717; server_core.cpp 1387-1485, 1592-1645) ---------------------------
 * A replica may ask the cluster to keep the versions at some lags behind the
 * newest published one reachable.  When the last durable copy of such a
 * version unpublishes (or updates away), its client first parks it in pinned
 * host memory (POSIX shared memory registered with CUDA) and the registry
 * adds replica "<owner>+offload@<v>", which serves readers like any copy
 * (the pull kernel reads host memory over PCIe) until a worker holds the
 * version again or it leaves the retained window.  rs_unpublish/rs_update do
 * all of this; the split-phase calls below let a multi-process caller do it. */
int rs_set_retention(rs_handle* h, const uint64_t* lags, size_t n);  /* before the first op */
/* ClientCore::open (client_core.hpp:83): join the cluster without an op (a
 * pure observer whose retention rule keeps versions reachable). */
int rs_connect(rs_handle* h);
int rs_offload_lanes(rs_handle* h, uint64_t version);                 /* park v (local shards) */
int rs_lane_export(rs_handle* h, uint32_t shard, uint64_t version, void* buf, size_t cap,
                   size_t* len);
int rs_offload_release(rs_handle* h, uint64_t version);
int rs_poll(rs_handle* h);  /* free the lanes the registry released */
int rs_lanes(rs_handle* h, uint64_t* versions, size_t cap, size_t* n);
int rs_server_set_retention(rs_cluster* c, const char* model, const char* replica,
                            const uint64_t* lags, size_t n);
/* 1 (and *version) while the replica's unpublish/update waits for an offload. */
int rs_server_offload_pending(rs_cluster* c, const char* model, const char* replica,
                              uint64_t* version);
int rs_server_offload_confirm(rs_cluster* c, const char* model, const char* replica,
                              uint32_t shard, uint64_t version, int ok, const char* endpoint);
int rs_server_take_releases(rs_cluster* c, const char* model, const char* owner,
                            uint64_t* versions, size_t cap, size_t* n);
int rs_cluster_kind(rs_cluster* c, const char* model, const char* replica, char* buf, size_t cap,
                    size_t* len);  /* "worker" | "offload" */

/* ---- cross-link seed buffers (client_core.cpp:1720-1812; server_core.cpp
 * 88-99, 915-970, 1124-1204) ------------------------------------------------
 * With rs_config.offload_seed, rs_update against a source in another
 * datacenter returns changed = 0 and starts a background fill of the version
 * into pinned host memory (the pull kernel lands it over PCIe, verifying
 * every chunk); the registry masks the version for this datacenter until the
 * seed completes, then plans same-datacenter readers onto it, and the
 * owner's next rs_update consumes it locally (local_seed_consume).  The seed
 * is released once consumed and drained (rs_poll frees it). */
int rs_seed_lanes(rs_handle* h, uint64_t* versions, size_t cap, size_t* n);  /* after the fill */
int rs_seed_wait(rs_handle* h);  /* wait for a running seed fill (and its report) */
/* Split phase (the registry replicated through an operation log): start the
 * seed fill the replica's last update outcome carries, without reporting it
 * to the local registry; after the fill, rs_seed_status gives each local
 * shard's outcome (to append as a role-seed completion) and rs_seed_export
 * the lane's serve state for other processes (rs_serve_import). */
int rs_seed_fill(rs_handle* h);
int rs_seed_status(rs_handle* h, uint32_t shard);
int rs_seed_export(rs_handle* h, uint32_t shard, uint64_t version, void* buf, size_t cap,
                   size_t* len);
int rs_server_set_offload_seed(rs_cluster* c, const char* model, const char* replica, int on);
/* the shard's assignment in the replica's last replicate/update outcome */
int rs_server_assignment(rs_cluster* c, const char* model, const char* replica, uint32_t shard,
                         rs_assignment* out);
/* 1 (and the shard's seed assignment) when the replica's last update started a seed */
int rs_server_seed_start(rs_cluster* c, const char* model, const char* replica, uint32_t shard,
                         rs_assignment* out);
/* ProgressMsg / CompleteMsg with TransferRole::seed for the seed of `version` */
int rs_server_seed_progress(rs_cluster* c, const char* model, const char* replica, uint32_t shard,
                            uint64_t items, uint64_t version);
int rs_server_seed_complete(rs_cluster* c, const char* model, const char* replica, uint32_t shard,
                            int outcome, uint64_t version);

/* ---- off-box data plane (transport_stream.hpp:36-76)
 * Serve this process's serve states over TCP (port 0: any free port).  A
 * reader whose assigned source endpoint is "tcp:<host>:<port>" (set with
 * rs_set_endpoint on the source) receives the source's chunk map, digest
 * table and payload batches into pinned, device-mapped host memory; its pull
 * kernel lands and verifies them, chasing per-batch host watermarks. */
int rs_cluster_listen(rs_cluster* c, const char* host, int port, int* bound_port);

/* ---- dynamic membership: the registry's sequenced operation log -----------
 * (the reference's one metadata server that clients dial at
 * any time, StreamServerHost / StreamControl, transport_stream.cpp:582-797.)
 * Every process keeps a registry replica (rs_cluster) and applies one totally
 * ordered log of registry operations; the log server orders them.  A process
 * that starts late replays the log from entry 0 and joins with the same
 * registry state as the others (paper_2604_09107_b200/shared.py drives it). */
typedef struct rs_oplog_server rs_oplog_server;
typedef struct rs_oplog rs_oplog;
int rs_oplog_serve(const char* host, int port, int* bound_port, rs_oplog_server** out);
void rs_oplog_server_stop(rs_oplog_server* s);
uint64_t rs_oplog_server_size(rs_oplog_server* s);
int rs_oplog_connect(const char* host, int port, double timeout_s, rs_oplog** out);
/* Appends one entry (opaque bytes); *seq is its position in the log. */
int rs_oplog_append(rs_oplog* l, const void* entry, size_t len, uint64_t* seq);
/* Fetches up to max_entries entries from position `from` (long-polls up to
 * wait_ms when none exist yet); read them with rs_oplog_entry, valid until the
 * next fetch on this connection. */
int rs_oplog_fetch(rs_oplog* l, uint64_t from, int wait_ms, uint32_t max_entries, uint64_t* count);
int rs_oplog_entry(rs_oplog* l, uint64_t i, const void** data, size_t* len);
void rs_oplog_close(rs_oplog* l);

/* ---- device primitives (kernel boundary) --------------------------------- */
/* digest64 (digest.cpp:79-106) of n device spans; out is host memory. */
int rs_digest_spans(const uint64_t* dev_ptrs, const uint64_t* lens, int n, uint64_t* out,
                    int device);
/* Synthetic bf16 weights into device memory. */
int rs_synth_bf16(void* dev_dst, uint64_t n_elems, uint64_t seed, uint64_t first_elem,
                  void* cuda_stream);
/* Saturating RNE bf16 -> fp8 e4m3 on device. */
int rs_bf16_to_e4m3(const void* dev_src, void* dev_dst, uint64_t n_elems, void* cuda_stream);
/* copy_slice_locked (transport.cpp:51-69) + chunk verification, standalone:
 * copy n_items (src -> dst, len) spans cut into chunk_bytes chunks, verify
 * against expect (device, may be NULL) and write the computed chunk digests
 * to out_digests (device, may be NULL).  Both tables are indexed batch
 * aligned: item i's chunks start at round_up(end of item i-1, 32); entries
 * in between are unused.  Reports the kernel status. */
int rs_pull_spans(const uint64_t* src_ptrs, const uint64_t* dst_ptrs, const uint64_t* lens,
                  int n_items, uint64_t chunk_bytes, const uint64_t* expect_dev,
                  uint64_t* out_digests_dev, int device, void* cuda_stream, int* kernel_code,
                  float* kernel_ms);

#ifdef __cplusplus
}
#endif
#endif /* ROS_B200_H */
