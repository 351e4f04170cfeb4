// Host-visible descriptors and launchers of the sm_100a kernels
// (kernels.cu).  No torch types; plain device pointers.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

namespace rsb::dev {

// Flag word values (per watermark batch, device memory of the serving GPU):
//   flag == epoch              -> batch landed AND verified in fill `epoch`
//   flag <  epoch              -> not yet
//   flag == (epoch | kAbort)   -> the serving fill gave up on this batch
//   anything else (> epoch)    -> the server moved on to a newer fill
constexpr std::uint32_t kAbort = 0x80000000u;
constexpr int kBatchChunks = 32;  // chunks per warp batch = per watermark flag
constexpr int kPiece = 256;       // bytes of each chunk staged per step

// One segment of the landing stream as the reader sees it: where its chunks
// come from (any address the reader's device can load: local HBM, a peer
// GPU through NVLink/UVA, or an IPC-mapped peer allocation), where they land
// and how they map.  Landing chunk k of the segment (k = 0..) is source
// chunk (row t = k / q, column j = k % q) of a source item whose rows are m
// chunks long: source offset (t*m + j) * chunk_len, source chunk index
// src_chunk0 + t*m + j.  It lands densely at dst + k * chunk_len.  q == m is
// a contiguous copy (an identity pull, or a dim-0 reshard); q < m takes a
// column band of every row (a dim-1 / row-parallel reshard).
struct ItemDesc {
  std::uint64_t src;         // source address of the segment's first chunk
  std::uint64_t dst;         // landing address of the first chunk (0: hash-only)
  std::uint64_t len;         // source bytes of the segment (landed as-is, or halved by kCastE4M3)
  std::uint32_t chunk0;      // landing chunk index of the first chunk (global)
  std::uint32_t chunk_len;   // chunk length | kHasMap | kMap3D
  std::uint32_t src_chunk0;  // source chunk index of the first chunk
  std::uint16_t q, m;        // chunks taken per source row / chunks per source row
  std::uint32_t src_id;      // index into PullParams.srcs
  std::uint32_t pad;         // link class of the source (0: local HBM, 1: host, 2 + d: peer d);
                             // only the schedule order reads it
};
static_assert(sizeof(ItemDesc) == 48, "ItemDesc layout");
// chunk_len flags: the segment has TMA tensor maps at PullParams.maps +
// 256*i (source) and + 256*i + 128 (destination).  Source map: 2-D
// [rows = chunks][chunk_len] when q == m, 3-D [rows][q][chunk_len] (row
// stride m*chunk_len, kMap3D) when q < m.  Destination map: 2-D.
constexpr std::uint32_t kHasMap = 0x80000000u;
constexpr std::uint32_t kMap3D = 0x40000000u;
// The segment lands as fp8 e4m3 (K5): source chunks are bf16; landing chunk
// k holds chunk_len/2 bytes at dst + k*chunk_len/2 (saturating RNE cast,
// oracle ro_bf16_to_e4m3).  Verification is on the bf16 bytes.
constexpr std::uint32_t kCastE4M3 = 0x20000000u;
// A cast segment whose e4m3 landing has a destination tensor map (2-D
// [chunks][chunk_len/2], 128B swizzle) at maps + 256*i + 128: the consumer
// converts into the stage and lands it with tensor stores.
constexpr std::uint32_t kCastMap = 0x10000000u;
constexpr std::uint32_t kChunkLenMask = 0x0fffffffu;
constexpr int kMapBoxCols = 128;  // TMA box: 128 bytes x 32 chunks, 128B swizzle

// A source serve state as the reader's device sees it.
struct SrcDesc {
  const std::uint64_t* digests;  // source chunk-digest table (null: compute only)
  const std::uint32_t* flags;    // source watermarks (null: source complete)
  std::uint32_t epoch;           // source fill epoch to wait for
  std::uint32_t flag_shift;      // source batch b is covered by flags[b >> flag_shift]
};

enum PullCode : std::uint32_t {
  kPullOk = 0,
  kPullChecksum = 1,     // a chunk failed verification twice
  kPullTimeout = 2,      // upstream watermark did not advance in time
  kPullNotServing = 3,   // upstream moved to another fill / aborted
  kPullAborted = 4,      // another warp failed; stopped early
};

struct PullStatus {
  std::uint32_t code;
  std::uint32_t bad_chunk;
  std::uint32_t batches_done;
  std::uint32_t retried_batches;
  std::uint64_t bytes;  // bytes landed+verified
  std::uint64_t pad;
};

struct PullParams {
  const ItemDesc* items;             // segments, sorted by chunk0
  std::uint32_t n_items;
  std::uint32_t n_chunks;
  std::uint32_t n_batches;
  std::uint32_t first_batch;         // batches below this are skipped
  const SrcDesc* srcs;               // source table (segments' src_id)
  std::uint32_t n_srcs;
  std::uint32_t dst_epoch;
  std::uint64_t* dst_digests;        // own table to fill (null: don't)
  std::uint32_t* dst_flags;          // own watermarks (null: not serving)
  std::uint32_t* work;               // [0] batch ticket, [1] abort
  PullStatus* status;
  std::uint64_t timeout_ns;
  std::uint32_t resume;              // dst_flags may already hold dst_epoch
  std::uint32_t has_cast;            // some segment lands as e4m3 (kernel shape choice)
  const void* maps;                  // CUtensorMap pairs per segment (or null)
  const std::uint32_t* batch_seg;    // per batch: last segment with chunk0 <= 32*batch
  std::uint32_t remote;              // 0 local / host, 1 some source is a peer GPU, 2 a plain
                                     // peer pull (identity, no cast): kernel shape choice
  // Schedule: positions 0..n_sched-1 map to batches order[pos] (first_batch
  // then unused); null order: batches first_batch..n_batches-1 in order.
  // The order lists only the batches some segment touches (a hash pass over
  // a few items of a large payload walks just those) and interleaves the
  // batches of sources behind different links (schedule_order).
  std::uint32_t n_sched;
  const std::uint32_t* order;
  // Stream-ordered follow-up work: when set and *guard != 0 (the failure
  // code of the fill this pass follows), the kernel does nothing.
  const std::uint32_t* guard;
};

// Uploads a pull plan (segment table + source table + TMA tensor maps +
// batch -> segment table + work/status words) into `up->scratch` on
// `device` and points `p` at it (n_chunks / n_batches included).  Segments
// whose addresses are 16-byte aligned and whose geometry fits a box get
// tensor maps (kHasMap).  A plan byte-identical to the previous upload into
// the same scratch only resets the work/status words.  pullplan.cpp.
struct PlanUpload {
  void* scratch = nullptr;       // device buffer (grown by the callee)
  std::size_t scratch_bytes = 0;
  std::size_t h2d_bytes = 0;     // bytes uploaded by the last call
  std::vector<std::uint8_t> last;  // host image of the resident plan
  // the inputs the resident plan was built from: an identical request skips
  // the host build (tensor-map encoding) and only resets work/status words
  std::vector<ItemDesc> key_items;
  std::vector<SrcDesc> key_srcs;
  std::uint32_t key_chunks = 0;
  PullParams built{};
};
cudaError_t upload_pull_plan(int device, cudaStream_t s, ItemDesc* items, std::uint32_t n_items,
                             const SrcDesc* srcs, std::uint32_t n_srcs, std::uint32_t n_chunks,
                             PlanUpload* up, PullParams* p);
void free_pull_plan(int device, PlanUpload* up);
// The schedule order of a plan (see PullParams.order; empty: every batch,
// in order).  `bseg`: per batch, the segment holding its first chunk.
std::vector<std::uint32_t> schedule_order(const ItemDesc* items, std::uint32_t n,
                                          const std::vector<std::uint32_t>& bseg);

// Fused mover: copy + per-chunk XXH64 verify + watermark publish.  `sms` is
// the device's SM count (pull_grid); the persistent grid is sized from it.
cudaError_t launch_pull(const PullParams& p, int sms, cudaStream_t s);
// launch_pull starts a kernel only when the plan has batches to do.
inline bool pull_has_work(const PullParams& p) { return p.order ? p.n_sched != 0 : p.n_batches > p.first_batch; }
int pull_grid(int device);  // SM count of the device
const char* pull_kernel_name();

// XXH64 (reference digest64) of n spans, one warp per span.
cudaError_t launch_span_digests(const std::uint64_t* ptrs, const std::uint64_t* lens,
                                std::uint64_t* out, int n, cudaStream_t s);

// Gather/scatter copies: span i copies lens[i] bytes srcs[i] -> dsts[i].
// lens[i] | kSpanCastE4M3: the span's bf16 bytes land as e4m3 (lens/2 bytes).
constexpr std::uint64_t kSpanCastE4M3 = 1ull << 63;
// tile0[i]: first tile (copy_span_tiles units) of span i; tiles: the total.
// guard (may be null): skip the copy when *guard != 0 (a failed fill's code).
cudaError_t launch_copy_spans(const std::uint64_t* srcs, const std::uint64_t* dsts,
                              const std::uint64_t* lens, const std::uint64_t* tile0, int n,
                              std::uint64_t tiles, cudaStream_t s,
                              const std::uint32_t* guard = nullptr);
std::uint64_t copy_span_tiles(std::uint64_t len);  // tiles of one span (len may carry the cast flag)

// Synthetic bf16 weights (SURVEY.md §8d generator; oracle ro_synth_bf16).
cudaError_t launch_synth_bf16(std::uint16_t* dst, std::uint64_t n, std::uint64_t seed,
                              std::uint64_t first, cudaStream_t s);

// Saturating RNE bf16 -> fp8 e4m3 (oracle ro_bf16_to_e4m3).
cudaError_t launch_bf16_to_e4m3(const std::uint16_t* src, std::uint8_t* dst,
                                std::uint64_t n, cudaStream_t s);

}  // namespace rsb::dev
