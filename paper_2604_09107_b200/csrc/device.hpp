// Host-visible descriptors and launchers of the sm_100a kernels
// (kernels.cu).  No torch types; plain device pointers.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace rsb::dev {

// Flag word values (per watermark batch, device memory of the serving GPU):
//   flag == epoch              -> batch landed AND verified in fill `epoch`
//   flag <  epoch              -> not yet
//   flag == (epoch | kAbort)   -> the serving fill gave up on this batch
//   anything else (> epoch)    -> the server moved on to a newer fill
constexpr std::uint32_t kAbort = 0x80000000u;
constexpr int kBatchChunks = 32;  // chunks per warp batch = per watermark flag
constexpr int kPiece = 256;       // bytes of each chunk staged per step

// One transfer item as the reader sees it: where its bytes come from (any
// address the reader's device can load: local HBM, a peer GPU through
// NVLink/UVA, or an IPC-mapped peer allocation), where they land, and how
// the item is cut into digest chunks.
struct ItemDesc {
  std::uint64_t src;        // source address (0: hash-only / dst is source)
  std::uint64_t dst;        // landing address (0: hash-only)
  std::uint64_t len;        // bytes
  std::uint32_t chunk0;     // global index of the item's first chunk
  std::uint32_t chunk_len;  // uniform chunk length inside the item | kHasMap
};
// ItemDesc.chunk_len flag: the item has TMA tensor maps (2-D view
// [len / chunk_len rows][chunk_len bytes]) at PullParams.maps + 256*i
// (source) and + 256*i + 128 (destination).
constexpr std::uint32_t kHasMap = 0x80000000u;
constexpr std::uint32_t kChunkLenMask = 0x7fffffffu;
constexpr int kMapBoxCols = 128;  // TMA box: 128 bytes x 32 rows, 128B swizzle

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
  const ItemDesc* items;
  std::uint32_t n_items;
  std::uint32_t n_chunks;
  std::uint32_t n_batches;
  std::uint32_t first_batch;   // batches below this are skipped (resume)
  const std::uint64_t* src_digests;  // expected per chunk (null: compute only)
  std::uint64_t* dst_digests;        // own table to fill (null: don't)
  const std::uint32_t* src_flags;    // upstream watermarks (null: complete)
  std::uint32_t src_epoch;
  std::uint32_t dst_epoch;
  std::uint32_t* dst_flags;          // own watermarks (null: not serving)
  std::uint32_t* work;               // [0] batch ticket, [1] abort
  PullStatus* status;
  std::uint64_t timeout_ns;
  std::uint32_t resume;              // dst_flags may already hold dst_epoch
  std::uint32_t pad;
  const void* maps;                  // CUtensorMap pairs per item (or null)
};

// Uploads a pull plan (item table + TMA tensor maps + work/status words)
// into `scratch` on `device` and points `p` at it.  Items whose source (and
// destination) are 16-byte aligned get tensor maps (kHasMap).  Declared
// here, implemented in pullplan.cpp.
struct PlanUpload {
  void* scratch = nullptr;       // device buffer (grown by the callee)
  std::size_t scratch_bytes = 0;
  std::size_t h2d_bytes = 0;     // bytes uploaded by the last call
};
cudaError_t upload_pull_plan(int device, cudaStream_t s, ItemDesc* items, std::uint32_t n_items,
                             PlanUpload* up, PullParams* p);
void free_pull_plan(int device, PlanUpload* up);

// Fused mover: copy + per-chunk XXH64 verify + watermark publish.  `sms` is
// the device's SM count (pull_grid); the persistent grid is sized from it.
cudaError_t launch_pull(const PullParams& p, int sms, cudaStream_t s);
int pull_grid(int device);  // SM count of the device
const char* pull_kernel_name();

// XXH64 (reference digest64) of n spans, one warp per span.
cudaError_t launch_span_digests(const std::uint64_t* ptrs, const std::uint64_t* lens,
                                std::uint64_t* out, int n, cudaStream_t s);

// Gather/scatter copies: span i copies lens[i] bytes srcs[i] -> dsts[i].
cudaError_t launch_copy_spans(const std::uint64_t* srcs, const std::uint64_t* dsts,
                              const std::uint64_t* lens, int n, cudaStream_t s);

// Synthetic bf16 weights (SURVEY.md §8d generator; oracle ro_synth_bf16).
cudaError_t launch_synth_bf16(std::uint16_t* dst, std::uint64_t n, std::uint64_t seed,
                              std::uint64_t first, cudaStream_t s);

// Saturating RNE bf16 -> fp8 e4m3 (oracle ro_bf16_to_e4m3).
cudaError_t launch_bf16_to_e4m3(const std::uint16_t* src, std::uint8_t* dst,
                                std::uint64_t n, cudaStream_t s);

}  // namespace rsb::dev
