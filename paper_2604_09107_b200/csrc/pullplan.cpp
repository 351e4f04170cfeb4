// Host side of a pull launch: segment table + source table + TMA tensor maps
// + batch -> segment table + schedule order + work/status words, uploaded in
// one H2D copy.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <map>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "device.hpp"

namespace rsb::dev {

namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 2-D [rows][c] or 3-D [rows][q][c] (row stride m*c) byte tensor at `base`;
// box 128 B x 32 chunks, 128B swizzle.
bool encode(CUtensorMap* map, std::uint64_t base, std::uint64_t c, std::uint64_t q,
            std::uint64_t m, std::uint64_t rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint32_t estr[3] = {1, 1, 1};
  if (q == m) {
    cuuint64_t dims[2] = {c, rows};
    cuuint64_t strides[1] = {c};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kMapBoxCols), 32};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, reinterpret_cast<void*>(base), dims, strides,
              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  cuuint64_t dims[3] = {c, q, rows};
  cuuint64_t strides[2] = {c, m * c};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(kMapBoxCols), static_cast<cuuint32_t>(q),
                       static_cast<cuuint32_t>(32 / q)};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, reinterpret_cast<void*>(base), dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr std::size_t kHdr = 128;  // work words (64 B) + PullStatus (32 B), padded

bool peer_boxes() {  // A/B knob: tensor-map boxes for peer / host segments too
  static const bool v = std::getenv("RSB_PEER_BOXES") != nullptr;
  return v;
}

bool maps_disabled() {
  static const bool v = std::getenv("RSB_NO_MAPS") != nullptr;  // diagnostic knob
  return v;
}

bool plan_debug() {
  static const bool v = std::getenv("RSB_PLAN_STATS") != nullptr;  // diagnostic knob
  return v;
}

// How the kernel will take each batch (box: one tensor load per 128-byte
// column of a whole-chunk batch; slot: per-lane bulk copies), by bytes.
void print_plan_stats(const ItemDesc* items, std::uint32_t n, const std::vector<std::uint32_t>& bseg,
                      std::uint32_t n_chunks) {
  std::uint64_t box_b = 0, slot_b = 0, box_n = 0, slot_n = 0, band_b = 0;
  std::map<std::uint32_t, std::uint64_t> by_len, by_class;
  for (std::uint32_t b = 0; b < bseg.size(); ++b) {
    const std::uint32_t s0 = bseg[b];
    const ItemDesc& d = items[s0];
    const std::uint32_t c = d.chunk_len & kChunkLenMask;
    const std::uint32_t k0 = b * kBatchChunks - d.chunk0;
    const std::uint64_t full = c ? d.len / c : 0;
    const bool whole = k0 + kBatchChunks <= full && b * kBatchChunks + kBatchChunks <= n_chunks &&
                       (s0 + 1 >= n || items[s0 + 1].chunk0 >= (b + 1) * kBatchChunks);
    const bool box = (d.chunk_len & kHasMap) && whole && (k0 % (d.q ? d.q : 1)) == 0;
    std::uint64_t bytes = 0;
    for (std::uint32_t l = 0; l < kBatchChunks; ++l) {
      const std::uint32_t ch = b * kBatchChunks + l;
      if (ch >= n_chunks) break;
      std::uint32_t sg = s0;
      while (sg + 1 < n && items[sg + 1].chunk0 <= ch) ++sg;
      const ItemDesc& e = items[sg];
      const std::uint32_t cl = e.chunk_len & kChunkLenMask;
      const std::uint64_t k = ch - e.chunk0;
      if (cl == 0 || k * cl >= e.len) continue;
      bytes += std::min<std::uint64_t>(cl, e.len - k * cl);
    }
    (box ? box_b : slot_b) += bytes;
    (box ? box_n : slot_n) += 1;
    if (box && (d.chunk_len & kMap3D)) band_b += bytes;
    by_len[c] += bytes;
    by_class[d.pad] += bytes;
  }
  std::fprintf(stderr, "[rsb] plan: %u segments, %zu batches: box %llu (%.3f GB, %.3f GB column bands), "
               "slot %llu (%.3f GB)\n[rsb] plan: bytes by chunk length:",
               n, bseg.size(), (unsigned long long)box_n, box_b / 1e9, band_b / 1e9,
               (unsigned long long)slot_n, slot_b / 1e9);
  for (const auto& [len, bytes] : by_len) std::fprintf(stderr, " %u:%.3fGB", len, bytes / 1e9);
  std::fprintf(stderr, "\n[rsb] plan: bytes by link class:");
  for (const auto& [c, bytes] : by_class) std::fprintf(stderr, " %u:%.3fGB", c, bytes / 1e9);
  std::fprintf(stderr, "\n");
}

}  // namespace

std::vector<std::uint32_t> schedule_order(const ItemDesc* items, std::uint32_t n,
                                          const std::vector<std::uint32_t>& bseg) {
  // The batches some segment touches (empty result: all, in batch order).
  // When the segments' sources sit behind different links (ItemDesc.pad =
  // link class: 0 local HBM, 1 host memory, 2 + d peer d), the classes' batches
  // are interleaved in proportion to their counts: batch b, the r-th of its
  // class's n_c batches, goes at key (r + 1/2) / n_c, so every link stays
  // busy for the whole pull instead of one at a time, and each class keeps
  // its own front-to-back order (what a chaser downstream waits on).
  // Sources behind one link are not interleaved: that only scatters the
  // landing writes (measured +1.5% on config 3 at N=1).  Config 3 at N=2
  // (FSDP-2 -> TP-2, 16% of each shard over NVLink): 14.8 -> 13.1 ms; with
  // the peer only serving, 13.3 -> 9.7 ms (tools/mix_probe.py).  Finishing
  // the remote class earlier (keys scaled by 0.2-0.8) moved it by <= 2%.
  static const bool no_mix = std::getenv("RSB_BATCH_ORDER") &&
                             std::getenv("RSB_BATCH_ORDER")[0] == '0';  // A/B knob
  const std::uint32_t nb = static_cast<std::uint32_t>(bseg.size());
  std::vector<std::uint8_t> touched(nb, 0);
  for (std::uint32_t i = 0; i < n; ++i) {
    const std::uint64_t c = items[i].chunk_len & kChunkLenMask;
    if (c == 0 || items[i].len == 0) continue;
    const std::uint64_t last = items[i].chunk0 + (items[i].len + c - 1) / c - 1;
    for (std::uint64_t b = items[i].chunk0 / kBatchChunks; b <= last / kBatchChunks && b < nb; ++b)
      touched[b] = 1;
  }
  std::vector<std::uint32_t> cls(nb, 0), count;
  std::uint32_t n_touched = 0;
  for (std::uint32_t b = 0; b < nb; ++b) {
    if (!touched[b]) continue;
    ++n_touched;
    const std::uint32_t c = no_mix ? 0 : items[bseg[b]].pad;
    cls[b] = c;
    if (c >= count.size()) count.resize(c + 1, 0);
    ++count[c];
  }
  int classes = 0;
  for (std::uint32_t c : count) classes += c != 0;
  if (classes < 2 && n_touched == nb) return {};
  std::vector<std::uint32_t> rank(count.size(), 0);
  std::vector<std::pair<double, std::uint32_t>> key;
  key.reserve(n_touched);
  for (std::uint32_t b = 0; b < nb; ++b) {
    if (!touched[b]) continue;
    const std::uint32_t c = cls[b];
    key.push_back({(rank[c]++ + 0.5) / count[c], b});
  }
  if (classes > 1) std::sort(key.begin(), key.end());
  std::vector<std::uint32_t> order(key.size());
  for (std::size_t i = 0; i < key.size(); ++i) order[i] = key[i].second;
  return order;
}

cudaError_t upload_pull_plan(int device, cudaStream_t s, ItemDesc* items, std::uint32_t n,
                             const SrcDesc* srcs, std::uint32_t n_srcs, std::uint32_t n_chunks,
                             PlanUpload* up, PullParams* p) {
  const std::uint32_t n_batches = (n_chunks + kBatchChunks - 1) / kBatchChunks;
  if (up->scratch && up->key_chunks == n_chunks && up->key_items.size() == n &&
      up->key_srcs.size() == n_srcs &&
      (n == 0 || std::memcmp(up->key_items.data(), items, n * sizeof(ItemDesc)) == 0) &&
      (n_srcs == 0 || std::memcmp(up->key_srcs.data(), srcs, n_srcs * sizeof(SrcDesc)) == 0)) {
    cudaError_t e = cudaMemsetAsync(up->scratch, 0, kHdr, s);  // fresh work/status words
    if (e != cudaSuccess) return e;
    up->h2d_bytes = 0;
    const PullParams& b = up->built;
    p->work = b.work;
    p->status = b.status;
    p->items = b.items;
    p->n_items = b.n_items;
    p->srcs = b.srcs;
    p->n_srcs = b.n_srcs;
    p->maps = b.maps;
    p->batch_seg = b.batch_seg;
    p->n_chunks = b.n_chunks;
    p->n_batches = b.n_batches;
    p->has_cast = b.has_cast;
    p->order = b.order;
    p->n_sched = b.n_sched;
    return cudaSuccess;
  }
  std::vector<ItemDesc> key(items, items + n);  // the request, before flags are added below
  const std::size_t items_off = kHdr;
  const std::size_t srcs_off = items_off + n * sizeof(ItemDesc);
  const std::size_t maps_off = (srcs_off + n_srcs * sizeof(SrcDesc) + 255) / 256 * 256;
  const std::size_t bseg_off = maps_off + std::size_t(n) * 256;
  // batch -> last segment starting at or before the batch's first chunk
  std::vector<std::uint32_t> bseg(n_batches);
  for (std::uint32_t b = 0, sgi = 0; b < n_batches; ++b) {
    while (sgi + 1 < n && items[sgi + 1].chunk0 <= b * kBatchChunks) ++sgi;
    bseg[b] = sgi;
  }
  const std::vector<std::uint32_t> order = schedule_order(items, n, bseg);
  const std::size_t order_off = bseg_off + std::size_t(n_batches) * 4;
  const std::size_t total = order_off + order.size() * 4;
  if (up->scratch_bytes < total) {
    if (up->scratch) cudaFree(up->scratch);
    up->scratch = nullptr;
    up->scratch_bytes = 0;
    up->last.clear();
    cudaError_t e = cudaMalloc(&up->scratch, total);
    if (e != cudaSuccess) return e;
    up->scratch_bytes = total;
  }
  std::vector<std::uint8_t> host(total, 0);
  bool any_map = false;
  std::uint32_t any_cast = 0;
  for (std::uint32_t i = 0; i < n; ++i) {
    ItemDesc& d = items[i];
    const std::uint64_t c = d.chunk_len & kChunkLenMask;
    const bool cast = (d.chunk_len & kCastE4M3) != 0;
    any_cast |= cast ? 1u : 0u;  // lands from registers: no dst map
    d.chunk_len = static_cast<std::uint32_t>(c) | (cast ? kCastE4M3 : 0u);
    if (d.q == 0) d.q = 1;
    if (d.m == 0) d.m = d.q;
    const std::uint64_t q = d.q, m = d.m;
    const std::uint64_t full = c ? d.len / c : 0;  // whole chunks in the segment
    // A segment read from a peer GPU (link class >= 2) takes the slot path:
    // per-lane bulk copies read each chunk as contiguous 512-byte pieces,
    // which the peer's HBM serves better than 32-row boxes of 128 bytes when
    // it is busy with its own pull (config 3 at N=2: 13.1 -> 12.3 ms with
    // every segment on slots); one-way and ring pulls are equal either way.
    bool ok = !maps_disabled() && d.src && (d.pad == 0 || peer_boxes()) && c % kMapBoxCols == 0 &&
              d.src % 16 == 0 &&
              d.dst % 16 == 0 && full >= 32 && (32 % q) == 0 && (full % q) == 0;
    if (ok) {
      auto* mp = reinterpret_cast<CUtensorMap*>(host.data() + maps_off + 256 * std::size_t(i));
      // 2-D: one row per chunk; 3-D: one row per source row (q chunks each)
      ok = encode(mp, d.src, c, q, m, q == m ? full : full / q);
      if (ok && d.dst && !cast) ok = encode(mp + 1, d.dst, c, 1, 1, full);
      // e4m3 landing rows of c/2 bytes: whole 128-byte boxes needed
      if (ok && d.dst && cast && c / 2 >= kMapBoxCols && encode(mp + 1, d.dst, c / 2, 1, 1, full))
        d.chunk_len |= kCastMap;
    }
    if (ok) {
      d.chunk_len |= kHasMap | (q < m ? kMap3D : 0u);
      any_map = true;
    }
  }
  std::memcpy(host.data() + items_off, items, n * sizeof(ItemDesc));
  if (n_srcs) std::memcpy(host.data() + srcs_off, srcs, n_srcs * sizeof(SrcDesc));
  if (n_batches) std::memcpy(host.data() + bseg_off, bseg.data(), std::size_t(n_batches) * 4);
  if (!order.empty()) std::memcpy(host.data() + order_off, order.data(), order.size() * 4);
  if (plan_debug()) print_plan_stats(items, n, bseg, n_chunks);
  auto* base = static_cast<std::uint8_t*>(up->scratch);
  cudaError_t e;
  if (up->last.size() == total && std::memcmp(up->last.data(), host.data(), total) == 0) {
    e = cudaMemsetAsync(base, 0, kHdr, s);  // same plan resident: fresh work/status words
    up->h2d_bytes = 0;
  } else {
    e = cudaMemcpyAsync(base, host.data(), total, cudaMemcpyHostToDevice, s);
    up->h2d_bytes = total;
    up->last = std::move(host);
  }
  if (e != cudaSuccess) return e;
  p->work = reinterpret_cast<std::uint32_t*>(base);
  p->status = reinterpret_cast<PullStatus*>(base + 64);
  p->items = reinterpret_cast<const ItemDesc*>(base + items_off);
  p->n_items = n;
  p->srcs = reinterpret_cast<const SrcDesc*>(base + srcs_off);
  p->n_srcs = n_srcs;
  p->maps = any_map ? base + maps_off : nullptr;
  p->batch_seg = reinterpret_cast<const std::uint32_t*>(base + bseg_off);
  p->n_chunks = n_chunks;
  p->has_cast = any_cast;
  p->n_batches = n_batches;
  p->order = order.empty() ? nullptr : reinterpret_cast<const std::uint32_t*>(base + order_off);
  p->n_sched = static_cast<std::uint32_t>(order.size());
  up->built = *p;
  up->key_items = std::move(key);
  up->key_srcs.assign(srcs, srcs + n_srcs);
  up->key_chunks = n_chunks;
  (void)device;
  return cudaSuccess;
}

void free_pull_plan(int device, PlanUpload* up) {
  if (!up->scratch) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaFree(up->scratch);
  cudaSetDevice(prev);
  up->scratch = nullptr;
  up->scratch_bytes = 0;
  up->last.clear();
  up->key_items.clear();
  up->key_srcs.clear();
}

}  // namespace rsb::dev
