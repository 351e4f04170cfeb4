// K1+K2 (+K4 reshard) on the TMA path: the fused pull + per-chunk XXH64
// verify + watermark kernel.  Replaces copy_slice_locked (transport.cpp:51-69)
// and the per-item digest64 check of TransferTask::verify_ready
// (client_core.cpp:306-334); with segment mappings (ItemDesc q < m, several
// sources) it also performs the TP/FSDP reshard gather/split.
//
// Warp-specialized, persistent: a pipeline is one producer warp and one
// consumer warp sharing a ring of S stages in shared memory; a CTA holds
// PIPES pipelines (default: one CTA per SM with four, so the four hashing
// consumers sit on the four SM sub-partitions).  A stage holds the next P
// bytes of each of the 32 chunks of one watermark batch; lane l of the
// consumer hashes landing chunk 32b+l.
//
// Two stage layouts:
//  * box (the common case: all 32 chunks of the batch are whole chunks of one
//    segment that has TMA tensor maps).  A stage is P/128 boxes of
//    [32 chunks x 128 B] with 128-byte swizzle, each moved by ONE
//    cp.async.bulk.tensor load (2-D for contiguous segments, 3-D
//    [rows][q][chunk] for a column band of a row-split reshard) and landed by
//    ONE 2-D tensor store, both issued by a single lane.  The swizzle keeps
//    the per-chunk 128-bit reads of the hash lanes bank-conflict free.
//  * slot (batches with a short last chunk, holes, mixed segments, unaligned
//    regions): one padded slot of P+16 bytes per chunk, every lane issuing
//    its own cp.async.bulk copy (plain loads/stores for unaligned bytes).
//
//   producer  walks its batches (static schedule: position pipeline +
//             k*pipelines of the plan's batches in order, so the landed
//             prefix advances front to back), waits the source
//             watermark(s) when a source is still filling, fills stages.
//   consumer  per stage: lands the stage (tensor store / bulk stores), hashes
//             (XXH64 32-byte stripes), frees the stage once the stores have
//             read it.  After a batch's last step it verifies the 32 chunk
//             digests against the sources' tables (one quiet re-pull of a bad
//             chunk), writes its own digest table, and one stage later --
//             when the batch's stores have completed -- publishes the batch
//             watermark (fence.proxy.async + st.release.sys, cumulative over
//             the warp through __syncwarp).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "dev_common.cuh"
#include "device.hpp"

namespace rsb::dev {

using namespace detail;

namespace {

constexpr std::uint32_t kPill = 0xffffffffu;

__device__ __forceinline__ void tensor_load_2d(void* smem, const void* map, int x, int y,
                                               unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(smem)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tensor_load_3d(void* smem, const void* map, int x, int y, int z,
                                               unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(smem)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tensor_store_2d(const void* map, int x, int y, const void* smem) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(map),
      "r"(x), "r"(y), "r"(smem_u32(smem))
      : "memory");
}

template <int P, int S, int CTAS, int ITEMS, int PIPES = 1, int REL = 4, bool DYN = false>
struct Cfg {
  static constexpr int kRelease = REL;  // verified batches per watermark release (one sys fence)
  // DYN: pipelines claim schedule positions from a global ticket (work[0])
  // instead of the static stride, so a pipeline held up by a slow batch (a
  // remote source whose HBM is busy) does not hold back the positions after it
  static constexpr bool kDynamic = DYN;
  static constexpr int kPipes = PIPES;  // producer/consumer pairs per CTA
  static constexpr int kThreads = 64 * PIPES;
  static constexpr int kP = P;
  static constexpr int kSlot = P + 16;
  static constexpr int kStage = (32 * kSlot + 1023) / 1024 * 1024;  // box layout needs 1 KiB
  static constexpr int kStages = S;
  static constexpr int kCtas = CTAS;
  static constexpr int kItems = ITEMS;
  static_assert(P % kMapBoxCols == 0, "piece must be whole boxes");

  struct Meta {
    std::uint32_t batch;
    std::uint32_t step;
    std::uint32_t last;
    std::uint32_t box;     // 1: box layout
    std::uint32_t item;    // box layout: segment index
    std::uint32_t k0;      // box layout: first chunk of the batch within the segment
    std::uint32_t g;       // box layout: byte offset of the step within the chunk
    std::uint32_t bpiece;  // box layout: bytes per chunk in this step
    std::uint32_t cast;    // lanes whose chunk lands as e4m3
    std::uint32_t verify;  // lanes whose chunk has a source digest to check
    std::uint32_t store;   // box layout: land the boxes with tensor stores
    std::uint32_t pad;
    std::uint64_t dst[32];
    std::uint32_t piece[32];
    std::uint32_t clen[32];
    std::uint32_t seg[32];  // segment of each lane's chunk
    std::uint64_t expect[32];
  };
  // One pipeline: a ring of S stages between a producer and a consumer warp.
  struct alignas(1024) Pipe {
    std::uint8_t stage[S][kStage];
    Meta meta[S];
    unsigned long long full[S];
    unsigned long long empty[S];
  };
  struct Smem {
    Pipe pipes[PIPES];
    // ITEMS == 0: segments stay in global; copied in with 16-byte vectors
    alignas(16) ItemDesc items[ITEMS > 0 ? ITEMS : 1];
  };
  static constexpr int kSmemBytes = static_cast<int>(sizeof(Smem)) + 1024;
};

template <class C>
__global__ void __launch_bounds__(C::kThreads, C::kCtas) pull_tma_kernel(const PullParams p) {
  if (p.guard && *reinterpret_cast<const volatile std::uint32_t*>(p.guard) != 0) return;  // follow-up of a failed fill
  using Smem = typename C::Smem;
  using Meta = typename C::Meta;
  constexpr int kP = C::kP;
  constexpr int kStages = C::kStages;
  extern __shared__ __align__(1024) std::uint8_t smraw[];
  const std::uint32_t mis = smem_u32(smraw) & 1023u;  // 1 KiB-align the stages
  Smem& sm = *reinterpret_cast<Smem*>(smraw + (mis ? 1024 - mis : 0));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const std::uint8_t* maps = static_cast<const std::uint8_t*>(p.maps);
  auto advance = [](int& stage, unsigned& phase) {
    if (++stage == kStages) {
      stage = 0;
      phase ^= 1;
    }
  };

  const bool smem_items = C::kItems > 0 && p.n_items <= static_cast<std::uint32_t>(C::kItems);
  if (smem_items) {
    const uint4* s = reinterpret_cast<const uint4*>(p.items);
    uint4* d = reinterpret_cast<uint4*>(sm.items);
    const std::uint32_t n16 = p.n_items * (sizeof(ItemDesc) / 16);
    for (std::uint32_t i = threadIdx.x; i < n16; i += blockDim.x) d[i] = s[i];
  }
  if (threadIdx.x == 0) {
    for (int qq = 0; qq < C::kPipes; ++qq)
      for (int s = 0; s < kStages; ++s) {
        mbar_init(&sm.pipes[qq].full[s], 1);
        mbar_init(&sm.pipes[qq].empty[s], 1);
      }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const ItemDesc* items = smem_items ? sm.items : p.items;
  // Warps 0..PIPES-1 consume, PIPES..2*PIPES-1 produce; pipeline q pairs
  // consumer q with producer PIPES+q.  With PIPES == 4 the four consumers
  // (the hashing warps) sit on the four SM sub-partitions, one each.
  const int q = warp % C::kPipes;
  typename C::Pipe& pp = sm.pipes[q];
  // each pipeline is a virtual CTA of the persistent batch schedule
  const std::uint32_t vcta = blockIdx.x * C::kPipes + q;
  const std::uint32_t vgrid = gridDim.x * C::kPipes;

  if (warp >= C::kPipes) {
    // ================================ producer ==============================
    int stage = 0;
    unsigned phase = 0;
    std::uint32_t abort_seen = 0;
    const std::uint32_t* order = p.order;
    const std::uint32_t pos_end = order ? p.n_sched : p.n_batches;
    const std::uint32_t pos0 = order ? 0 : p.first_batch;
    auto claim = [&]() {  // next position of this pipeline
      std::uint32_t t = 0;
      if (lane == 0) t = atomicAdd(&p.work[0], 1u);
      return pos0 + __shfl_sync(full, t, 0);
    };
    std::uint32_t next = C::kDynamic ? claim() : pos0 + vcta;
    for (std::uint32_t pos = next; pos < pos_end; pos = next) {
      next = C::kDynamic ? claim() : pos + vgrid;  // claimed a batch ahead: latency hidden
      if (abort_seen) break;
      const std::uint32_t b = order ? __ldg(&order[pos]) : pos;
      const std::uint32_t abort_next = ld_volatile(&p.work[1]);  // acted on next batch
      if (p.resume && ld_volatile(&p.dst_flags[b]) == p.dst_epoch) {  // landed already
        abort_seen = abort_next;
        continue;
      }
      const std::uint32_t c = b * kBatchChunks + lane;
      ChunkRef r{nullptr, nullptr, 0u, 0u};
      std::uint32_t seg = 0xffffffffu, cunit = 0, itflags = 0, k = 0, src_id = 0;
      const std::uint32_t bseg = __ldg(&p.batch_seg[b]);
      if (c < p.n_chunks) {
        seg = seg_of(items, p.n_items, bseg, c);
        const ItemDesc d = items[seg];
        cunit = d.chunk_len & kChunkLenMask;
        itflags = d.chunk_len & (kHasMap | kMap3D);
        k = c - d.chunk0;
        r = chunk_ref(d, k);
        src_id = d.src_id;
      }
      // Chase the source watermark(s) when the source is still filling.
      const SrcDesc* sd = r.clen ? &p.srcs[src_id] : nullptr;
      std::uint32_t code = kPullOk;
      const std::uint32_t sbatch = r.src_chunk / kBatchChunks;
      const std::uint32_t sb0 = __shfl_sync(full, sbatch, 0);
      const std::uint32_t sid0 = __shfl_sync(full, src_id, 0);
      const bool need0 = __shfl_sync(full, sd != nullptr && sd->flags != nullptr, 0);
      if (lane == 0 && need0)
        code = wait_flag(&sd->flags[sbatch >> sd->flag_shift], sd->epoch, p.timeout_ns, &p.work[1]);
      if (sd && sd->flags && (sbatch != sb0 || src_id != sid0) && lane != 0)
        code = wait_flag(&sd->flags[sbatch >> sd->flag_shift], sd->epoch, p.timeout_ns, &p.work[1]);
      const std::uint32_t worst = __reduce_max_sync(full, code);
      if (worst != kPullOk) {
        // diagnostics: the source batch and the watermark value that failed
        const unsigned bad_lanes = __ballot_sync(full, code == worst);
        const int bl = __ffs(bad_lanes) - 1;
        const std::uint32_t bsb = __shfl_sync(full, sbatch, bl);
        const std::uint32_t bfv = (lane == bl && sd && sd->flags) ? ld_volatile(&sd->flags[sbatch >> sd->flag_shift]) : 0u;
        const std::uint32_t bflag = __shfl_sync(full, bfv, bl);
        if (lane == 0) {
          if (worst != kPullAborted) {
            atomicCAS(&p.status->code, 0u, worst);
            atomicExch(&p.status->bad_chunk, b * kBatchChunks);
            atomicExch(reinterpret_cast<unsigned long long*>(&p.status->pad),
                       (static_cast<unsigned long long>(bsb) << 32) | bflag);
          }
          atomicExch(&p.work[1], 1u);
          if (p.dst_flags) st_release_sys(&p.dst_flags[b], p.dst_epoch | kAbort);
        }
        break;
      }
      if (__any_sync(full, sd != nullptr && sd->flags != nullptr)) fence_proxy_async_global();
      const bool has_expect = sd && sd->digests;
      // Expected digests: when the batch's 32 source chunks are consecutive
      // in one source table (the common case) they arrive as ONE 256-byte
      // bulk copy into the last stage's metadata, asynchronously like the
      // data; otherwise each lane loads its own (that load's latency then
      // stalls this warp once per batch -- costly when the link is loaded).
      const std::uint32_t sc0 = __shfl_sync(full, r.src_chunk, 0);
      const bool dig_bulk = __all_sync(full, has_expect && r.clen != 0 && src_id == sid0 &&
                                                 r.src_chunk == sc0 + lane) &&
                            (sc0 & 1u) == 0;
      const std::uint64_t* dig_src = dig_bulk ? p.srcs[sid0].digests + sc0 : nullptr;
      const std::uint64_t expect = (has_expect && !dig_bulk) ? __ldcg(&sd->digests[r.src_chunk]) : 0;
      const std::uint32_t verify_mask = __ballot_sync(full, has_expect);
      const bool is_cast = r.clen && seg < p.n_items && (items[seg].chunk_len & kCastE4M3);
      const std::uint32_t cast_mask = __ballot_sync(full, is_cast);
      const std::uint32_t seg0 = __shfl_sync(full, seg, 0);
      const std::uint32_t k0 = __shfl_sync(full, k, 0);
      const std::uint32_t q0 = seg0 < p.n_items ? items[seg0].q : 1;
      const bool box = maps != nullptr &&
                       __all_sync(full, seg == seg0 && (itflags & kHasMap) && r.clen == cunit &&
                                            r.clen != 0) &&
                       (k0 % q0) == 0;
      const bool map3d = box && (items[seg0].chunk_len & kMap3D) != 0;
      // 1: land the boxes with tensor stores; 2: cast into the stage, then
      // land the e4m3 boxes with tensor stores; 0: the consumer stores
      const std::uint32_t box_store =
          !box ? 0u
               : cast_mask == 0 ? (items[seg0].dst != 0 ? 1u : 0u)
                                : (cast_mask == full && (items[seg0].chunk_len & kCastMap) ? 2u : 0u);
      std::uint32_t maxlen = r.clen;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(full, maxlen, o));
      const std::uint32_t nsteps = (maxlen + kP - 1) / kP;
      const bool src_vec = (reinterpret_cast<std::uintptr_t>(r.src) & 15) == 0;
      for (std::uint32_t s = 0; s < nsteps; ++s) {
        mbar_wait(&pp.empty[stage], phase ^ 1);
        Meta& m = pp.meta[stage];
        const std::uint32_t g = s * kP;
        const std::uint32_t piece =
            g < r.clen ? min(static_cast<std::uint32_t>(kP), r.clen - g) : 0;
        const bool last = s + 1 == nsteps;
        m.piece[lane] = piece;
        m.clen[lane] = r.clen;
        m.dst[lane] = r.dst ? reinterpret_cast<std::uint64_t>(r.dst + (is_cast ? g / 2 : g)) : 0;
        if (last) {
          if (!dig_bulk) m.expect[lane] = expect;
          m.seg[lane] = seg;
        }
        const std::uint32_t dig_tx = (last && dig_bulk) ? 256u : 0u;
        if (dig_tx && lane == 0) fence_proxy_async_smem();  // earlier generic writes of m.expect
        if (lane == 0) {
          m.cast = cast_mask;
          m.verify = verify_mask;
          m.store = box_store;
        }
        if (box) {
          if (lane == 0) {
            m.batch = b;
            m.step = s;
            m.last = last;
            m.box = 1;
            m.item = seg0;
            m.k0 = k0;
            m.g = g;
            m.bpiece = piece;
          }
          __syncwarp();
          if (lane == 0) {
            mbar_arrive_tx(&pp.full[stage], 32 * piece + dig_tx);
            if (dig_tx) bulk_g2s(m.expect, dig_src, dig_tx, &pp.full[stage]);
            const void* map = maps + 256 * std::size_t(seg0);
            const std::uint32_t qq = q0;
            for (std::uint32_t j = 0; j < piece / kMapBoxCols; ++j) {
              const int x = static_cast<int>(g + j * kMapBoxCols);
              if (map3d)
                tensor_load_3d(pp.stage[stage] + j * 4096, map, x, 0, static_cast<int>(k0 / qq),
                               &pp.full[stage]);
              else
                tensor_load_2d(pp.stage[stage] + j * 4096, map, x, static_cast<int>(k0),
                               &pp.full[stage]);
            }
          }
        } else {
          std::uint8_t* slot = pp.stage[stage] + lane * C::kSlot;
          const std::uint32_t bulk = src_vec ? (piece & ~15u) : 0;
          for (std::uint32_t kk = bulk; kk < piece; ++kk) slot[kk] = __ldcg(r.src + g + kk);
          std::uint32_t tx = bulk;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) tx += __shfl_xor_sync(full, tx, o);
          if (lane == 0) {
            m.batch = b;
            m.step = s;
            m.last = last;
            m.box = 0;
          }
          __syncwarp();
          if (lane == 0) {
            mbar_arrive_tx(&pp.full[stage], tx + dig_tx);
            if (dig_tx) bulk_g2s(m.expect, dig_src, dig_tx, &pp.full[stage]);
          }
          __syncwarp();
          if (bulk) bulk_g2s(slot, r.src + g, bulk, &pp.full[stage]);
        }
        advance(stage, phase);
      }
      abort_seen = abort_next;
    }
    mbar_wait(&pp.empty[stage], phase ^ 1);  // poison pill: nothing more
    if (lane == 0) {
      pp.meta[stage].batch = kPill;
      mbar_arrive(&pp.full[stage]);
    }
  } else {
    // ================================ consumer ==============================
    int stage = 0;
    unsigned phase = 0;
    std::uint64_t v1 = 0, v2 = 0, v3 = 0, v4 = 0, digest = 0;
    // Verified batches whose watermarks await their stores.  Released
    // kRelease at a time: one system-scope fence per group of flags.
    constexpr int kRelease = C::kRelease;
    std::uint32_t pend[kRelease];
    int npend = 0;
    std::uint64_t pend_bytes = 0, done_bytes = 0;
    bool failed = false;
    const std::uint32_t swz = (static_cast<std::uint32_t>(lane) & 7u) << 4;
    auto release_pending = [&](bool newer_group, bool force) {
      if (npend == 0 || (!force && npend < kRelease)) return;
      if (newer_group) bulk_wait<1>();
      else bulk_wait<0>();
      fence_proxy_async_global();
      __syncwarp();
      if (lane == 0 && p.dst_flags) {
        fence_release_sys();
#pragma unroll
        for (int i = 0; i < kRelease; ++i)
          if (i < npend) st_relaxed_sys(&p.dst_flags[pend[i]], p.dst_epoch);
      }
      if (lane == 0) atomicAdd(&p.status->batches_done, static_cast<std::uint32_t>(npend));
      done_bytes += pend_bytes;
      npend = 0;
      pend_bytes = 0;
    };
    for (;;) {
      mbar_wait(&pp.full[stage], phase);
      const Meta& m = pp.meta[stage];
      const std::uint32_t b = m.batch;
      if (b == kPill) break;
      if (failed) {  // drain until the pill
        __syncwarp();
        if (lane == 0) mbar_arrive(&pp.empty[stage]);
        advance(stage, phase);
        continue;
      }
      const std::uint32_t s = m.step;
      const std::uint32_t piece = m.piece[lane];
      const std::uint32_t clen = m.clen[lane];
      const bool last = m.last != 0;
      const bool box = m.box != 0;
      std::uint8_t* st = pp.stage[stage];
      bool committed = false;
      if (s == 0) {
        v1 = kP1 + kP2;
        v2 = kP2;
        v3 = 0;
        v4 = 0 - kP1;
      }
      const int stripes = static_cast<int>(piece >> 5);
      const bool lane_cast = (m.cast >> lane) & 1u;
      auto* castp = reinterpret_cast<uint4*>(lane_cast ? m.dst[lane] : 0);  // e4m3 landing
      if (box) {
        // 1) land: one tensor store per box, issued by lane 0 (a cast batch
        //    lands from registers in the hash loop instead)
        if (lane == 0 && m.store == 1) {
          const std::uint8_t* dmap = maps + 256 * std::size_t(m.item) + 128;
          fence_proxy_async_smem();
          for (std::uint32_t j = 0; j < m.bpiece / kMapBoxCols; ++j)
            tensor_store_2d(dmap, static_cast<int>(m.g + j * kMapBoxCols), static_cast<int>(m.k0),
                            st + j * 4096);
          bulk_commit();
          committed = true;
        }
        // 2) hash chunk `lane` = row `lane` of the swizzled boxes (a cast
        //    lane also lands the e4m3 of each stripe; separate loops keep
        //    the plain loop free of the cast)
        const std::uint8_t* rowbase = st + lane * 128;
        auto box_stripe = [&](int kk, uint4& a, uint4& q) {
          const std::uint8_t* boxp = rowbase + (kk >> 2) * 4096;
          const std::uint32_t x = static_cast<std::uint32_t>(kk & 3) * 32;
          a = *reinterpret_cast<const uint4*>(boxp + (x ^ swz));
          q = *reinterpret_cast<const uint4*>(boxp + ((x + 16) ^ swz));
          v1 = xround(v1, (std::uint64_t(a.y) << 32) | a.x);
          v2 = xround(v2, (std::uint64_t(a.w) << 32) | a.z);
          v3 = xround(v3, (std::uint64_t(q.y) << 32) | q.x);
          v4 = xround(v4, (std::uint64_t(q.w) << 32) | q.z);
        };
        if (m.store == 2) {
          // e4m3 of stripe kk = 16-byte granule kk of the lane's output row,
          // written in place over stage bytes already read (output box kk>>3
          // lies in input box <= kk>>2, output granule kk&7 at or before the
          // input granules just read), in the same 128B-swizzled box layout
#pragma unroll 4
          for (int kk = 0; kk < stripes; ++kk) {
            uint4 a, q;
            box_stripe(kk, a, q);
            *reinterpret_cast<uint4*>(st + (kk >> 3) * 4096 + lane * 128 +
                                      ((static_cast<std::uint32_t>(kk & 7) << 4) ^ swz)) =
                cvt16_e4m3(a, q);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const std::uint8_t* dmap = maps + 256 * std::size_t(m.item) + 128;
            for (std::uint32_t j = 0; j < (m.bpiece / 2 + kMapBoxCols - 1) / kMapBoxCols; ++j)
              tensor_store_2d(dmap, static_cast<int>(m.g / 2 + j * kMapBoxCols), static_cast<int>(m.k0),
                              st + j * 4096);
            bulk_commit();
            committed = true;
          }
        } else if (castp) {
#pragma unroll 4
          for (int kk = 0; kk < stripes; ++kk) {
            uint4 a, q;
            box_stripe(kk, a, q);
            castp[kk] = cvt16_e4m3(a, q);
          }
        } else {
#pragma unroll 4
          for (int kk = 0; kk < stripes; ++kk) {
            uint4 a, q;
            box_stripe(kk, a, q);
          }
        }
        if (clen && s * kP + piece == clen) {
          std::uint64_t h = clen >= 32 ? merge4(v1, v2, v3, v4) : kP5;
          h += clen;
          digest = finish_tail(h, nullptr, 0);  // whole 128-byte rows: no tail
        }
      } else {
        std::uint8_t* slot = st + lane * C::kSlot;
        const std::uint64_t dstp = m.dst[lane];
        if (dstp && piece && !lane_cast) {
          const std::uint32_t bulk = (dstp & 15) == 0 ? (piece & ~15u) : 0;
          if (bulk) {
            fence_proxy_async_smem();
            bulk_s2g(reinterpret_cast<void*>(dstp), slot, bulk);
            bulk_commit();
            committed = true;
          }
          for (std::uint32_t kk = bulk; kk < piece; ++kk)
            reinterpret_cast<std::uint8_t*>(dstp)[kk] = slot[kk];
        }
        auto slot_stripe = [&](int kk, uint4& a, uint4& q) {
          a = *reinterpret_cast<const uint4*>(slot + 32 * kk);
          q = *reinterpret_cast<const uint4*>(slot + 32 * kk + 16);
          v1 = xround(v1, (std::uint64_t(a.y) << 32) | a.x);
          v2 = xround(v2, (std::uint64_t(a.w) << 32) | a.z);
          v3 = xround(v3, (std::uint64_t(q.y) << 32) | q.x);
          v4 = xround(v4, (std::uint64_t(q.w) << 32) | q.z);
        };
        if (!castp) {
#pragma unroll 4
          for (int kk = 0; kk < stripes; ++kk) {
            uint4 a, q;
            slot_stripe(kk, a, q);
          }
        } else if ((reinterpret_cast<std::uintptr_t>(castp) & 15) == 0) {
#pragma unroll 4
          for (int kk = 0; kk < stripes; ++kk) {
            uint4 a, q;
            slot_stripe(kk, a, q);
            castp[kk] = cvt16_e4m3(a, q);
          }
        } else {  // unaligned e4m3 landing: byte stores
          for (int kk = 0; kk < stripes; ++kk) {
            uint4 a, q;
            slot_stripe(kk, a, q);
            const uint4 o = cvt16_e4m3(a, q);
            auto* cb = reinterpret_cast<std::uint8_t*>(castp) + 16 * kk;
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
              cb[bb] = static_cast<std::uint8_t>(o.x >> (8 * bb));
              cb[4 + bb] = static_cast<std::uint8_t>(o.y >> (8 * bb));
              cb[8 + bb] = static_cast<std::uint8_t>(o.z >> (8 * bb));
              cb[12 + bb] = static_cast<std::uint8_t>(o.w >> (8 * bb));
            }
          }
        }
        if (castp && (piece & 31u))
          cvt_tail_e4m3(slot + (piece & ~31u), reinterpret_cast<std::uint8_t*>(castp) + (piece & ~31u) / 2,
                        static_cast<int>(piece & 31u));
        if (clen && s * kP + piece == clen) {
          std::uint64_t h = clen >= 32 ? merge4(v1, v2, v3, v4) : kP5;
          h += clen;
          digest = finish_tail(h, slot + (piece & ~31u), static_cast<int>(piece & 31u));
        }
      }
      const std::uint64_t expect = last ? m.expect[lane] : 0;
      const std::uint32_t myseg = last ? m.seg[lane] : 0;
      const bool verify = (m.verify >> lane) & 1u;
      // 3) earlier batches' stores are done by now: publish their watermarks
      release_pending(committed, false);
      // 4) free the stage once the stores issued from it have read it
      if (committed) bulk_wait_read<0>();
      __syncwarp();
      if (lane == 0) mbar_arrive(&pp.empty[stage]);
      advance(stage, phase);
      if (!last) continue;
      // 5) batch complete: verify and record
      const std::uint32_t c = b * kBatchChunks + lane;
      bool lane_ok = !clen || !verify || digest == expect;
      if (__ballot_sync(full, !lane_ok)) {
        if (lane == 0) atomicAdd(&p.status->retried_batches, 1u);
        bulk_wait<0>();  // earlier stores of these chunks must not land after the re-pull
        if (!lane_ok) {
          const ItemDesc* dseg = &items[myseg];
          const ChunkRef rr = chunk_ref(*dseg, c - dseg->chunk0);
          digest = repull_chunk(rr.src, rr.dst, clen, (dseg->chunk_len & kCastE4M3) != 0);
          lane_ok = digest == expect;
        }
        const unsigned bad = __ballot_sync(full, !lane_ok);
        if (bad) {
          if (lane == 0) {
            atomicCAS(&p.status->code, 0u, static_cast<std::uint32_t>(kPullChecksum));
            atomicExch(&p.status->bad_chunk, b * kBatchChunks + (__ffs(bad) - 1));
            atomicExch(&p.work[1], 1u);
            if (p.dst_flags) st_release_sys(&p.dst_flags[b], p.dst_epoch | kAbort);
          }
          failed = true;
          continue;
        }
      }
      if (p.dst_digests && clen) p.dst_digests[c] = digest;
      std::uint64_t landed = clen;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) landed += __shfl_xor_sync(full, landed, o);
#pragma unroll
      for (int i = kRelease - 1; i > 0; --i) pend[i] = pend[i - 1];  // registers: constant indices
      pend[0] = b;
      ++npend;
      pend_bytes += landed;
    }
    release_pending(false, true);
    bulk_wait<0>();
    if (lane == 0 && done_bytes)
      atomicAdd(reinterpret_cast<unsigned long long*>(&p.status->bytes),
                static_cast<unsigned long long>(done_bytes));
  }
}

template <class C>
cudaError_t launch_variant(const PullParams& p, int sms, cudaStream_t s) {
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(pull_tma_kernel<C>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  const std::uint32_t todo = p.order ? p.n_sched : p.n_batches - p.first_batch;
  int grid = sms * C::kCtas;
  const auto per = static_cast<std::uint32_t>(C::kPipes);
  if (static_cast<std::uint32_t>(grid) * per > todo) grid = static_cast<int>((todo + per - 1) / per);
  pull_tma_kernel<C><<<grid, C::kThreads, C::kSmemBytes, s>>>(p);
  return cudaGetLastError();
}

// The three shapes the product path launches.
using V13 = Cfg<512, 2, 1, 320, 4, 4, true>;  // 4 two-stage pipelines per SM, dynamic batch claiming
using V16 = Cfg<512, 2, 1, 320, 4, 1, true>;  // V13 releasing every batch at once (chain hops)
using V15 = Cfg<512, 3, 1, 0, 4, 4, true>;    // 3 stages, segments in global: fused-cast pulls
#ifdef RSB_ALL_VARIANTS
// Diagnostic shapes from the round-1 sweeps (profiles/r1/variants*.txt);
// built only with RSB_ALL_VARIANTS=1 (python -m paper_2604_09107_b200.build).
using V0 = Cfg<512, 3, 3, 320>;
using V1 = Cfg<512, 4, 2, 576>;
using V2 = Cfg<1024, 3, 2, 192>;
using V3 = Cfg<256, 6, 3, 192>;
using V4 = Cfg<512, 3, 4, 0>;  // segment table in global (L1-cached): 4 CTAs per SM
using V5 = Cfg<512, 2, 6, 0>;  // 2-stage rings, 6 CTAs per SM
using V6 = Cfg<256, 3, 7, 0>;  // 7 CTAs per SM
using V7 = Cfg<512, 3, 1, 0, 4>;    // one CTA per SM: 4 pipelines, consumers on 4 sub-partitions
using V8 = Cfg<512, 2, 1, 320, 4>;  // 4 two-stage pipelines + the segment table in smem
using V9 = Cfg<256, 4, 1, 320, 4>;  // 4 four-stage pipelines of 256-byte pieces
using V10 = Cfg<256, 5, 1, 128, 4>;
using V11 = Cfg<512, 2, 1, 320, 4, 8>;   // V8, releasing 8 batches per fence
using V12 = Cfg<512, 2, 1, 320, 4, 16>;  // V8, releasing 16 batches per fence
using V14 = Cfg<256, 4, 1, 320, 4, 4, true>;  // V9 (4 stages of 256 B) with dynamic claiming
using V17 = Cfg<512, 2, 1, 320, 4, 8, true>;  // V13 releasing 8 batches per fence
#endif

int variant() {  // -1: by workload
  static const int v = [] {
    const char* e = std::getenv("RSB_TMA_VARIANT");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}

}  // namespace

cudaError_t launch_pull_tma(const PullParams& p, int sms, cudaStream_t s) {
  // Default V13: one CTA per SM with four producer/consumer pipelines (two
  // stages each), so the four hashing warps sit on the four sub-partitions,
  // claiming batches dynamically.  A plain peer pull (remote == 2: a chain
  // hop) takes V16, the same shape releasing every verified batch at once:
  // the chaser behind it sees batches sooner (config 2 N=4 last hop
  // 646-649 -> 653-657 GB/s), while local cast and reshard pulls lose 8-15%
  // with per-batch fences and stay on V13.  Measured on B200: local plain pull 99.9%
  // of the measured HBM copy peak (V8, the same shape on a static stride:
  // 91-92%, its fastest pipelines idling at the tail; V0, 3 two-warp CTAs:
  // 88-90%), FSDP-8 -> TP-2 reshard 97.5% (V8: 91%); over NVLink equal to V8
  // (785 GB/s one way, 672 with both directions busy).
  // A pull that lands e4m3 (has_cast) takes V15, a third stage per
  // pipeline: the consumers also convert every value into the stage before
  // the tensor store, and the deeper ring hides it (config 5 N=1: 4.17 ->
  // 3.95 ms; V17, releasing 8 batches per fence: 4.08).
  int v = variant();
  if (v < 0) v = p.remote == 2 ? 16 : p.has_cast ? 15 : 13;
  switch (v) {
    case 13: return launch_variant<V13>(p, sms, s);
    case 16: return launch_variant<V16>(p, sms, s);
    case 15: return launch_variant<V15>(p, sms, s);
#ifdef RSB_ALL_VARIANTS
    case 0: return launch_variant<V0>(p, sms, s);
    case 1: return launch_variant<V1>(p, sms, s);
    case 2: return launch_variant<V2>(p, sms, s);
    case 3: return launch_variant<V3>(p, sms, s);
    case 4: return launch_variant<V4>(p, sms, s);
    case 5: return launch_variant<V5>(p, sms, s);
    case 6: return launch_variant<V6>(p, sms, s);
    case 7: return launch_variant<V7>(p, sms, s);
    case 8: return launch_variant<V8>(p, sms, s);
    case 9: return launch_variant<V9>(p, sms, s);
    case 10: return launch_variant<V10>(p, sms, s);
    case 11: return launch_variant<V11>(p, sms, s);
    case 12: return launch_variant<V12>(p, sms, s);
    case 14: return launch_variant<V14>(p, sms, s);
    case 17: return launch_variant<V17>(p, sms, s);
#endif
    default: return cudaErrorNotSupported;  // a shape this build does not carry: fail loudly
  }
}

}  // namespace rsb::dev
