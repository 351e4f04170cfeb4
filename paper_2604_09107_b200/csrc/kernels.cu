// sm_100a kernels of the ROS read path (besides the TMA pull in pull_tma.cu).
//
//   pull_kernel        K1+K2 on the LDGSTS path (RSB_PULL_KERNEL=ldg): the
//                      same contract as pull_tma_kernel with cp.async 16-byte
//                      copies issued by every lane; kept as the variant for
//                      comparisons and as a fallback.
//   span_digest_kernel K6: reference-identical XXH64 of whole items/groups
//                      (digest64, digest.cpp:79-106) for the manifest.
//   copy_spans_kernel  K3: pack/unpack of tiny-tensor groups
//                      (pack_group / unpack_group, manifest.cpp:204-225).
//   synth_bf16_kernel  synthetic weights.
//   e4m3_kernel        K5: saturating RNE bf16 -> fp8 e4m3.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "dev_common.cuh"
#include "device.hpp"

namespace rsb::dev {

using namespace detail;

cudaError_t launch_pull_tma(const PullParams& p, int sms, cudaStream_t s);

namespace {

// ------------------------------------------------------- K1+K2, LDGSTS ----
// A warp owns one batch (lane l hashes chunk 32b+l); each step it stages the
// next 256 B of all 32 chunks with cp.async (16 B per lane, 256 B contiguous
// per half-warp), writes the stage to the destination with 128-bit stores
// and hashes its own slot.
constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;
constexpr int kSlot = kPiece + 16;
constexpr int kStageBytes = 32 * kSlot;
constexpr int kStages = 3;
constexpr int kSmemBytes = kWarps * kStages * kStageBytes;
constexpr int kUnits = 32 * kPiece / 16 / 32;

struct LaneChunk {
  const std::uint8_t* src;
  std::uint8_t* dst;
  std::uint32_t len;
  std::uint32_t cast;  // lands as e4m3 (the owning lane converts from its slot)
};

__device__ __forceinline__ void load_step(const LaneChunk* refs, std::uint8_t* stage, int s,
                                          int lane) {
  const int half = lane >> 4;
  const int off = (lane & 15) * 16;
#pragma unroll
  for (int u = 0; u < kUnits; ++u) {
    const int k = 2 * u + half;
    const LaneChunk r = refs[k];
    const std::uint32_t g = static_cast<std::uint32_t>(s) * kPiece + off;
    if (g >= r.len) continue;
    const std::uint8_t* src = r.src + g;
    std::uint8_t* dst = stage + k * kSlot + off;
    const std::uint32_t n = r.len - g;
    if (n >= 16 && (reinterpret_cast<std::uintptr_t>(src) & 15) == 0) {
      cp_async16(dst, src);
    } else {
      const std::uint32_t m = n < 16 ? n : 16;
      for (std::uint32_t b = 0; b < m; ++b) dst[b] = __ldcg(src + b);
    }
  }
}

__device__ __forceinline__ void store_step(const LaneChunk* refs, const std::uint8_t* stage,
                                           int s, int lane) {
  const int half = lane >> 4;
  const int off = (lane & 15) * 16;
#pragma unroll
  for (int u = 0; u < kUnits; ++u) {
    const int k = 2 * u + half;
    const LaneChunk r = refs[k];
    const std::uint32_t g = static_cast<std::uint32_t>(s) * kPiece + off;
    if (r.dst == nullptr || r.cast || g >= r.len) continue;
    const std::uint8_t* src = stage + k * kSlot + off;
    std::uint8_t* dst = r.dst + g;
    const std::uint32_t n = r.len - g;
    if (n >= 16 && (reinterpret_cast<std::uintptr_t>(dst) & 15) == 0) {
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
    } else {
      const std::uint32_t m = n < 16 ? n : 16;
      for (std::uint32_t b = 0; b < m; ++b) dst[b] = src[b];
    }
  }
}

__global__ void __launch_bounds__(kThreads, 2) pull_kernel(const PullParams p) {
  if (p.guard && *reinterpret_cast<const volatile std::uint32_t*>(p.guard) != 0) return;
  extern __shared__ __align__(128) std::uint8_t smem[];
  __shared__ LaneChunk refs_all[kWarps][32];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  std::uint8_t* wbuf = smem + warp * (kStages * kStageBytes);
  LaneChunk* refs = refs_all[warp];
  const unsigned full = 0xffffffffu;

  for (;;) {
    std::uint32_t b = 0;
    if (lane == 0) b = atomicAdd(&p.work[0], 1u) + (p.order ? 0u : p.first_batch);
    b = __shfl_sync(full, b, 0);
    if (b >= (p.order ? p.n_sched : p.n_batches)) break;
    if (p.order) b = __ldg(&p.order[b]);
    if (ld_volatile(&p.work[1])) break;
    if (p.resume && ld_volatile(&p.dst_flags[b]) == p.dst_epoch) continue;  // landed already
    const std::uint32_t c = b * kBatchChunks + lane;
    LaneChunk mine{nullptr, nullptr, 0u, 0u};
    std::uint64_t expect = 0;
    const SrcDesc* sd = nullptr;
    ChunkRef r{nullptr, nullptr, 0u, 0u};
    if (c < p.n_chunks) {
      const ItemDesc it = p.items[seg_of(p.items, p.n_items, p.batch_seg[b], c)];
      r = chunk_ref(it, c - it.chunk0);
      if (r.clen) {
        mine = {r.src, r.dst, r.clen, (it.chunk_len & kCastE4M3) ? 1u : 0u};
        sd = &p.srcs[it.src_id];
      }
    }
    // chase the source watermark (every lane its own source batch)
    std::uint32_t code = kPullOk;
    if (sd && sd->flags)
      code = wait_flag(&sd->flags[(r.src_chunk / kBatchChunks) >> sd->flag_shift], sd->epoch, p.timeout_ns,
                       &p.work[1]);
    code = __reduce_max_sync(full, code);
    if (code != kPullOk) {
      if (lane == 0) {
        if (code != kPullAborted) {
          atomicCAS(&p.status->code, 0u, code);
          atomicExch(&p.status->bad_chunk, b * kBatchChunks);
        }
        atomicExch(&p.work[1], 1u);
        if (p.dst_flags) st_release_sys(&p.dst_flags[b], p.dst_epoch | kAbort);
      }
      break;
    }
    const bool verify = sd && sd->digests;
    if (verify) expect = __ldcg(&sd->digests[r.src_chunk]);
    refs[lane] = mine;
    std::uint32_t maxlen = mine.len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(full, maxlen, o));
    const int nsteps = static_cast<int>((maxlen + kPiece - 1) / kPiece);
    __syncwarp();

    std::uint64_t digest = 0;
    bool good = false;
    for (int attempt = 0; attempt < 2 && !good; ++attempt) {
      std::uint64_t v1 = kP1 + kP2, v2 = kP2, v3 = 0, v4 = 0 - kP1;
#pragma unroll
      for (int s = 0; s < kStages - 1; ++s) {
        if (s < nsteps) load_step(refs, wbuf + s * kStageBytes, s, lane);
        cp_async_commit();
      }
      for (int s = 0; s < nsteps; ++s) {
        const int pre = s + kStages - 1;
        if (pre < nsteps) load_step(refs, wbuf + (pre % kStages) * kStageBytes, pre, lane);
        cp_async_commit();
        cp_async_wait<kStages - 1>();
        __syncwarp();
        const std::uint8_t* st = wbuf + (s % kStages) * kStageBytes;
        store_step(refs, st, s, lane);
        const std::uint32_t g = static_cast<std::uint32_t>(s) * kPiece;
        if (g < mine.len) {
          const std::uint32_t n = min(static_cast<std::uint32_t>(kPiece), mine.len - g);
          const std::uint8_t* slot = st + lane * kSlot;
          const int stripes = static_cast<int>(n >> 5);
          for (int k = 0; k < stripes; ++k) {
            const uint4 a = *reinterpret_cast<const uint4*>(slot + 32 * k);
            const uint4 bq = *reinterpret_cast<const uint4*>(slot + 32 * k + 16);
            v1 = xround(v1, (std::uint64_t(a.y) << 32) | a.x);
            v2 = xround(v2, (std::uint64_t(a.w) << 32) | a.z);
            v3 = xround(v3, (std::uint64_t(bq.y) << 32) | bq.x);
            v4 = xround(v4, (std::uint64_t(bq.w) << 32) | bq.z);
            if (mine.cast && mine.dst) {
              const uint4 o = cvt16_e4m3(a, bq);
              const std::uint32_t ow[4] = {o.x, o.y, o.z, o.w};
              std::uint8_t* cb = mine.dst + g / 2 + 16 * k;
              for (int bb = 0; bb < 16; ++bb) cb[bb] = static_cast<std::uint8_t>(ow[bb >> 2] >> (8 * (bb & 3)));
            }
          }
          if (mine.cast && mine.dst && (n & 31u))
            cvt_tail_e4m3(slot + (n & ~31u), mine.dst + (g + (n & ~31u)) / 2, static_cast<int>(n & 31u));
          if (g + n == mine.len) {
            std::uint64_t h = mine.len >= 32 ? merge4(v1, v2, v3, v4) : kP5;
            h += mine.len;
            digest = finish_tail(h, slot + (n & ~31u), static_cast<int>(n & 31u));
          }
        }
        __syncwarp();
      }
      cp_async_wait<0>();
      const bool lane_ok = mine.len == 0 || !verify || digest == expect;
      good = __all_sync(full, lane_ok);
      if (!good && lane == 0 && attempt == 0) atomicAdd(&p.status->retried_batches, 1u);
      __syncwarp();
    }
    if (!good) {
      const bool lane_ok = mine.len == 0 || !verify || digest == expect;
      const unsigned bad = __ballot_sync(full, !lane_ok);
      if (lane == 0) {
        atomicCAS(&p.status->code, 0u, static_cast<std::uint32_t>(kPullChecksum));
        atomicExch(&p.status->bad_chunk, b * kBatchChunks + (__ffs(bad) - 1));
        atomicExch(&p.work[1], 1u);
        if (p.dst_flags) st_release_sys(&p.dst_flags[b], p.dst_epoch | kAbort);
      }
      break;
    }
    if (p.dst_digests && mine.len) p.dst_digests[c] = digest;
    __threadfence_system();
    __syncwarp();
    if (lane == 0) {
      if (p.dst_flags) st_release_sys(&p.dst_flags[b], p.dst_epoch);
      atomicAdd(&p.status->batches_done, 1u);
    }
    std::uint64_t landed = mine.len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) landed += __shfl_xor_sync(full, landed, o);
    if (lane == 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(&p.status->bytes),
                static_cast<unsigned long long>(landed));
  }
}

// ---------------------------------------------------------------- K6 -----
// XXH64 is serial within a span: each of the reference's four accumulators
// (digest.cpp:89-95) is a dependent chain of round64, 28 cycles per round on
// B200 (tools/micro/xxh_chain.cu), so a span hashes at most ~2.27 GB/s.  To
// keep the chain itself the only thing on the critical path, a span gets a
// warp pair:
//   feeder warp   lane 0 streams the span through a ring of 16 KiB slots (one
//                 cp.async.bulk per slot); all 32 lanes then replace every
//                 word of a landed slot by its product w * P2 (the part of
//                 round64 that does not depend on the accumulator)
//   chain warp    lanes 0..3 run the four accumulators on the products,
//                 acc = rotl(acc + p, 31) * P1 (carried one add ahead, the
//                 next product folded into the multiply), and free the slot
// The chain lane 0 merges and finalizes; the < 32-byte tail is read from
// global memory.  A span that is not 16-byte aligned is hashed by the chain
// warp straight from global memory.
constexpr int kDigSpans = 4;  // warp pairs per CTA
constexpr int kDigSlot = 16384;
constexpr int kDigSlots = 3;

__global__ void __launch_bounds__(kDigSpans * 64)
    span_digest_kernel(const std::uint64_t* ptrs, const std::uint64_t* lens, std::uint64_t* out,
                       int n) {
  extern __shared__ __align__(1024) std::uint8_t dsm[];
  __shared__ __align__(8) unsigned long long full[kDigSpans][kDigSlots];
  __shared__ __align__(8) unsigned long long ready[kDigSpans][kDigSlots];
  __shared__ __align__(8) unsigned long long empty[kDigSpans][kDigSlots];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int pair = warp >> 1;
  const bool feeder = (warp & 1) != 0;
  const int span = blockIdx.x * kDigSpans + pair;
  if (threadIdx.x == 0) {
    for (int q = 0; q < kDigSpans; ++q)
      for (int k = 0; k < kDigSlots; ++k) {
        mbar_init(&full[q][k], 1);
        mbar_init(&ready[q][k], 1);
        mbar_init(&empty[q][k], 1);
      }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (span >= n) return;
  std::uint8_t* ring = dsm + pair * (kDigSlots * kDigSlot);
  const std::uint8_t* base = reinterpret_cast<const std::uint8_t*>(ptrs[span]);
  const std::uint64_t len = lens[span];
  const std::uint64_t full_stripes = len >> 5;
  const std::uint64_t nslots = (len + kDigSlot - 1) / kDigSlot;
  constexpr int kSlotStripes = kDigSlot / 32;
  const bool aligned = (reinterpret_cast<std::uintptr_t>(base) & 15) == 0;
  if (feeder) {
    if (!aligned) return;
    for (std::uint64_t k = 0; k < nslots; ++k) {
      const int slot = static_cast<int>(k % kDigSlots);
      const auto use = static_cast<unsigned>((k / kDigSlots) & 1);
      if (k >= kDigSlots) mbar_wait(&empty[pair][slot], use ^ 1);  // chain done with it
      std::uint8_t* st = ring + slot * kDigSlot;
      if (lane == 0) {
        const std::uint64_t rem = len - k * kDigSlot;
        const auto bytes = static_cast<unsigned>((rem < kDigSlot ? rem : kDigSlot) & ~15ull);
        fence_proxy_async_smem();  // products written there by the generic proxy
        if (bytes) {
          mbar_arrive_tx(&full[pair][slot], bytes);
          bulk_g2s(st, base + k * kDigSlot, bytes, &full[pair][slot]);
        } else {
          mbar_arrive(&full[pair][slot]);
        }
      }
      mbar_wait(&full[pair][slot], use);
      // every word of the slot's whole stripes -> w * P2, in place
      const std::uint64_t first = k * kSlotStripes;
      const std::uint64_t cnt64 = full_stripes > first ? full_stripes - first : 0;
      const int words = 4 * static_cast<int>(cnt64 < kSlotStripes ? cnt64 : kSlotStripes);
      auto* w = reinterpret_cast<std::uint64_t*>(st);
#pragma unroll 4
      for (int x = lane; x < words; x += 32) w[x] *= kP2;
      __syncwarp();
      if (lane == 0) mbar_arrive(&ready[pair][slot]);
    }
    return;
  }
  // chain warp
  std::uint64_t acc = lane == 0 ? kP1 + kP2 : lane == 1 ? kP2 : lane == 2 ? 0 : 0 - kP1;
  if (aligned) {
    // y = acc + next product (one add ahead: xround_fused folds each product
    // into the previous round's multiply, 25 instead of 28 cycles per round)
    std::uint64_t y = acc;
    bool primed = false;
    for (std::uint64_t k = 0; k < nslots; ++k) {
      const int slot = static_cast<int>(k % kDigSlots);
      mbar_wait(&ready[pair][slot], static_cast<unsigned>((k / kDigSlots) & 1));
      if (lane < 4) {
        const std::uint64_t first = k * kSlotStripes;
        const std::uint64_t c64 = full_stripes > first ? full_stripes - first : 0;
        const int cnt = static_cast<int>(c64 < kSlotStripes ? c64 : kSlotStripes);
        const std::uint8_t* pw = ring + slot * kDigSlot + 8 * lane;
        int r = 0;
        if (!primed && cnt > 0) {
          y += *reinterpret_cast<const std::uint64_t*>(pw);
          primed = true;
          r = 1;
        }
        for (; r + 16 <= cnt; r += 16) {
          std::uint64_t p[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) p[j] = *reinterpret_cast<const std::uint64_t*>(pw + 32 * (r + j));
#pragma unroll
          for (int j = 0; j < 16; ++j) y = xround_fused(y, p[j]);
        }
        for (; r < cnt; ++r) y = xround_fused(y, *reinterpret_cast<const std::uint64_t*>(pw + 32 * r));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[pair][slot]);
    }
    acc = primed ? xround_fused(y, 0) : y;
  } else if (lane < 4) {
    for (std::uint64_t k = 0; k < full_stripes; ++k) {
      std::uint64_t w = 0;
      const std::uint8_t* q = base + 32 * k + 8 * lane;
#pragma unroll
      for (int b = 0; b < 8; ++b) w |= std::uint64_t(q[b]) << (8 * b);
      acc = xround(acc, w);
    }
  }
  const std::uint64_t a = __shfl_sync(0xffffffffu, acc, 0);
  const std::uint64_t b = __shfl_sync(0xffffffffu, acc, 1);
  const std::uint64_t c = __shfl_sync(0xffffffffu, acc, 2);
  const std::uint64_t d = __shfl_sync(0xffffffffu, acc, 3);
  if (lane == 0) {
    std::uint64_t h = len >= 32 ? merge4(a, b, c, d) : kP5;
    h += len;
    const std::uint64_t tail_at = full_stripes * 32;
    out[span] = finish_tail(h, base + tail_at, static_cast<int>(len - tail_at));
  }
}

// Tiles of kCopyTile source bytes over all spans (tile0[i] = first tile of
// span i): a block per tile, so many tiny spans and a few huge ones both
// spread over the whole grid.
constexpr std::uint64_t kCopyTile = 16384;

__global__ void __launch_bounds__(256) copy_spans_kernel(const std::uint64_t* srcs,
                                                         const std::uint64_t* dsts,
                                                         const std::uint64_t* lens,
                                                         const std::uint64_t* tile0, int n,
                                                         std::uint64_t tiles,
                                                         const std::uint32_t* guard) {
  __shared__ int span_s;
  if (guard && *reinterpret_cast<const volatile std::uint32_t*>(guard) != 0) return;
  for (std::uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    if (threadIdx.x == 0) {
      int lo = 0, hi = n;  // last span with tile0 <= t
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (tile0[mid] <= t) lo = mid;
        else hi = mid;
      }
      span_s = lo;
    }
    __syncthreads();
    const int span = span_s;
    __syncthreads();
    const std::uint8_t* src = reinterpret_cast<const std::uint8_t*>(srcs[span]);
    std::uint8_t* dst = reinterpret_cast<std::uint8_t*>(dsts[span]);
    const std::uint64_t raw = lens[span];
    const std::uint64_t len = raw & ~kSpanCastE4M3;
    const std::uint64_t off = (t - tile0[span]) * kCopyTile;
    const std::uint64_t end = off + kCopyTile < len ? off + kCopyTile : len;
    if (raw & kSpanCastE4M3) {  // bf16 in, e4m3 out (half the bytes)
      const bool v8 = ((reinterpret_cast<std::uintptr_t>(src) | off) & 15) == 0 &&
                      (reinterpret_cast<std::uintptr_t>(dst) & 7) == 0;
      std::uint64_t i = off;
      if (v8) {
        for (std::uint64_t k = off + 16 * threadIdx.x; k + 16 <= end; k += 16 * blockDim.x) {
          const uint4 a = *reinterpret_cast<const uint4*>(src + k);
          *reinterpret_cast<uint2*>(dst + k / 2) = make_uint2(cvt4_e4m3(a.x, a.y), cvt4_e4m3(a.z, a.w));
        }
        i = off + (end - off) / 16 * 16;
      }
      for (std::uint64_t k = i + 2 * threadIdx.x; k + 1 < end; k += 2 * blockDim.x) {
        const std::uint32_t w = std::uint32_t(src[k]) | (std::uint32_t(src[k + 1]) << 8);
        dst[k / 2] = static_cast<std::uint8_t>(cvt4_e4m3(w, 0) & 0xFF);
      }
      continue;
    }
    const bool vec =
        ((reinterpret_cast<std::uintptr_t>(src) | reinterpret_cast<std::uintptr_t>(dst) | off) & 15) == 0;
    std::uint64_t i = off;
    if (vec) {
      for (std::uint64_t k = off + 16 * threadIdx.x; k + 16 <= end; k += 16 * blockDim.x)
        *reinterpret_cast<uint4*>(dst + k) = *reinterpret_cast<const uint4*>(src + k);
      i = off + (end - off) / 16 * 16;
    }
    for (std::uint64_t k = i + threadIdx.x; k < end; k += blockDim.x) dst[k] = src[k];
  }
}

// --------------------------------------------------------------- synth ---
__device__ __forceinline__ std::uint64_t splitmix(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ std::uint16_t synth_one(std::uint64_t seed, std::uint64_t i) {
  const std::uint64_t z = splitmix(seed + (i + 1) * 0x9E3779B97F4A7C15ULL);
  const int q = static_cast<int>(z >> 40) - (1 << 23);
  const float f = static_cast<float>(q) * (1.0f / 8388608.0f);
  std::uint32_t u = __float_as_uint(f);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<std::uint16_t>(u >> 16);
}

__global__ void synth_bf16_kernel(std::uint16_t* dst, std::uint64_t n, std::uint64_t seed,
                                  std::uint64_t first) {
  const std::uint64_t stride = std::uint64_t(gridDim.x) * blockDim.x * 8;
  for (std::uint64_t i = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; i < n;
       i += stride) {
    if (i + 8 <= n && (reinterpret_cast<std::uintptr_t>(dst + i) & 15) == 0) {
      std::uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        w[k] = std::uint32_t(synth_one(seed, first + i + 2 * k)) |
               (std::uint32_t(synth_one(seed, first + i + 2 * k + 1)) << 16);
      *reinterpret_cast<uint4*>(dst + i) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      for (std::uint64_t k = i; k < n && k < i + 8; ++k) dst[k] = synth_one(seed, first + k);
    }
  }
}

// ------------------------------------------------------------------ K5 ---
__device__ __forceinline__ std::uint8_t bf16_to_e4m3(std::uint16_t x) {
  const float f = __uint_as_float(std::uint32_t(x) << 16);
  std::uint16_t r;
  // cvt.rn.satfinite.e4m3x2.f32 d, a, b packs a -> high byte, b -> low byte.
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;\n" : "=h"(r) : "f"(0.0f), "f"(f));
  return static_cast<std::uint8_t>(r & 0xFF);
}

__global__ void e4m3_kernel(const std::uint16_t* src, std::uint8_t* dst, std::uint64_t n) {
  const std::uint64_t stride = std::uint64_t(gridDim.x) * blockDim.x;
  for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = bf16_to_e4m3(src[i]);
}

bool use_ldg_kernel() {
  static const bool v = [] {
    const char* e = std::getenv("RSB_PULL_KERNEL");
    return e && std::strcmp(e, "ldg") == 0;
  }();
  return v;
}

}  // namespace

// ------------------------------------------------------------ launchers --

int pull_grid(int device) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return sms;
}

const char* pull_kernel_name() { return use_ldg_kernel() ? "pull_kernel" : "pull_tma_kernel"; }

cudaError_t launch_pull(const PullParams& p, int sms, cudaStream_t s) {
  if (p.order ? p.n_sched == 0 : p.n_batches <= p.first_batch) return cudaSuccess;
  if (!use_ldg_kernel()) return launch_pull_tma(p, sms, s);
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(pull_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  const std::uint32_t todo = p.order ? p.n_sched : p.n_batches - p.first_batch;
  const std::uint32_t need = (todo + kWarps - 1) / kWarps;
  int grid = 2 * sms;
  if (static_cast<std::uint32_t>(grid) > need) grid = static_cast<int>(need);
  pull_kernel<<<grid, kThreads, kSmemBytes, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_span_digests(const std::uint64_t* ptrs, const std::uint64_t* lens,
                                std::uint64_t* out, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  constexpr int smem = kDigSpans * kDigSlots * kDigSlot;
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_done[dev]) {
    cudaError_t e =
        cudaFuncSetAttribute(span_digest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_done[dev] = true;
  }
  span_digest_kernel<<<(n + kDigSpans - 1) / kDigSpans, kDigSpans * 64, smem, s>>>(ptrs, lens,
                                                                                   out, n);
  return cudaGetLastError();
}

cudaError_t launch_copy_spans(const std::uint64_t* srcs, const std::uint64_t* dsts,
                              const std::uint64_t* lens, const std::uint64_t* tile0, int n,
                              std::uint64_t tiles, cudaStream_t s, const std::uint32_t* guard) {
  if (n <= 0 || tiles == 0) return cudaSuccess;
  int dev = 0;
  cudaGetDevice(&dev);
  const std::uint64_t cap = static_cast<std::uint64_t>(pull_grid(dev)) * 8;
  const auto grid = static_cast<unsigned>(tiles < cap ? tiles : cap);
  copy_spans_kernel<<<grid, 256, 0, s>>>(srcs, dsts, lens, tile0, n, tiles, guard);
  return cudaGetLastError();
}

std::uint64_t copy_span_tiles(std::uint64_t len) {
  len &= ~kSpanCastE4M3;
  return (len + kCopyTile - 1) / kCopyTile;
}

cudaError_t launch_synth_bf16(std::uint16_t* dst, std::uint64_t n, std::uint64_t seed,
                              std::uint64_t first, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  std::uint64_t blocks = (n / 8 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks == 0) blocks = 1;
  synth_bf16_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(dst, n, seed, first);
  return cudaGetLastError();
}

cudaError_t launch_bf16_to_e4m3(const std::uint16_t* src, std::uint8_t* dst, std::uint64_t n,
                                cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  std::uint64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  e4m3_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(src, dst, n);
  return cudaGetLastError();
}

}  // namespace rsb::dev
