// Device helpers shared by the sm_100a kernels: XXH64 pieces (reference
// digest.cpp:13-75 restated for the device), PTX wrappers for cp.async,
// TMA bulk copies, mbarriers and system-scope acquire/release.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "device.hpp"

namespace rsb::dev::detail {

constexpr std::uint64_t kP1 = 0x9E3779B185EBCA87ULL;
constexpr std::uint64_t kP2 = 0xC2B2AE3D27D4EB4FULL;
constexpr std::uint64_t kP3 = 0x165667B19E3779F9ULL;
constexpr std::uint64_t kP4 = 0x85EBCA77C2B2AE63ULL;
constexpr std::uint64_t kP5 = 0x27D4EB2F165667C5ULL;

__device__ __forceinline__ std::uint64_t rotl64(std::uint64_t x, int r) {
  return (x << r) | (x >> (64 - r));
}
// One accumulator step of the 32-byte stripe loop (round64):
//   acc = rotl64(acc + w * P2, 31) * P1.
// Written on 32-bit halves so the serial chain through `acc` is five
// dependent instructions: the 64-bit add (lo, hi+carry), the rotation as two
// independent funnel shifts, and the product as one wide multiply plus two
// cross products folded by a 3-input add.  (w * P2 does not depend on acc.)
__device__ __forceinline__ std::uint64_t xround_pre(std::uint64_t acc, std::uint64_t wp2) {
  const std::uint64_t t = acc + wp2;  // wp2 = w * P2
  const std::uint32_t lo = static_cast<std::uint32_t>(t), hi = static_cast<std::uint32_t>(t >> 32);
  const std::uint32_t rlo = __funnelshift_l(hi, lo, 31);  // (lo << 31) | (hi >> 1)
  const std::uint32_t rhi = __funnelshift_l(lo, hi, 31);  // (hi << 31) | (lo >> 1)
  constexpr std::uint32_t p1lo = static_cast<std::uint32_t>(kP1);
  constexpr std::uint32_t p1hi = static_cast<std::uint32_t>(kP1 >> 32);
  const std::uint64_t wl = static_cast<std::uint64_t>(rlo) * p1lo;
  const std::uint32_t h = static_cast<std::uint32_t>(wl >> 32) + rhi * p1lo + rlo * p1hi;
  return (static_cast<std::uint64_t>(h) << 32) | static_cast<std::uint32_t>(wl);
}
__device__ __forceinline__ std::uint64_t xround(std::uint64_t acc, std::uint64_t w) {
  return xround_pre(acc, w * kP2);
}
// The chain carried one add ahead: y = acc + p holds the next round's
// rotation input, and the following product is added inside the multiply
// (wide multiply-add with a 64-bit addend), so the serial chain per round is
// the rotation, one wide IMAD and one 3-input add:
//   returns rotl64(y, 31) * P1 + p_next   (= the next y; p_next = 0 at the end: acc)
__device__ __forceinline__ std::uint64_t xround_fused(std::uint64_t y, std::uint64_t p_next) {
  const std::uint32_t lo = static_cast<std::uint32_t>(y), hi = static_cast<std::uint32_t>(y >> 32);
  const std::uint32_t rlo = __funnelshift_l(hi, lo, 31);
  const std::uint32_t rhi = __funnelshift_l(lo, hi, 31);
  constexpr std::uint32_t p1lo = static_cast<std::uint32_t>(kP1);
  constexpr std::uint32_t p1hi = static_cast<std::uint32_t>(kP1 >> 32);
  const std::uint64_t wl = static_cast<std::uint64_t>(rlo) * p1lo + p_next;
  const std::uint32_t h = static_cast<std::uint32_t>(wl >> 32) + rhi * p1lo + rlo * p1hi;
  return (static_cast<std::uint64_t>(h) << 32) | static_cast<std::uint32_t>(wl);
}
__device__ __forceinline__ std::uint64_t avalanche(std::uint64_t h) {
  h ^= h >> 33;
  h *= kP2;
  h ^= h >> 29;
  h *= kP3;
  h ^= h >> 32;
  return h;
}
// Fold of the four accumulators (merge_round x4).
__device__ __forceinline__ std::uint64_t merge4(std::uint64_t a, std::uint64_t b,
                                                std::uint64_t c, std::uint64_t d) {
  std::uint64_t h = rotl64(a, 1) + rotl64(b, 7) + rotl64(c, 12) + rotl64(d, 18);
  h = (h ^ xround(0, a)) * kP1 + kP4;
  h = (h ^ xround(0, b)) * kP1 + kP4;
  h = (h ^ xround(0, c)) * kP1 + kP4;
  h = (h ^ xround(0, d)) * kP1 + kP4;
  return h;
}
// Tail (< 32 bytes), then avalanche (finalize).
static __device__ __noinline__ std::uint64_t finish_tail(std::uint64_t h, const std::uint8_t* p, int n) {
  while (n >= 8) {
    std::uint64_t w = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) w |= std::uint64_t(p[k]) << (8 * k);
    h ^= xround(0, w);
    h = rotl64(h, 27) * kP1 + kP4;
    p += 8;
    n -= 8;
  }
  if (n >= 4) {
    std::uint32_t w = std::uint32_t(p[0]) | (std::uint32_t(p[1]) << 8) |
                      (std::uint32_t(p[2]) << 16) | (std::uint32_t(p[3]) << 24);
    h ^= std::uint64_t(w) * kP1;
    h = rotl64(h, 23) * kP2 + kP3;
    p += 4;
    n -= 4;
  }
  while (n > 0) {
    h ^= std::uint64_t(*p) * kP5;
    h = rotl64(h, 11) * kP1;
    ++p;
    --n;
  }
  return avalanche(h);
}

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ std::uint32_t ld_acquire_sys(const std::uint32_t* p) {
  std::uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(std::uint32_t* p, std::uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// One release fence for several flag stores (fence + relaxed store = release).
// fence.release (no acquire half) skips the L1 invalidation (CCTL.IVALL)
// that fence.acq_rel.sys carries.
__device__ __forceinline__ void fence_release_sys() {
  asm volatile("fence.release.sys;\n" ::: "memory");
}
__device__ __forceinline__ void st_relaxed_sys(std::uint32_t* p, std::uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ std::uint64_t globaltimer() {
  std::uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
  return t;
}
__device__ __forceinline__ std::uint32_t ld_volatile(const std::uint32_t* p) {
  return *reinterpret_cast<const volatile std::uint32_t*>(p);
}

#ifndef RSB_MAX_POLL_NS
#define RSB_MAX_POLL_NS 1024
#endif
constexpr unsigned kMaxPollNs = RSB_MAX_POLL_NS;  // back-off ceiling of a watermark poll

// Waits until the upstream watermark of a batch reaches `epoch`.
static __device__ __noinline__ std::uint32_t wait_flag(const std::uint32_t* flag, std::uint32_t epoch,
                                                std::uint64_t timeout_ns,
                                                const std::uint32_t* abort) {
  std::uint64_t t0 = 0;
  unsigned ns = 32;
  for (;;) {
    std::uint32_t v = ld_acquire_sys(flag);
    if (v == epoch) return kPullOk;
    if (v > epoch) return kPullNotServing;  // newer fill or abort bit
    if (ld_volatile(abort)) return kPullAborted;
    std::uint64_t now = globaltimer();
    if (t0 == 0) t0 = now;
    if (now - t0 > timeout_ns) return kPullTimeout;
    __nanosleep(ns);
    if (ns < kMaxPollNs) ns <<= 1;
  }
}

// ---- mbarrier / TMA bulk ---------------------------------------------------
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)),
               "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];\n" ::"r"(smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gmem),
               "r"(smem_u32(smem)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// Four bf16 (two words, little-endian order) -> four e4m3 bytes (RNE,
// satfinite), element 0 in the low byte.
__device__ __forceinline__ std::uint32_t cvt4_e4m3(std::uint32_t a, std::uint32_t b) {
  const float f0 = __uint_as_float(a << 16), f1 = __uint_as_float(a & 0xffff0000u);
  const float f2 = __uint_as_float(b << 16), f3 = __uint_as_float(b & 0xffff0000u);
  std::uint16_t lo, hi;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;\n" : "=h"(lo) : "f"(f1), "f"(f0));
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;\n" : "=h"(hi) : "f"(f3), "f"(f2));
  return std::uint32_t(lo) | (std::uint32_t(hi) << 16);
}
// 16 bf16 (one 32-byte stripe) -> 16 e4m3 bytes.
__device__ __forceinline__ uint4 cvt16_e4m3(const uint4& a, const uint4& b) {
  return make_uint4(cvt4_e4m3(a.x, a.y), cvt4_e4m3(a.z, a.w), cvt4_e4m3(b.x, b.y),
                    cvt4_e4m3(b.z, b.w));
}
// Tail bf16 elements (n bytes, even) -> e4m3 bytes.
__device__ __forceinline__ void cvt_tail_e4m3(const std::uint8_t* src, std::uint8_t* dst, int n) {
  for (int i = 0; i + 1 < n; i += 2) {
    const std::uint32_t w = std::uint32_t(src[i]) | (std::uint32_t(src[i + 1]) << 8);
    dst[i / 2] = static_cast<std::uint8_t>(cvt4_e4m3(w, 0) & 0xFF);
  }
}

// XXH64 of one chunk straight from (possibly peer) global memory, optionally
// storing it to dst (as e4m3 when cast): the quiet same-source retry after a
// mismatch (client_core.cpp:336-357).  Rare path.
static __device__ __noinline__ std::uint64_t repull_chunk(const std::uint8_t* src, std::uint8_t* dst,
                                                   std::uint32_t len, bool cast = false) {
  std::uint64_t v1 = kP1 + kP2, v2 = kP2, v3 = 0, v4 = 0 - kP1;
  std::uint32_t i = 0;
  std::uint8_t tail[32];
  for (; i + 32 <= len; i += 32) {
    std::uint64_t w[4];
    for (int k = 0; k < 4; ++k) {
      std::uint64_t x = 0;
      for (int b = 0; b < 8; ++b) x |= std::uint64_t(__ldcg(src + i + 8 * k + b)) << (8 * b);
      w[k] = x;
    }
    v1 = xround(v1, w[0]);
    v2 = xround(v2, w[1]);
    v3 = xround(v3, w[2]);
    v4 = xround(v4, w[3]);
    if (dst && cast) {
      const uint4 a = make_uint4(static_cast<std::uint32_t>(w[0]), static_cast<std::uint32_t>(w[0] >> 32),
                                 static_cast<std::uint32_t>(w[1]), static_cast<std::uint32_t>(w[1] >> 32));
      const uint4 q = make_uint4(static_cast<std::uint32_t>(w[2]), static_cast<std::uint32_t>(w[2] >> 32),
                                 static_cast<std::uint32_t>(w[3]), static_cast<std::uint32_t>(w[3] >> 32));
      const uint4 o = cvt16_e4m3(a, q);
      const std::uint32_t ow[4] = {o.x, o.y, o.z, o.w};
      for (int b = 0; b < 16; ++b) dst[i / 2 + b] = static_cast<std::uint8_t>(ow[b >> 2] >> (8 * (b & 3)));
    } else if (dst) {
      for (int b = 0; b < 32; ++b) dst[i + b] = static_cast<std::uint8_t>(w[b >> 3] >> (8 * (b & 7)));
    }
  }
  const int t = static_cast<int>(len - i);
  for (int b = 0; b < t; ++b) {
    tail[b] = __ldcg(src + i + b);
    if (dst && !cast) dst[i + b] = tail[b];
  }
  if (dst && cast) cvt_tail_e4m3(tail, dst + i / 2, t);
  std::uint64_t h = len >= 32 ? merge4(v1, v2, v3, v4) : kP5;
  h += len;
  return finish_tail(h, tail, t);
}

// Landing chunk k of a segment: its source/landing addresses, length and
// source chunk index (see ItemDesc).  clen == 0: a hole between segments.
struct ChunkRef {
  const std::uint8_t* src;
  std::uint8_t* dst;
  std::uint32_t clen;
  std::uint32_t src_chunk;
};
__device__ __forceinline__ ChunkRef chunk_ref(const ItemDesc& d, std::uint32_t k) {
  const std::uint32_t c = d.chunk_len & kChunkLenMask;
  const std::uint64_t doff = std::uint64_t(k) * c;
  const std::uint64_t land = (d.chunk_len & kCastE4M3) ? doff / 2 : doff;
  ChunkRef r{nullptr, nullptr, 0u, 0u};
  if (doff >= d.len) return r;
  std::uint64_t soff;
  if (d.q == d.m) {
    soff = doff;
    r.src_chunk = d.src_chunk0 + k;
  } else {
    const std::uint32_t t = k / d.q, j = k - t * d.q;
    const std::uint32_t sc = t * d.m + j;
    soff = std::uint64_t(sc) * c;
    r.src_chunk = d.src_chunk0 + sc;
  }
  r.src = reinterpret_cast<const std::uint8_t*>(d.src) + soff;
  r.dst = d.dst ? reinterpret_cast<std::uint8_t*>(d.dst) + land : nullptr;
  const std::uint64_t rem = d.len - doff;
  r.clen = static_cast<std::uint32_t>(rem < c ? rem : c);
  return r;
}

// Last segment whose first chunk is <= c (segments sorted by chunk0),
// starting from the batch's first candidate (PullParams.batch_seg): O(1)
// for identity pulls, a short forward scan when segments share a batch.
__device__ __forceinline__ std::uint32_t seg_of(const ItemDesc* items, std::uint32_t n,
                                                std::uint32_t first, std::uint32_t c) {
  std::uint32_t s = first;
  while (s + 1 < n && items[s + 1].chunk0 <= c) ++s;
  return s;
}

}  // namespace rsb::dev::detail
