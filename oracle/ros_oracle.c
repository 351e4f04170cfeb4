/* TEST INFRASTRUCTURE ONLY -- CPU oracle for the ROS read path.
 * See ros_oracle.h for what each function restates and how it is pinned.
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline) load this.
 */
#include "ros_oracle.h"

#include <math.h>
#include <string.h>

/* ---------------------------------------------------------------- XXH64 --
 * Restates /root/reference/proj/src/digest.cpp:13-106 (constants 13-17,
 * round64 30-35, merge_round 37-42, avalanche 44-51, finalize 54-75,
 * digest64 79-106).  Little-endian loads, as the reference asserts. */
#define P1 0x9E3779B185EBCA87ULL
#define P2 0xC2B2AE3D27D4EB4FULL
#define P3 0x165667B19E3779F9ULL
#define P4 0x85EBCA77C2B2AE63ULL
#define P5 0x27D4EB2F165667C5ULL

static inline uint64_t rotl(uint64_t x, unsigned r) { return (x << r) | (x >> (64 - r)); }
static inline uint64_t ld64(const uint8_t* p) { uint64_t v; memcpy(&v, p, 8); return v; }
static inline uint32_t ld32(const uint8_t* p) { uint32_t v; memcpy(&v, p, 4); return v; }
static inline uint64_t lane_step(uint64_t acc, uint64_t w) { return rotl(acc + w * P2, 31) * P1; }

uint64_t ro_xxh64(const void* data, size_t len) {
  const uint8_t* p = (const uint8_t*)data;
  size_t left = len;
  uint64_t h;
  if (len >= 32) {
    uint64_t a = P1 + P2, b = P2, c = 0, d = (uint64_t)0 - P1;
    while (left >= 32) {
      a = lane_step(a, ld64(p));
      b = lane_step(b, ld64(p + 8));
      c = lane_step(c, ld64(p + 16));
      d = lane_step(d, ld64(p + 24));
      p += 32;
      left -= 32;
    }
    h = rotl(a, 1) + rotl(b, 7) + rotl(c, 12) + rotl(d, 18);
    const uint64_t lanes[4] = {a, b, c, d};
    for (int i = 0; i < 4; ++i) h = (h ^ lane_step(0, lanes[i])) * P1 + P4;
  } else {
    h = P5;
  }
  h += (uint64_t)len;
  for (; left >= 8; left -= 8, p += 8) h = rotl(h ^ lane_step(0, ld64(p)), 27) * P1 + P4;
  if (left >= 4) {
    h = rotl(h ^ ((uint64_t)ld32(p) * P1), 23) * P2 + P3;
    p += 4;
    left -= 4;
  }
  for (; left > 0; --left, ++p) h = rotl(h ^ ((uint64_t)(*p) * P5), 11) * P1;
  h ^= h >> 33;
  h *= P2;
  h ^= h >> 29;
  h *= P3;
  h ^= h >> 32;
  return h;
}

/* ------------------------------------------------------- byte generators */
static inline uint64_t splitmix_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

void ro_splitmix_bytes(uint64_t seed, size_t n, uint8_t* out) {
  uint64_t x = seed;
  for (size_t i = 0; i < n; ++i) {
    x += 0x9E3779B97F4A7C15ULL;
    out[i] = (uint8_t)(splitmix_mix(x) & 0xFF);
  }
}

void ro_pattern_bytes(size_t n, uint8_t* out) {
  for (size_t i = 0; i < n; ++i) out[i] = (uint8_t)((i * 17 + 3) & 0xFF);
}

void ro_fill_pattern(uint64_t salt, size_t n, uint8_t* out) {
  for (size_t i = 0; i < n; ++i) out[i] = (uint8_t)((salt * 1315423911u + i * 131u) & 0xFF);
}

static inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

void ro_synth_bf16(uint64_t seed, uint64_t first_elem, size_t n, uint16_t* out) {
  for (size_t k = 0; k < n; ++k) {
    uint64_t i = first_elem + k;
    uint64_t z = splitmix_mix(seed + (i + 1) * 0x9E3779B97F4A7C15ULL);
    int32_t q = (int32_t)(z >> 40) - (1 << 23); /* [-2^23, 2^23) */
    float f = (float)q * (1.0f / 8388608.0f);   /* exact: [-1, 1) */
    out[k] = f32_to_bf16_rne(f);
  }
}

/* ------------------------------------------------------- chunk digests --- */
size_t ro_chunk_digests(const uint8_t* const* items, const uint64_t* lens,
                        size_t n_items, uint64_t chunk, uint64_t* out) {
  size_t k = 0;
  for (size_t i = 0; i < n_items; ++i) {
    for (uint64_t off = 0; off < lens[i]; off += chunk) {
      uint64_t take = lens[i] - off < chunk ? lens[i] - off : chunk;
      if (out) out[k] = ro_xxh64(items[i] + off, (size_t)take);
      ++k;
    }
  }
  return k;
}

/* ------------------------------------------------------------ manifest --
 * Packing rule restated from manifest.cpp:179-202. */
int ro_assemble(size_t n, const uint64_t* lens, uint64_t tiny, uint64_t target,
                int32_t* group_of, uint64_t* offset) {
  int groups = 0;
  int open = 0; /* the open group has members */
  uint64_t packed = 0;
  for (size_t e = 0; e < n; ++e) {
    group_of[e] = -1;
    offset[e] = 0;
    if (lens[e] >= tiny) continue;
    if (open && packed + lens[e] > target) {
      ++groups;
      open = 0;
      packed = 0;
    }
    group_of[e] = groups;
    offset[e] = packed;
    packed += lens[e];
    open = 1;
  }
  return groups + (open ? 1 : 0);
}

/* Tagged big-endian field encoding (codec.cpp:28-60): tag u8, wire type u8
 * (1 = u64, 2 = bytes, 3 = list), then the payload. */
typedef struct {
  uint8_t* p;
  size_t n;
} Buf;

static void put_raw(Buf* b, const void* src, size_t len) {
  if (b->p) memcpy(b->p + b->n, src, len);
  b->n += len;
}
static void put_be32(Buf* b, uint32_t v) {
  uint8_t t[4] = {(uint8_t)(v >> 24), (uint8_t)(v >> 16), (uint8_t)(v >> 8), (uint8_t)v};
  put_raw(b, t, 4);
}
static void put_be64(Buf* b, uint64_t v) {
  put_be32(b, (uint32_t)(v >> 32));
  put_be32(b, (uint32_t)v);
}
static void put_hdr(Buf* b, uint8_t tag, uint8_t wt) {
  uint8_t t[2] = {tag, wt};
  put_raw(b, t, 2);
}
static void field_u64(Buf* b, uint8_t tag, uint64_t v) {
  put_hdr(b, tag, 1);
  put_be64(b, v);
}

size_t ro_manifest_encode(size_t n, const char* const* names,
                          const uint64_t* lens, const uint64_t* digests,
                          const int32_t* group_of, const uint64_t* offset,
                          int n_groups, const uint64_t* group_digests,
                          uint8_t* out) {
  Buf b = {out, 0};
  field_u64(&b, 1, 1); /* format version (manifest.cpp:105) */
  field_u64(&b, 2, 1); /* kDigestAlgXxh64 (digest.hpp:13)  */
  /* field 3: list of entry blobs {1: name, 2: length, 3: digest} */
  put_hdr(&b, 3, 3);
  put_be32(&b, (uint32_t)n);
  for (size_t e = 0; e < n; ++e) {
    size_t nl = strlen(names[e]);
    put_be32(&b, (uint32_t)(2 + 4 + nl + 2 * 10));
    put_hdr(&b, 1, 2);
    put_be32(&b, (uint32_t)nl);
    put_raw(&b, names[e], nl);
    field_u64(&b, 2, lens[e]);
    field_u64(&b, 3, digests[e]);
  }
  /* field 4: list of group blobs {1: packed_length, 2: digest,
   * 3: bytes = members as (u32 entry, u64 offset) big-endian} */
  put_hdr(&b, 4, 3);
  put_be32(&b, (uint32_t)n_groups);
  for (int g = 0; g < n_groups; ++g) {
    uint64_t packed = 0;
    size_t members = 0;
    for (size_t e = 0; e < n; ++e)
      if (group_of[e] == g) {
        packed += lens[e];
        ++members;
      }
    put_be32(&b, (uint32_t)(2 * 10 + 2 + 4 + 12 * members));
    field_u64(&b, 1, packed);
    field_u64(&b, 2, group_digests[g]);
    put_hdr(&b, 3, 2);
    put_be32(&b, (uint32_t)(12 * members));
    for (size_t e = 0; e < n; ++e)
      if (group_of[e] == g) {
        put_be32(&b, (uint32_t)e);
        put_be64(&b, offset[e]);
      }
  }
  return b.n;
}

/* ------------------------------------------------------ reshard chunks -- */
static uint64_t gcd64(uint64_t a, uint64_t b) {
  while (b) {
    uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

uint32_t ro_chunk_len_for(uint64_t row_bytes, uint64_t nc, uint64_t chunk_bytes, uint32_t align) {
  if (row_bytes == 0 || align == 0 || row_bytes % align || nc == 0) return (uint32_t)chunk_bytes;
  uint64_t g = gcd64(nc, row_bytes / align);
  uint64_t start = (chunk_bytes < g ? chunk_bytes : g) / 128 * 128;
  for (uint64_t c = start; c >= 128; c -= 128)
    if (g % c == 0) return (uint32_t)c;
  return (uint32_t)chunk_bytes;
}

/* -------------------------------------------------------- bf16 -> e4m3 -- */
void ro_bf16_to_e4m3(const uint16_t* in, size_t n, uint8_t* out) {
  for (size_t i = 0; i < n; ++i) {
    uint32_t u = (uint32_t)in[i] << 16;
    float f;
    memcpy(&f, &u, 4);
    uint8_t sign = (uint8_t)((u >> 24) & 0x80);
    if (isnan(f)) {
      out[i] = 0x7F;
      continue;
    }
    double a = fabs((double)f);
    uint8_t code;
    if (a > 448.0) {
      code = 0x7E; /* satfinite: max finite 1.75 * 2^8 */
    } else if (a < 0.015625) { /* below 2^-6: subnormal grid of 2^-9 */
      double q = nearbyint(a * 512.0);
      code = (uint8_t)q; /* q == 8 encodes the min normal */
    } else {
      int e;
      double m = frexp(a, &e); /* a = m * 2^e, m in [0.5, 1) */
      e -= 1;                  /* a = (2m) * 2^e, 2m in [1, 2) */
      double q = nearbyint((2.0 * m - 1.0) * 8.0);
      if (q >= 8.0) {
        q = 0.0;
        e += 1;
      }
      code = (uint8_t)(((e + 7) << 3) | (int)q);
      if (code > 0x7E) code = 0x7E;
    }
    out[i] = (uint8_t)(sign | code);
  }
}
