/* TEST INFRASTRUCTURE ONLY.  Plain-C restatement of the reference ROS read
 * path's byte/integer arithmetic, used as the CPU oracle by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.  Never
 * linked into or called by the product library (paper_2604_09107_b200/).
 *
 * Parity pinning: ro_xxh64 is pinned by the reference's frozen vectors
 * (tests/unit/test_digest.cpp:42-69, re-hosted in tests/golden/) and by the
 * reference library itself (oracle/_ref).  The packing rule and manifest
 * encoding are pinned against the reference's own outputs (oracle/_ref).
 * The chunk-digest partition, the TP reshard maps and the bf16->fp8 cast have
 * no counterpart in the reference: they are defined HERE
 * ("parity unpinned" beyond the digest function they use).
 */
#ifndef ROS_ORACLE_H
#define ROS_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* XXH64, seed 0 (digest.cpp:79-106). */
uint64_t ro_xxh64(const void* data, size_t len);

/* Deterministic byte streams of the reference tests. */
void ro_splitmix_bytes(uint64_t seed, size_t n, uint8_t* out); /* test_digest.cpp:13-26 */
void ro_pattern_bytes(size_t n, uint8_t* out);                 /* test_digest.cpp:28-33 */
void ro_fill_pattern(uint64_t salt, size_t n, uint8_t* out);   /* test_client_core.cpp:76-81 */

/* Synthetic bf16 weights: element i of a tensor with seed s is
 * splitmix64 step i+1 from s, top 24 bits -> uniform [-1,1) f32 -> RNE bf16. */
void ro_synth_bf16(uint64_t seed, uint64_t first_elem, size_t n, uint16_t* out);

/* Per-chunk digest table (NEW, not in the reference): every item is cut into
 * ceil(len/chunk) chunks, item-relative; chunk j of item i covers
 * [j*chunk, min((j+1)*chunk, len)).  Digest = ro_xxh64 of those bytes.
 * Writes sum_i ceil(len_i/chunk) digests in item order; returns that count. */
size_t ro_chunk_digests(const uint8_t* const* items, const uint64_t* lens,
                        size_t n_items, uint64_t chunk, uint64_t* out);

/* Manifest packing rule (manifest.cpp:179-202): entry e with len < tiny goes
 * into the open group; the group closes when packed+len > target.
 * group_of[e] = group index or -1; offset[e] = offset inside its group.
 * Returns the number of groups. */
int ro_assemble(size_t n, const uint64_t* lens, uint64_t tiny, uint64_t target,
                int32_t* group_of, uint64_t* offset);

/* Canonical manifest bytes (manifest.cpp:103-139 + codec.cpp:28-60).
 * groups given by group_of/offset from ro_assemble plus group digests.
 * Returns bytes written (or needed when out==NULL). */
size_t ro_manifest_encode(size_t n, const char* const* names,
                          const uint64_t* lens, const uint64_t* digests,
                          const int32_t* group_of, const uint64_t* offset,
                          int n_groups, const uint64_t* group_digests,
                          uint8_t* out);

/* Reshard chunk rule (NEW, pinned here): for a region holding nc bytes of
 * every row of a logical tensor with row_bytes bytes per row, the chunk
 * length is the largest multiple of 128 that is <= chunk_bytes and divides
 * gcd(nc, row_bytes / align); chunk_bytes when row_bytes % align != 0 or no
 * such multiple exists, or the region has no geometry (row_bytes == 0). */
uint32_t ro_chunk_len_for(uint64_t row_bytes, uint64_t nc, uint64_t chunk_bytes, uint32_t align);

/* bf16 -> fp8 e4m3fn, round-to-nearest-even, saturating to +-448, NaN ->
 * 0x7F (NEW: the reference has no cast; this is the pinned definition). */
void ro_bf16_to_e4m3(const uint16_t* in, size_t n, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
