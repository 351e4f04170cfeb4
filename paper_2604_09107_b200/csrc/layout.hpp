// Tensor geometry, chunk layouts and the TP/FSDP reshard planner (K4).
//
// NEW relative to the reference, which requires readers and sources to have
// equal shard counts (server_core.cpp:816-819) and identical entry names and
// lengths (client_core.cpp:1601-1608): here every registered region may carry
// a 2-D geometry -- the logical tensor [rows x row_bytes] and the slice the
// region holds -- and a reader whose slicing differs from its source's pulls
// exactly its slice, gathered from every source shard that holds part of it.
//
// Chunk rule (pinned here; the oracle restates it): a big item with geometry
// (row_bytes W, slice width nc) is cut into chunks of
//     c = the largest multiple of 128 <= chunk_bytes that divides
//         gcd(nc, W / align)                           (align = 2 by default)
// so every TP <= align split along either dimension is a union of whole
// chunks on both sides (no over-read to verify).  Items without geometry and
// geometries the rule cannot serve use chunk_bytes.
//
// Member rule (packed groups): a group with a member that carries a geometry
// is cut member by member -- each member starts a run of chunks of its own
// length (the chunk rule on its geometry, else chunk_bytes), so a region that
// is a whole member, or a chunk-aligned slice of one, maps chunk-for-chunk
// onto the group (an FSDP k/v slice packed by the reference's tiny rule
// lands straight into a TP reader's region, verified).  Its layout records
// chunk length 0; plain groups keep one run of chunk_bytes.
#pragma once

#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

#include "common.hpp"
#include "device.hpp"
#include "manifest.hpp"

namespace rsb {

struct Geometry {
  std::uint64_t rows = 0;       // logical tensor rows (0: no geometry)
  std::uint64_t row_bytes = 0;  // logical tensor row bytes
  std::uint64_t r0 = 0, nr = 0;  // slice rows
  std::uint64_t c0 = 0, nc = 0;  // slice byte columns
  bool has() const { return rows != 0; }
  bool operator==(const Geometry&) const = default;
};

std::uint32_t chunk_len_for(const Geometry& g, std::uint64_t chunk_bytes, std::uint32_t align);

// A run of equal chunks inside an item (a member of a member-cut group).
struct ChunkPart {
  std::uint64_t off = 0;        // bytes into the item
  std::uint64_t len = 0;
  std::uint32_t chunk_len = 0;
  std::uint32_t first = 0;      // its first chunk, relative to the item's chunk0
};

// Per shard of a published (or derived) layout: geometry per manifest entry
// and the chunk length per transfer item.
struct ShardLayout {
  std::vector<Geometry> geo;             // per manifest entry
  std::vector<std::uint32_t> chunk_len;  // per manifest item
  std::string encode() const;
  static Result<ShardLayout> decode(std::string_view s);
};

// Chunk lengths of a shard's items from its entries' geometries (0: a
// member-cut group).
std::vector<std::uint32_t> item_chunk_lens(const Manifest& m, const std::vector<Geometry>& geo,
                                           std::uint64_t chunk_bytes, std::uint32_t align);
// Per entry: the chunk length of its run inside a member-cut group.
std::vector<std::uint32_t> member_chunk_lens(const Manifest& m, const std::vector<Geometry>& geo,
                                             std::uint64_t chunk_bytes, std::uint32_t align);

// One source shard as the reshard planner sees it.
struct SourceShard {
  Manifest manifest;
  ShardLayout layout;
  std::vector<std::uint64_t> item_ptrs;  // reader-VA address per item (0: not mapped yet)
  std::vector<std::uint32_t> chunk0;     // source chunk index per item (batch aligned)
  std::vector<std::vector<ChunkPart>> parts;  // per item: its runs when member-cut
};

// A reader entry the segments cannot serve directly (it lives in a source
// group, or its slice is not chunk-aligned): gathered via a whole source item.
struct GatherNeed {
  std::uint32_t src_shard = 0;
  std::uint32_t src_item = 0;
};
struct SliceCopy {  // rows x nc bytes from a gathered source item into a region
  std::uint32_t src_shard = 0, src_item = 0;
  std::uint64_t src_off = 0, src_stride = 0;
  std::uint64_t dst = 0, dst_stride = 0;
  std::uint64_t rows = 0, nc = 0;
  bool cast = false;  // region lands as e4m3: dst/dst_stride in e4m3 bytes, nc in bf16 bytes
};

struct ReshardPlan {
  std::vector<dev::ItemDesc> segs;  // src addresses filled from SourceShard.item_ptrs
  std::vector<GatherNeed> gathers;  // whole source items to land in staging
  std::vector<SliceCopy> copies;    // staging -> reader regions
  std::vector<std::uint32_t> rehash;  // reader big items (partly) filled by copies
  // reader groups landed straight into their staging by the fill (every
  // member direct): unpacked to the regions, not re-digested
  std::vector<std::uint32_t> direct_groups;
};

// Reader entry e (name, region address, geometry, own item index + chunk0 +
// chunk_len) for every reader entry.
struct ReaderEntry {
  std::string name;
  std::uint64_t ptr = 0;
  std::uint64_t len = 0;
  Geometry geo;
  bool cast = false;            // lands as e4m3 (ptr holds len/2 bytes)
  bool in_group = false;        // reader packs it into a group
  std::uint32_t item = 0;       // reader item (big entries)
  std::uint32_t chunk0 = 0;     // reader landing chunk index of the item
  std::uint32_t chunk_len = 0;  // reader chunk length of the item
  // a member of the reader's own member-cut group: where it sits in the
  // group's staging and its run of chunks (stage_ptr 0: not eligible)
  std::uint64_t stage_ptr = 0;
  std::uint32_t stage_chunk0 = 0;
  std::uint32_t stage_chunk_len = 0;
  std::uint32_t group_item = 0;
};

Status plan_reshard(const std::vector<ReaderEntry>& reader, const std::vector<SourceShard>& srcs,
                    ReshardPlan* out);

}  // namespace rsb
