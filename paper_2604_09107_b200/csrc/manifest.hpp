// Tensor manifest: per-shard entry table, tiny-tensor packing and the ordered
// transfer-item stream.  Behaviour (validation, item order, packing rule,
// canonical bytes) follows the reference TensorManifest
// (/root/reference/proj/include/refstore/manifest.hpp:18-113,
//  src/manifest.cpp:12-249); the implementation is independent.
#pragma once

#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

#include "common.hpp"

namespace rsb {

struct ManifestEntry {
  std::string name;
  std::uint64_t length = 0;
  std::uint64_t digest = 0;
};

struct GroupMember {
  std::uint32_t entry = 0;
  std::uint64_t offset = 0;
};

struct PackGroup {
  std::uint64_t packed_length = 0;
  std::uint64_t digest = 0;
  std::vector<GroupMember> members;
};

// One transfer unit: a big entry, or a packed group carried at the position
// of its first member (manifest.hpp:35-44).
struct StreamItem {
  bool is_group = false;
  std::uint32_t index = 0;
  std::uint64_t length = 0;
  std::uint64_t digest = 0;
  std::uint64_t stream_offset = 0;
};

struct PackLimits {
  std::uint64_t tiny_threshold = 2ull << 20;
  std::uint64_t group_target = 64ull << 20;
};

// Digest algorithm tag carried by the manifest (field 2).  1 = reference
// XXH64 of every entry / group (digest.hpp:13).  2 = derived reshard layout:
// entry and group digests are not computed (0); the bytes were verified
// chunk by chunk against the source layout's chunk digests.
constexpr std::uint8_t kAlgXxh64 = 1;
constexpr std::uint8_t kAlgDerived = 2;

class Manifest {
 public:
  std::vector<ManifestEntry> entries;
  std::vector<PackGroup> groups;
  std::uint8_t alg = kAlgXxh64;

  Status finalize();  // validates + derives items (manifest.cpp:12-72)
  const std::vector<StreamItem>& items() const { return items_; }
  std::uint64_t total_bytes() const { return total_; }
  int group_of(std::uint32_t entry) const { return owner_[entry]; }
  void set_group_digest(std::uint32_t g, std::uint64_t d);
  void set_entry_digest(std::uint32_t e, std::uint64_t d);
  // Same entries (names, lengths), groups (packing) and algorithm tag: the
  // manifests differ at most in their digests.
  bool same_structure(const Manifest& o) const;

  std::string encode() const;  // canonical bytes (manifest.cpp:103-139)
  static Result<Manifest> decode(std::string_view bytes);

 private:
  std::vector<StreamItem> items_;
  std::vector<int> owner_;
  std::uint64_t total_ = 0;
};

struct EntryInfo {
  std::string name;
  std::uint64_t length = 0;
  std::uint64_t digest = 0;
};

// assemble_manifest (manifest.cpp:179-202): registration order, entries under
// the tiny threshold packed into groups that close before exceeding target.
Result<Manifest> assemble(const std::vector<EntryInfo>& entries,
                          const PackLimits& limits);

}  // namespace rsb
