#include "manifest.hpp"

#include <unordered_set>

namespace rsb {

namespace {

// ---- tagged big-endian fields (wire format of codec.cpp:28-150) ----------
enum Wire : std::uint8_t { kU64 = 1, kBytes = 2, kList = 3 };

void be32(std::string& o, std::uint32_t v) {
  for (int s = 24; s >= 0; s -= 8) o.push_back(static_cast<char>(v >> s));
}
void be64(std::string& o, std::uint64_t v) {
  be32(o, static_cast<std::uint32_t>(v >> 32));
  be32(o, static_cast<std::uint32_t>(v));
}
std::uint32_t rd32(const unsigned char* p) {
  return (std::uint32_t(p[0]) << 24) | (std::uint32_t(p[1]) << 16) |
         (std::uint32_t(p[2]) << 8) | std::uint32_t(p[3]);
}
std::uint64_t rd64(const unsigned char* p) {
  return (std::uint64_t(rd32(p)) << 32) | rd32(p + 4);
}

void field_u64(std::string& o, std::uint8_t tag, std::uint64_t v) {
  o.push_back(static_cast<char>(tag));
  o.push_back(static_cast<char>(kU64));
  be64(o, v);
}
void field_bytes(std::string& o, std::uint8_t tag, std::string_view b) {
  o.push_back(static_cast<char>(tag));
  o.push_back(static_cast<char>(kBytes));
  be32(o, static_cast<std::uint32_t>(b.size()));
  o.append(b);
}
void field_list(std::string& o, std::uint8_t tag,
                const std::vector<std::string>& elems) {
  o.push_back(static_cast<char>(tag));
  o.push_back(static_cast<char>(kList));
  be32(o, static_cast<std::uint32_t>(elems.size()));
  for (const auto& e : elems) {
    be32(o, static_cast<std::uint32_t>(e.size()));
    o.append(e);
  }
}

// Parsed view of one field record; first occurrence of a tag wins.
struct Fields {
  struct F {
    std::uint8_t tag, wire;
    std::string_view body;
  };
  std::vector<F> fs;
  bool ok = true;

  explicit Fields(std::string_view d) {
    auto* p = reinterpret_cast<const unsigned char*>(d.data());
    std::size_t n = d.size(), i = 0;
    while (i < n) {
      if (n - i < 2) { fail(); return; }
      F f{p[i], p[i + 1], {}};
      i += 2;
      std::size_t start = i;
      if (f.wire == kU64) {
        if (n - i < 8) { fail(); return; }
        i += 8;
      } else if (f.wire == kBytes) {
        if (n - i < 4) { fail(); return; }
        std::uint32_t len = rd32(p + i);
        i += 4;
        start = i;
        if (n - i < len) { fail(); return; }
        i += len;
      } else if (f.wire == kList) {
        if (n - i < 4) { fail(); return; }
        std::uint32_t cnt = rd32(p + i);
        i += 4;
        for (std::uint32_t k = 0; k < cnt; ++k) {
          if (n - i < 4) { fail(); return; }
          std::uint32_t len = rd32(p + i);
          i += 4;
          if (n - i < len) { fail(); return; }
          i += len;
        }
      } else {
        { fail(); return; }
      }
      f.body = d.substr(start, i - start);
      fs.push_back(f);
    }
  }
  void fail() { ok = false; }
  const F* find(std::uint8_t tag, std::uint8_t wire) const {
    for (const auto& f : fs)
      if (f.tag == tag) return f.wire == wire ? &f : nullptr;
    return nullptr;
  }
  bool u64(std::uint8_t tag, std::uint64_t& out) const {
    auto* f = find(tag, kU64);
    if (!f) return false;
    out = rd64(reinterpret_cast<const unsigned char*>(f->body.data()));
    return true;
  }
  bool bytes(std::uint8_t tag, std::string_view& out) const {
    auto* f = find(tag, kBytes);
    if (!f) return false;
    out = f->body;
    return true;
  }
  bool list(std::uint8_t tag, std::vector<std::string_view>& out) const {
    auto* f = find(tag, kList);
    if (!f) return false;
    auto* p = reinterpret_cast<const unsigned char*>(f->body.data());
    std::uint32_t cnt = rd32(p);
    std::size_t i = 4;
    for (std::uint32_t k = 0; k < cnt; ++k) {
      std::uint32_t len = rd32(p + i);
      out.push_back(f->body.substr(i + 4, len));
      i += 4 + len;
    }
    return true;
  }
};

}  // namespace

Status Manifest::finalize() {
  items_.clear();
  owner_.assign(entries.size(), -1);
  total_ = 0;
  std::unordered_set<std::string_view> seen;
  for (const auto& e : entries) {
    if (e.name.empty() || e.length == 0 || !seen.insert(e.name).second)
      return Status::invalid_argument;
    total_ += e.length;
  }
  for (std::size_t g = 0; g < groups.size(); ++g) {
    const auto& grp = groups[g];
    if (grp.members.empty()) return Status::invalid_argument;
    if (g > 0 && grp.members.front().entry <= groups[g - 1].members.front().entry)
      return Status::invalid_argument;
    std::uint64_t expect = 0;
    for (std::size_t k = 0; k < grp.members.size(); ++k) {
      const auto& m = grp.members[k];
      if (m.entry >= entries.size() || owner_[m.entry] != -1 ||
          m.offset != expect ||
          (k > 0 && m.entry <= grp.members[k - 1].entry))
        return Status::invalid_argument;
      owner_[m.entry] = static_cast<int>(g);
      expect += entries[m.entry].length;
    }
    if (expect != grp.packed_length) return Status::invalid_argument;
  }
  std::uint64_t pos = 0;
  for (std::uint32_t e = 0; e < entries.size(); ++e) {
    StreamItem it;
    int g = owner_[e];
    if (g < 0) {
      it = {false, e, entries[e].length, entries[e].digest, pos};
    } else if (groups[g].members.front().entry == e) {
      it = {true, static_cast<std::uint32_t>(g), groups[g].packed_length,
            groups[g].digest, pos};
    } else {
      continue;
    }
    pos += it.length;
    items_.push_back(it);
  }
  return Status::ok;
}

void Manifest::set_group_digest(std::uint32_t g, std::uint64_t d) {
  groups[g].digest = d;
  for (auto& it : items_)
    if (it.is_group && it.index == g) it.digest = d;
}

void Manifest::set_entry_digest(std::uint32_t e, std::uint64_t d) {
  entries[e].digest = d;
  for (auto& it : items_)
    if (!it.is_group && it.index == e) it.digest = d;
}

bool Manifest::same_structure(const Manifest& o) const {
  if (alg != o.alg || entries.size() != o.entries.size() || groups.size() != o.groups.size()) return false;
  for (std::size_t i = 0; i < entries.size(); ++i)
    if (entries[i].name != o.entries[i].name || entries[i].length != o.entries[i].length) return false;
  for (std::size_t g = 0; g < groups.size(); ++g) {
    if (groups[g].packed_length != o.groups[g].packed_length ||
        groups[g].members.size() != o.groups[g].members.size())
      return false;
    for (std::size_t k = 0; k < groups[g].members.size(); ++k)
      if (groups[g].members[k].entry != o.groups[g].members[k].entry ||
          groups[g].members[k].offset != o.groups[g].members[k].offset)
        return false;
  }
  return true;
}

std::string Manifest::encode() const {
  std::string out;
  field_u64(out, 1, 1);  // format version
  field_u64(out, 2, alg);  // digest algorithm tag: 1 = XXH64 seed 0
  std::vector<std::string> blobs;
  blobs.reserve(entries.size());
  for (const auto& e : entries) {
    std::string b;
    field_bytes(b, 1, e.name);
    field_u64(b, 2, e.length);
    field_u64(b, 3, e.digest);
    blobs.push_back(std::move(b));
  }
  field_list(out, 3, blobs);
  blobs.clear();
  for (const auto& g : groups) {
    std::string b, mem;
    field_u64(b, 1, g.packed_length);
    field_u64(b, 2, g.digest);
    for (const auto& m : g.members) {
      be32(mem, m.entry);
      be64(mem, m.offset);
    }
    field_bytes(b, 3, mem);
    blobs.push_back(std::move(b));
  }
  field_list(out, 4, blobs);
  return out;
}

Result<Manifest> Manifest::decode(std::string_view bytes) {
  Fields top(bytes);
  std::uint64_t fmt = 0, alg = 0;
  if (!top.ok) return Status::protocol_error;
  if (!top.u64(1, fmt) || fmt != 1 || !top.u64(2, alg) || (alg != kAlgXxh64 && alg != kAlgDerived))
    return Status::protocol_error;
  std::vector<std::string_view> eb, gb;
  if (!top.list(3, eb) || !top.list(4, gb)) return Status::protocol_error;
  Manifest m;
  m.alg = static_cast<std::uint8_t>(alg);
  for (auto blob : eb) {
    Fields f(blob);
    ManifestEntry e;
    std::string_view name;
    if (!f.ok || !f.bytes(1, name) || !f.u64(2, e.length) || !f.u64(3, e.digest))
      return Status::protocol_error;
    e.name = std::string(name);
    m.entries.push_back(std::move(e));
  }
  for (auto blob : gb) {
    Fields f(blob);
    PackGroup g;
    std::string_view mem;
    if (!f.ok || !f.u64(1, g.packed_length) || !f.u64(2, g.digest) ||
        !f.bytes(3, mem) || mem.size() % 12 != 0)
      return Status::protocol_error;
    auto* p = reinterpret_cast<const unsigned char*>(mem.data());
    for (std::size_t i = 0; i < mem.size(); i += 12)
      g.members.push_back({rd32(p + i), rd64(p + i + 4)});
    m.groups.push_back(std::move(g));
  }
  if (Status s = m.finalize(); !ok(s)) return s;
  return m;
}

Result<Manifest> assemble(const std::vector<EntryInfo>& infos,
                          const PackLimits& limits) {
  Manifest m;
  PackGroup cur;
  for (std::uint32_t e = 0; e < infos.size(); ++e) {
    const auto& in = infos[e];
    m.entries.push_back({in.name, in.length, in.digest});
    if (in.length >= limits.tiny_threshold) continue;
    if (!cur.members.empty() &&
        cur.packed_length + in.length > limits.group_target) {
      m.groups.push_back(std::move(cur));
      cur = PackGroup{};
    }
    cur.members.push_back({e, cur.packed_length});
    cur.packed_length += in.length;
  }
  if (!cur.members.empty()) m.groups.push_back(std::move(cur));
  if (Status s = m.finalize(); !ok(s)) return s;
  return m;
}

}  // namespace rsb
