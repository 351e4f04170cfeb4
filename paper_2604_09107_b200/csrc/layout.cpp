#include "layout.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <numeric>
#include <set>

namespace rsb {

std::uint32_t chunk_len_for(const Geometry& g, std::uint64_t chunk_bytes, std::uint32_t align) {
  const auto fallback = static_cast<std::uint32_t>(chunk_bytes);
  if (!g.has() || align == 0 || g.row_bytes % align || g.nc == 0) return fallback;
  const std::uint64_t band = g.row_bytes / align;
  const std::uint64_t gg = std::gcd(g.nc, band);
  for (std::uint64_t c = std::min<std::uint64_t>(chunk_bytes, gg) / 128 * 128; c >= 128; c -= 128)
    if (gg % c == 0) return static_cast<std::uint32_t>(c);
  return fallback;
}

std::string ShardLayout::encode() const {
  std::string s;
  auto put = [&](const void* p, std::size_t n) { s.append(static_cast<const char*>(p), n); };
  const auto ng = static_cast<std::uint32_t>(geo.size());
  const auto nc = static_cast<std::uint32_t>(chunk_len.size());
  put(&ng, 4);
  for (const auto& g : geo) {
    const std::uint64_t v[6] = {g.rows, g.row_bytes, g.r0, g.nr, g.c0, g.nc};
    put(v, sizeof(v));
  }
  put(&nc, 4);
  if (nc) put(chunk_len.data(), 4 * std::size_t(nc));
  return s;
}

Result<ShardLayout> ShardLayout::decode(std::string_view s) {
  ShardLayout l;
  std::size_t i = 0;
  auto get = [&](void* p, std::size_t n) {
    if (i + n > s.size()) return false;
    std::memcpy(p, s.data() + i, n);
    i += n;
    return true;
  };
  std::uint32_t ng = 0, nc = 0;
  if (!get(&ng, 4)) return Status::protocol_error;
  l.geo.resize(ng);
  for (auto& g : l.geo) {
    std::uint64_t v[6];
    if (!get(v, sizeof(v))) return Status::protocol_error;
    g = {v[0], v[1], v[2], v[3], v[4], v[5]};
  }
  if (!get(&nc, 4)) return Status::protocol_error;
  l.chunk_len.resize(nc);
  if (nc && !get(l.chunk_len.data(), 4 * std::size_t(nc))) return Status::protocol_error;
  if (i != s.size()) return Status::protocol_error;
  return l;
}

std::vector<std::uint32_t> item_chunk_lens(const Manifest& m, const std::vector<Geometry>& geo,
                                           std::uint64_t chunk_bytes, std::uint32_t align) {
  std::vector<std::uint32_t> out;
  for (const auto& it : m.items()) {
    if (!it.is_group && it.index < geo.size()) {
      out.push_back(chunk_len_for(geo[it.index], chunk_bytes, align));
    } else if (it.is_group) {
      bool cut = false;  // member rule: some member carries a geometry
      for (const auto& mem : m.groups[it.index].members)
        cut |= mem.entry < geo.size() && geo[mem.entry].has();
      out.push_back(cut ? 0u : static_cast<std::uint32_t>(chunk_bytes));
    } else {
      out.push_back(static_cast<std::uint32_t>(chunk_bytes));
    }
  }
  return out;
}

std::vector<std::uint32_t> member_chunk_lens(const Manifest& m, const std::vector<Geometry>& geo,
                                             std::uint64_t chunk_bytes, std::uint32_t align) {
  std::vector<std::uint32_t> out(m.entries.size(), static_cast<std::uint32_t>(chunk_bytes));
  for (std::size_t e = 0; e < out.size() && e < geo.size(); ++e)
    if (geo[e].has()) out[e] = chunk_len_for(geo[e], chunk_bytes, align);
  return out;
}

namespace {

// Entry index of `name` in a manifest (-1: absent).
int entry_of(const Manifest& m, const std::string& name) {
  for (std::size_t e = 0; e < m.entries.size(); ++e)
    if (m.entries[e].name == name) return static_cast<int>(e);
  return -1;
}

// Item carrying entry e, and the entry's offset inside it.
std::pair<std::uint32_t, std::uint64_t> item_of(const Manifest& m, std::uint32_t e) {
  const int g = m.group_of(e);
  const auto& items = m.items();
  for (std::uint32_t i = 0; i < items.size(); ++i) {
    if (g < 0 && !items[i].is_group && items[i].index == e) return {i, 0};
    if (g >= 0 && items[i].is_group && items[i].index == static_cast<std::uint32_t>(g)) {
      for (const auto& mem : m.groups[g].members)
        if (mem.entry == e) return {i, mem.offset};
    }
  }
  return {0, 0};
}

Geometry full_geometry(std::uint64_t len) { return {1, len, 0, 1, 0, len}; }

}  // namespace

Status plan_reshard(const std::vector<ReaderEntry>& reader, const std::vector<SourceShard>& srcs,
                    ReshardPlan* out) {
  out->segs.clear();
  out->gathers.clear();
  out->copies.clear();
  out->rehash.clear();
  out->direct_groups.clear();
  std::map<std::pair<std::uint32_t, std::uint32_t>, bool> gathered;
  // One reader entry's pieces, appended to `into`.  staged: the entry is a
  // member of the reader's member-cut group and may land straight in the
  // group's staging.
  auto plan_one = [&](const ReaderEntry& r, ReshardPlan* into, bool staged) -> Status {
    const Geometry rg = r.geo.has() ? r.geo : full_geometry(r.len);
    std::uint64_t covered = 0;
    // Source slices already taken for this region.  Replicated tensors (a
    // norm every TP rank holds whole) overlap identically: the first source
    // serves, the rest are skipped; TP/FSDP slices are disjoint.
    struct Rect {
      std::uint64_t a, b, c0, c1;
    };
    std::vector<Rect> taken;
    for (std::uint32_t si = 0; si < srcs.size(); ++si) {
      const SourceShard& ss = srcs[si];
      const int e = entry_of(ss.manifest, r.name);
      if (e < 0) continue;
      const std::uint64_t slen = ss.manifest.entries[e].length;
      const Geometry sg = (static_cast<std::size_t>(e) < ss.layout.geo.size() &&
                           ss.layout.geo[e].has())
                              ? ss.layout.geo[e]
                              : full_geometry(slen);
      if (sg.rows != rg.rows || sg.row_bytes != rg.row_bytes) return Status::invalid_argument;
      const std::uint64_t a = std::max(rg.r0, sg.r0), b = std::min(rg.r0 + rg.nr, sg.r0 + sg.nr);
      const std::uint64_t c0 = std::max(rg.c0, sg.c0), c1 = std::min(rg.c0 + rg.nc, sg.c0 + sg.nc);
      if (a >= b || c0 >= c1) continue;
      bool dup = false, partial = false;
      for (const Rect& t : taken) {
        const bool meet = a < t.b && t.a < b && c0 < t.c1 && t.c0 < c1;
        if (!meet) continue;
        if (a >= t.a && b <= t.b && c0 >= t.c0 && c1 <= t.c1) dup = true;
        else partial = true;
      }
      if (dup) continue;
      if (partial) return Status::invalid_argument;  // overlapping but unequal source slices
      taken.push_back({a, b, c0, c1});
      covered += (b - a) * (c1 - c0);
      const auto [item, ioff] = item_of(ss.manifest, static_cast<std::uint32_t>(e));
      const bool src_big = !ss.manifest.items()[item].is_group;
      std::uint32_t c = item < ss.layout.chunk_len.size() ? ss.layout.chunk_len[item] : 0;
      // a member of a member-cut group: its own run of chunks inside the item
      std::uint32_t run_first = 0;
      bool member_run = false;
      if (!src_big && item < ss.parts.size())
        for (const ChunkPart& p : ss.parts[item])
          if (p.off == ioff) {
            c = p.chunk_len;
            run_first = p.first;
            member_run = true;
          }
      // a member of this reader's own member-cut group lands in its group
      // staging (staged), else the region itself
      const std::uint32_t want_c = staged ? r.stage_chunk_len : r.chunk_len;
      const bool aligned = (!r.in_group || staged) && (src_big || member_run) && c != 0 && c == want_c &&
                           (c0 - sg.c0) % c == 0 && (c1 - c0) % c == 0 && sg.nc % c == 0 &&
                           (c1 - c0) == rg.nc && sg.nc / c <= 0xffff;
      if (aligned) {
        dev::ItemDesc d{};
        // offset in the source item; its base address is added by the caller
        d.src = ioff + ((a - sg.r0) * sg.nc + (c0 - sg.c0));
        d.dst = (staged ? r.stage_ptr : r.ptr) + (a - rg.r0) * rg.nc / (r.cast ? 2 : 1);
        d.len = (b - a) * (c1 - c0);
        const std::uint64_t m = sg.nc / c, q = (c1 - c0) / c;
        d.chunk0 = (staged ? r.stage_chunk0 : r.chunk0) + static_cast<std::uint32_t>((a - rg.r0) * q);
        d.chunk_len = c | (r.cast ? dev::kCastE4M3 : 0u);
        d.src_chunk0 = ss.chunk0[item] + run_first +
                       static_cast<std::uint32_t>((a - sg.r0) * m + (c0 - sg.c0) / c);
        d.q = static_cast<std::uint16_t>(q);
        d.m = static_cast<std::uint16_t>(m);
        d.src_id = si;
        d.pad = item;  // source item (base address looked up by the caller)
        into->segs.push_back(d);
      } else {
        if (!gathered[{si, item}]) {
          gathered[{si, item}] = true;
          into->gathers.push_back({si, item});
        }
        SliceCopy cp;
        cp.src_shard = si;
        cp.src_item = item;
        cp.src_off = ioff + (a - sg.r0) * sg.nc + (c0 - sg.c0);
        cp.src_stride = sg.nc;
        const std::uint64_t shrink = r.cast ? 2 : 1;
        cp.dst = r.ptr + ((a - rg.r0) * rg.nc + (c0 - rg.c0)) / shrink;
        cp.dst_stride = rg.nc / shrink;
        cp.rows = b - a;
        cp.nc = c1 - c0;
        cp.cast = r.cast;
        into->copies.push_back(cp);
        if (!r.in_group && !r.cast &&
            std::find(into->rehash.begin(), into->rehash.end(), r.item) == into->rehash.end())
          into->rehash.push_back(r.item);
      }
    }
    if (covered != rg.nr * rg.nc || rg.nr * rg.nc != r.len) return Status::version_unavailable;
    return Status::ok;
  };
  std::map<std::uint32_t, std::vector<const ReaderEntry*>> groups;  // reader group item -> members
  for (const auto& r : reader) {
    if (r.in_group && r.stage_ptr) {
      groups[r.group_item].push_back(&r);
      continue;
    }
    if (Status st = plan_one(r, out, false); !ok(st)) return st;
  }
  // A reader group lands straight from the sources only when every member
  // does: its watermarks are released by the fill, so no member may still
  // be on its way by copy.  Otherwise the whole group is copied and
  // re-digested as before.
  for (const auto& [gitem, members] : groups) {
    ReshardPlan trial;
    auto gathered_before = gathered;
    bool direct = true;
    for (const ReaderEntry* r : members) {
      if (Status st = plan_one(*r, &trial, true); !ok(st)) return st;
      if (!trial.copies.empty()) {
        direct = false;
        break;
      }
    }
    if (direct) {
      out->segs.insert(out->segs.end(), trial.segs.begin(), trial.segs.end());
      out->direct_groups.push_back(gitem);
      continue;
    }
    gathered = std::move(gathered_before);
    for (const ReaderEntry* r : members)
      if (Status st = plan_one(*r, out, false); !ok(st)) return st;
  }
  std::sort(out->segs.begin(), out->segs.end(),
            [](const dev::ItemDesc& x, const dev::ItemDesc& y) { return x.chunk0 < y.chunk0; });
  return Status::ok;
}

}  // namespace rsb
