#include "registry.hpp"

#include <algorithm>
#include <chrono>
#include <sstream>
#include <tuple>

#include "manifest.hpp"

namespace rsb {

namespace {
std::string n2s(std::uint64_t v) { return std::to_string(v); }
}  // namespace

std::string TraceLine::format() const {
  std::ostringstream o;
  o << seq << ' ' << kind;
  for (const auto& [k, v] : kv) o << ' ' << k << '=' << v;
  return o.str();
}

Registry::Registry(Config cfg) : cfg_(cfg) {
  topo_ = [](const std::string&, const std::string&) { return 0; };
}

void Registry::set_topology(TopoFn fn) {
  std::lock_guard lk(mu_);
  topo_ = fn ? std::move(fn)
             : TopoFn([](const std::string&, const std::string&) { return 0; });
}

const char* Registry::life_name(Life l) {
  switch (l) {
    case Life::registered: return "registered";
    case Life::replicating: return "replicating";
    case Life::published: return "published";
    case Life::failed: return "failed";
  }
  return "?";
}

Registry::Rep* Registry::find(const std::string& model,
                              const std::string& replica) {
  auto mit = models_.find(model);
  if (mit == models_.end()) return nullptr;
  auto it = mit->second.reps.find(replica);
  return it == mit->second.reps.end() ? nullptr : it->second.get();
}

void Registry::trace(std::string kind,
                     std::vector<std::pair<std::string, std::string>> kv) {
  TraceLine t;
  t.seq = trace_.size();
  t.kind = std::move(kind);
  t.kv = std::move(kv);
  trace_.push_back(std::move(t));
}

// ------------------------------------------------------------------ opening

Status Registry::open(const std::string& model, const std::string& replica,
                      std::uint32_t num_shards, const std::string& dc,
                      const std::vector<std::string>& endpoints, const std::string& layout,
                      const std::vector<std::string>& derived_manifests,
                      const std::vector<std::string>& derived_layouts) {
  std::lock_guard lk(mu_);
  if (model.empty() || replica.empty() || num_shards == 0 ||
      endpoints.size() != num_shards)
    return Status::invalid_argument;
  auto& m = ms(model);
  auto it = m.reps.find(replica);
  if (it != m.reps.end()) {
    Rep& r = *it->second;
    // Re-opening an idle record with the same geometry refreshes endpoints;
    // a failed record is replaced by a fresh one (reference evict + reopen).
    if (r.life != Life::failed) {
      if (r.num_shards != num_shards) return Status::invalid_argument;
      r.endpoints = endpoints;
      r.dc = dc;
      r.layout = layout;
      r.derived_manifests = derived_manifests;
      r.derived_layouts = derived_layouts;
      return Status::ok;
    }
    m.reps.erase(it);
  }
  auto r = std::make_unique<Rep>();
  r->model = model;
  r->name = replica;
  r->dc = dc;
  r->num_shards = num_shards;
  r->endpoints = endpoints;
  r->layout = layout;
  r->derived_manifests = derived_manifests;
  r->derived_layouts = derived_layouts;
  r->shards.assign(num_shards, {});
  m.reps.emplace(replica, std::move(r));
  trace("open", {{"model", model}, {"replica", replica}, {"shards", n2s(num_shards)}});
  return Status::ok;
}

Status Registry::close(const std::string& model, const std::string& replica) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (!r) return Status::not_found;
  bool busy = r->life == Life::published || r->life == Life::replicating ||
              r->txn.has_value();
  if (busy) fail_replica(*r, "closed");
  if (r->txn) finish_op(*r, Status::closed);
  auto& m = ms(model);
  // owned offload buffers die with their owner (server_core.cpp:1715-1733)
  std::vector<std::string> owned;
  for (const auto& [name, o] : m.reps)
    if (o->kind == Kind::offload && o->owner == replica) owned.push_back(name);
  for (const auto& name : owned) {
    auto it = m.reps.find(name);
    const VersionId v = it->second->offload_v;
    trace("offload_dropped", {{"model", model}, {"replica", name}, {"reason", "owner_closed"}});
    m.reps.erase(it);
    prune_version(m, v);
  }
  r = find(model, replica);
  if (r && r->serving == 0) {
    m.reps.erase(replica);
  }
  cv_.notify_all();
  return Status::ok;
}

// ------------------------------------------------------------- availability

std::set<VersionId> Registry::available(ModelState& m, const std::string& dc) {
  std::set<VersionId> out;
  for (const auto& [name, r] : m.reps)
    if (r->visible && r->life == Life::published && r->version &&
        r->complete_all())
      out.insert(*r->version);
  if (cfg_.smart_skipping) {
    // Hide versions this datacenter only holds as in-flight cross-DC seeds
    // (server_core.cpp:1496-1513).
    std::vector<VersionId> masked;
    for (VersionId v : out) {
      bool local_complete = false, local_seeding = false;
      for (const auto& [name, r] : m.reps) {
        if (r->version != v || r->dc != dc) continue;
        if (r->visible && r->life == Life::published && r->complete_all())
          local_complete = true;
        if (r->life == Life::replicating && r->seeding) local_seeding = true;
      }
      if (!local_complete && local_seeding) masked.push_back(v);
    }
    for (VersionId v : masked) out.erase(v);
  }
  return out;
}

bool Registry::still_good(const Rep& c, const Rep& reader, VersionId v) const {
  if (&c == &reader || c.life == Life::failed || c.version != v) return false;
  // A terminal copy (its regions hold a cast of the version's bytes) never
  // serves: its landed bytes are not the bytes the digests describe.
  if (terminal_layout(c.layout)) return false;
  bool complete_copy = c.visible && c.life == Life::published && c.complete_all();
  // A differently sliced copy serves only a reshard-capable reader, and only
  // once complete (chasing is item-for-item).
  if (c.layout != slicing(reader.layout)) return complete_copy && !slicing(reader.layout).empty();
  bool pipeline_copy = cfg_.pipeline && c.life == Life::replicating &&
                       !c.seeding && c.dc == reader.dc;
  return complete_copy || pipeline_copy;
}

bool Registry::servable(ModelState& m, VersionId v, const Rep& reader) {
  auto vit = m.versions.find(v);
  if (vit == m.versions.end()) return false;
  auto lit = vit->second.by_layout.find(slicing(reader.layout));
  if (lit != vit->second.by_layout.end()) return lit->second.num_shards == reader.num_shards;
  return !slicing(reader.layout).empty();  // reshard from another slicing
}

Registry::Rep* Registry::pick_source(ModelState& m, VersionId v,
                                     const Rep& reader) {
  const std::string& rep0 = reader.endpoints.empty() ? reader.name : reader.endpoints[0];
  // Reference key (own_seed, same_dc, serving, last_assigned, name) with two
  // B200 terms that are constant when every replica has the same slicing and
  // the box is uniform: same slicing first, then topology cost.
  auto key = [&](const Rep* c) {
    const std::string& ep0 = c->endpoints.empty() ? c->name : c->endpoints[0];
    const bool own_seed = c->kind == Kind::offload && c->seed && c->owner == reader.name;
    return std::make_tuple(own_seed ? 0 : 1, c->dc == reader.dc ? 0 : 1,
                           c->layout == slicing(reader.layout) ? 0 : 1, topo_(rep0, ep0), c->serving,
                           c->last_assigned, std::cref(c->name));
  };
  auto vit = m.versions.find(v);
  Rep* best = nullptr;
  for (auto& [name, rp] : m.reps) {
    Rep* c = rp.get();
    if (!still_good(*c, reader, v)) continue;
    // a copy is a source only once its slicing's metadata is known for v
    if (vit == m.versions.end() || !vit->second.by_layout.count(c->layout)) continue;
    if (!best || key(c) < key(best)) best = c;
  }
  return best;
}

Assignment Registry::make_assignment(ModelState& m, Rep& src, VersionId v,
                                     std::uint32_t shard, const Rep& reader) {
  Assignment a;
  a.version = v;
  a.source_replica = src.name;
  a.source_endpoint = shard < src.endpoints.size() ? src.endpoints[shard] : "";
  a.source_complete = src.life == Life::published && src.complete_all();
  a.cross_dc = src.dc != reader.dc;
  LayoutInfo& li = m.versions[v].by_layout[src.layout];
  a.provisional = li.provisional;
  if (src.layout == slicing(reader.layout)) {
    a.manifest = shard < li.manifests.size() ? li.manifests[shard] : "";
    a.layout = shard < li.layouts.size() ? li.layouts[shard] : "";
  } else {
    a.reshard = true;
    if (!li.man_sp) li.man_sp = std::make_shared<const std::vector<std::string>>(li.manifests);
    if (!li.lay_sp) li.lay_sp = std::make_shared<const std::vector<std::string>>(li.layouts);
    a.all_manifests = li.man_sp;
    a.all_layouts = li.lay_sp;
    a.all_endpoints = src.endpoints;
  }
  return a;
}

// ------------------------------------------------------------------ publish

Status Registry::publish(const std::string& model, const std::string& replica,
                         VersionId v, const std::vector<std::string>& manifests,
                         OpOutcome* out, const std::vector<std::string>& layouts,
                         bool provisional) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (!r) return Status::not_found;
  if (r->txn) return Status::invalid_state;
  if (manifests.size() != r->num_shards) return Status::invalid_argument;
  if (!layouts.empty() && layouts.size() != r->num_shards) return Status::invalid_argument;
  if (terminal_layout(r->layout)) return Status::invalid_state;  // holds a cast, not the bytes
  auto reject = [&](Status s, const char* why) {
    if (why)
      trace("publish_reject", {{"model", model}, {"replica", replica}, {"v", n2s(v)},
                               {"reason", why}});
    r->last = {true, s, std::nullopt, false, {}};
    if (out) *out = r->last;
    return s;
  };
  if (r->life == Life::published) return reject(Status::mutability_violation, "already_published");
  if (r->life != Life::registered) return reject(Status::invalid_state, nullptr);
  if (r->last_published && v <= *r->last_published)
    return reject(Status::version_regression, "regression");
  std::vector<std::uint64_t> items(r->num_shards);
  for (std::uint32_t s = 0; s < r->num_shards; ++s) {
    auto mf = Manifest::decode(manifests[s]);
    if (!mf) return reject(Status::manifest_conflict, nullptr);
    items[s] = mf->items().size();
  }
  auto& m = ms(model);
  // A version number already defined for this slicing must carry
  // byte-identical manifests (server_core.cpp:666-683).
  auto& vi = m.versions[v];
  auto lit = vi.by_layout.find(r->layout);
  if (lit != vi.by_layout.end()) {
    if (lit->second.num_shards != r->num_shards) return reject(Status::manifest_conflict, nullptr);
    for (std::uint32_t s = 0; s < r->num_shards; ++s) {
      if (lit->second.manifests[s] == manifests[s]) continue;
      // an early publish on either side: the structures must agree
      auto a = Manifest::decode(lit->second.manifests[s]), b = Manifest::decode(manifests[s]);
      if (!(provisional || lit->second.provisional) || !a || !b || !a->same_structure(*b))
        return reject(Status::manifest_conflict, "manifest_conflict");
    }
    if (lit->second.provisional && !provisional) {
      lit->second.manifests = manifests;  // this publisher brings the final bytes
      lit->second.provisional = false;
      lit->second.man_sp.reset();
    }
  } else {
    LayoutInfo li{r->num_shards, manifests, layouts, provisional};
    li.layouts.resize(r->num_shards);
    vi.by_layout.emplace(r->layout, std::move(li));
  }
  r->life = Life::published;
  r->visible = true;
  r->version = v;
  r->last_published = v;
  for (std::uint32_t s = 0; s < r->num_shards; ++s) r->shards[s] = {items[s], true};
  if (!m.max_published || v > *m.max_published) m.max_published = v;
  trace("publish_commit", {{"model", model}, {"replica", replica}, {"v", n2s(v)}});
  eval_offload_releases(model);
  r->last = {true, Status::ok, v, false, {}};
  if (out) *out = r->last;
  wake_blocked(model);
  cv_.notify_all();
  return Status::ok;
}

Status Registry::finalize_manifests(const std::string& model, const std::string& replica,
                                    VersionId v, const std::vector<std::string>& manifests) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (!r) return Status::not_found;
  auto& m = ms(model);
  auto vit = m.versions.find(v);
  if (vit == m.versions.end()) return Status::not_found;
  auto lit = vit->second.by_layout.find(r->layout);
  if (lit == vit->second.by_layout.end()) return Status::not_found;
  LayoutInfo& li = lit->second;
  if (manifests.size() != li.num_shards) return Status::invalid_argument;
  if (!li.provisional) return li.manifests == manifests ? Status::ok : Status::manifest_conflict;
  for (std::uint32_t s = 0; s < li.num_shards; ++s) {
    auto a = Manifest::decode(li.manifests[s]), b = Manifest::decode(manifests[s]);
    if (!a || !b || !a->same_structure(*b)) return Status::manifest_conflict;
  }
  li.manifests = manifests;
  li.provisional = false;
  li.man_sp.reset();
  trace("manifest_final", {{"model", model}, {"replica", replica}, {"v", n2s(v)}});
  cv_.notify_all();
  return Status::ok;
}

Status Registry::current_manifest(const std::string& model, VersionId v, const std::string& layout_key,
                                  std::uint32_t shard, std::string* bytes, bool* final_bytes) {
  std::lock_guard lk(mu_);
  auto& m = ms(model);
  auto vit = m.versions.find(v);
  if (vit == m.versions.end()) return Status::not_found;
  auto lit = vit->second.by_layout.find(slicing(layout_key));
  if (lit == vit->second.by_layout.end() || shard >= lit->second.manifests.size()) return Status::not_found;
  *bytes = lit->second.manifests[shard];
  *final_bytes = !lit->second.provisional;
  return Status::ok;
}

Status Registry::replica_manifest(const std::string& model, const std::string& replica, VersionId v,
                                  std::uint32_t shard, std::string* bytes, bool* final_bytes) {
  std::string key;
  {
    std::lock_guard lk(mu_);
    Rep* r = find(model, replica);
    if (!r) return Status::not_found;
    key = r->layout;
  }
  return current_manifest(model, v, key, shard, bytes, final_bytes);
}

Status Registry::add_layout(const std::string& model, VersionId v, const std::string& key,
                            const std::vector<std::string>& manifests,
                            const std::vector<std::string>& layouts) {
  std::lock_guard lk(mu_);
  auto& m = ms(model);
  auto vit = m.versions.find(v);
  if (vit == m.versions.end()) return Status::version_unavailable;
  auto lit = vit->second.by_layout.find(key);
  if (lit != vit->second.by_layout.end())
    return lit->second.manifests == manifests ? Status::ok : Status::manifest_conflict;
  LayoutInfo li{static_cast<std::uint32_t>(manifests.size()), manifests, layouts};
  li.layouts.resize(manifests.size());
  vit->second.by_layout.emplace(key, std::move(li));
  trace("layout_added", {{"model", model}, {"v", n2s(v)}, {"shards", n2s(manifests.size())}});
  return Status::ok;
}

// ---------------------------------------------------------------- unpublish

Status Registry::unpublish(const std::string& model, const std::string& replica,
                           OpOutcome* out) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (!r) return Status::not_found;
  if (r->txn) return Status::invalid_state;
  if (r->life != Life::published || !r->version) {
    r->last = {true, Status::invalid_state, std::nullopt, false, {}};
    if (out) *out = r->last;
    return Status::invalid_state;
  }
  Txn t;
  t.kind = OpKind::unpublish;
  t.order = ++order_;
  t.was_visible = r->visible;
  t.resolved = true;
  r->visible = false;  // no new readers from here on
  r->txn = t;
  r->last = {};
  auto& m = ms(model);
  const bool offload = needs_offload(m, *r, *r->version);
  trace("unpublish_start", {{"model", model}, {"replica", replica},
                            {"v", n2s(*r->version)}, {"offload_first", offload ? "1" : "0"},
                            {"serving", n2s(r->serving)}});
  if (offload) request_offload(*r, *r->txn, *r->version);
  try_settle(*r);
  if (out) *out = r->last;
  cv_.notify_all();
  return Status::ok;
}

// ---------------------------------------------------------------- replicate

Status Registry::replicate(const std::string& model, const std::string& replica,
                           const VersionSpec& spec, OpOutcome* out) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (!r) return Status::not_found;
  if (r->txn) return Status::invalid_state;
  Txn t;
  t.kind = OpKind::replicate;
  t.order = ++order_;
  t.spec = spec;
  r->txn = t;
  r->last = {};
  start_replicate(*r);
  if (out) *out = r->last;
  cv_.notify_all();
  return Status::ok;
}

void Registry::start_replicate(Rep& r) {
  Txn& t = *r.txn;
  if (r.life != Life::registered) return finish_op(r, Status::invalid_state);
  auto& m = ms(r.model);
  auto target = resolve_version(t.spec, available(m, r.dc));
  if (!target) {
    if (!t.blocked) {
      t.blocked = true;
      trace("replicate_blocked", {{"model", r.model}, {"replica", r.name},
                                  {"spec", t.spec.to_string()}});
    }
    return;  // parked; wake_blocked retries
  }
  if (!servable(m, *target, r)) return finish_op(r, Status::invalid_argument);
  Rep* src = pick_source(m, *target, r);
  if (!src) return finish_op(r, Status::version_unavailable);
  t.blocked = false;
  t.resolved = true;
  t.target = target;
  t.source = src->name;
  src->serving++;
  src->last_assigned = ++tick_;
  trace("replicate_resolved", {{"model", r.model}, {"replica", r.name},
                               {"v", n2s(*target)}, {"src", src->name}});
  try_settle(r);
}

// ------------------------------------------------------------------- update

Status Registry::update(const std::string& model, const std::string& replica,
                        const VersionSpec& spec, std::optional<VersionId> current,
                        OpOutcome* out) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (!r) return Status::not_found;
  if (r->txn) return Status::invalid_state;
  Txn t;
  t.kind = OpKind::update;
  t.order = ++order_;
  t.spec = spec;
  t.current = current;
  r->txn = t;
  r->last = {};
  start_update(*r);
  if (out) *out = r->last;
  cv_.notify_all();
  return Status::ok;
}

void Registry::start_update(Rep& r) {
  Txn& t = *r.txn;
  if (r.life != Life::registered && r.life != Life::published)
    return finish_op(r, Status::invalid_state);
  auto& m = ms(r.model);
  auto target = resolve_version(t.spec, available(m, r.dc));
  std::optional<VersionId> current = r.version ? r.version : t.current;
  auto no_change = [&] {
    trace("update_no_change",
          {{"model", r.model}, {"replica", r.name},
           {"current", current ? n2s(*current) : "none"},
           {"target", target ? n2s(*target) : "none"}});
    t.resolved = true;
    t.changed = false;
    r.last = {true, Status::ok, current, false, {}};
    r.txn.reset();
  };
  if (!target || (current && *target == *current)) return no_change();
  if (!servable(m, *target, r)) return finish_op(r, Status::invalid_argument);
  Rep* src = pick_source(m, *target, r);
  if (!src) return no_change();
  // A change over the cross-datacenter link with host seeding on: fill a
  // seed buffer in the background and stay on the current version until it
  // lands (server_core.cpp:915-970).
  if (src->dc != r.dc && r.offload_seed) {
    Rep* seed = find_seed(r);
    if (seed && seed->life == Life::replicating) {
      if (seed->version && *seed->version >= *target) return no_change();  // already under way
      void_replication(*seed, "stale_seed");  // it chases a stale version: restart
      release_offload(*seed);
    } else if (seed) {
      release_offload(*seed);  // a completed seed of another version: drop and refill
    }
    const std::string name = r.name + "+seed@" + n2s(*target);
    if (m.reps.count(name)) return no_change();  // the same buffer still draining
    auto rec = std::make_unique<Rep>();
    rec->model = r.model;
    rec->name = name;
    rec->kind = Kind::offload;
    rec->seed = true;
    rec->owner = r.name;
    rec->num_shards = r.num_shards;
    rec->dc = r.dc;
    rec->layout = r.layout;
    rec->endpoints = r.endpoints;
    rec->life = Life::replicating;
    rec->version = target;
    rec->offload_v = *target;
    rec->source = src->name;
    rec->seeding = true;
    rec->shards.assign(r.num_shards, {});
    src->serving++;
    src->last_assigned = ++tick_;
    SeedStart ss;
    ss.version = *target;
    ss.source = src->name;
    for (std::uint32_t s = 0; s < r.num_shards; ++s) {
      Assignment a = make_assignment(m, *src, *target, s, *rec);
      a.seeding = true;
      ss.assignments.push_back(std::move(a));
    }
    m.reps.emplace(name, std::move(rec));
    trace("seed_start", {{"model", r.model}, {"replica", r.name}, {"v", n2s(*target)},
                         {"src", src->name}});
    no_change();
    r.last.seed = std::move(ss);
    return;
  }
  t.resolved = true;
  t.changed = true;
  t.target = target;
  t.source = src->name;
  src->serving++;
  src->last_assigned = ++tick_;
  t.was_visible = r.visible;
  if (r.life == Life::published && r.version) r.visible = false;
  const bool offload = r.life == Life::published && r.version && needs_offload(m, r, *r.version);
  trace("update_change", {{"model", r.model}, {"replica", r.name},
                          {"from", current ? n2s(*current) : "none"},
                          {"to", n2s(*target)}, {"src", src->name},
                          {"offload_first", offload ? "1" : "0"}, {"serving", n2s(r.serving)}});
  if (offload) request_offload(r, t, *r.version);
  try_settle(r);
}

// ------------------------------------------------------------------- settle

void Registry::try_settle(Rep& r) {
  if (!r.txn) return;
  Txn& t = *r.txn;
  if (!t.resolved || t.settled || t.blocked) return;
  if (t.offload_needed && !t.offload_done) return;  // the client parks the version first
  bool needs_drain =
      t.kind == OpKind::unpublish || (t.kind == OpKind::update && t.changed);
  if (needs_drain && r.serving > 0) return;  // wait for readers to finish
  apply_settle(r);
}

Registry::Rep* Registry::settle_source(Rep& r, Txn& t) {
  auto& m = ms(r.model);
  auto sit = m.reps.find(t.source);
  if (sit != m.reps.end()) {
    Rep* c = sit->second.get();
    if (c->life != Life::failed && still_good(*c, r, *t.target)) return c;
    if (c->serving > 0) {
      c->serving--;
      check_drain(*c);
    }
  }
  t.source.clear();
  Rep* fresh = pick_source(m, *t.target, r);
  if (fresh) {
    t.source = fresh->name;
    fresh->serving++;
    fresh->last_assigned = ++tick_;
    trace("source_repick", {{"model", r.model}, {"replica", r.name},
                            {"v", n2s(*t.target)}, {"src", fresh->name}});
  }
  return fresh;
}

void Registry::apply_settle(Rep& r) {
  Txn& t = *r.txn;
  auto& m = ms(r.model);
  switch (t.kind) {
    case OpKind::unpublish: {
      VersionId v = *r.version;
      r.life = Life::registered;
      r.version.reset();
      for (auto& s : r.shards) s = {};
      trace("unpublish_ack", {{"model", r.model}, {"replica", r.name}, {"v", n2s(v)}});
      prune_version(m, v);
      r.last = {true, Status::ok, std::nullopt, false, {}};
      r.txn.reset();
      eval_offload_releases(r.model);
      return;
    }
    case OpKind::replicate:
    case OpKind::update: {
      bool is_update = t.kind == OpKind::update;
      Rep* src = settle_source(r, t);
      if (!src) {
        if (!is_update) {
          t.resolved = false;
          t.blocked = true;
          t.target.reset();
          trace("replicate_blocked", {{"model", r.model}, {"replica", r.name},
                                      {"spec", t.spec.to_string()}});
          return;
        }
        if (t.was_visible && r.life == Life::published) r.visible = true;
        trace("update_rescinded", {{"model", r.model}, {"replica", r.name}});
        r.last = {true, Status::ok, r.version, false, {}};
        r.txn.reset();
        return;
      }
      std::optional<VersionId> old = r.version;
      r.life = Life::replicating;
      r.visible = false;
      r.version = t.target;
      r.source = t.source;
      r.seeding = src->dc != r.dc;
      for (auto& s : r.shards) s = {};
      trace("assign", {{"model", r.model}, {"replica", r.name},
                       {"v", n2s(*t.target)}, {"src", t.source},
                       {"cross_dc", src->dc != r.dc ? "1" : "0"},
                       {"src_serving", n2s(src->serving)}});
      if (src->layout != r.layout && !terminal_layout(r.layout) &&
          r.derived_manifests.size() == r.num_shards) {
        // a resharding fill: its slicing becomes a layout of the version
        auto& vi = m.versions[*t.target];
        if (!vi.by_layout.count(r.layout)) {
          LayoutInfo li{r.num_shards, r.derived_manifests, r.derived_layouts};
          li.layouts.resize(r.num_shards);
          vi.by_layout.emplace(r.layout, std::move(li));
          trace("layout_added", {{"model", r.model}, {"v", n2s(*t.target)}, {"replica", r.name}});
        }
      }
      if (is_update && old && *old != *t.target) prune_version(m, *old);
      settle_ok(r);
      return;
    }
    default:
      return;
  }
}

void Registry::settle_ok(Rep& r) {
  Txn& t = *r.txn;
  auto& m = ms(r.model);
  OpOutcome o;
  o.done = true;
  o.status = Status::ok;
  o.version = t.target;
  o.changed = t.kind == OpKind::update;
  auto sit = m.reps.find(t.source);
  if (sit == m.reps.end()) {
    o.status = Status::version_unavailable;
  } else {
    for (std::uint32_t s = 0; s < r.num_shards; ++s) {
      Assignment a = make_assignment(m, *sit->second, *t.target, s, r);
      a.seeding = r.seeding;
      const Rep& src = *sit->second;
      a.local_seed_consume = src.kind == Kind::offload && src.seed && src.owner == r.name;
      o.assignments.push_back(std::move(a));
    }
  }
  r.last = std::move(o);
  r.txn.reset();
}

void Registry::finish_op(Rep& r, Status st) {
  r.last = {true, st, std::nullopt, false, {}};
  r.txn.reset();
}

void Registry::wake_blocked(const std::string& model) {
  auto& m = ms(model);
  std::vector<std::pair<std::uint64_t, std::string>> parked;
  for (auto& [name, r] : m.reps)
    if (r->txn && r->txn->blocked && r->txn->kind == OpKind::replicate)
      parked.emplace_back(r->txn->order, name);
  std::sort(parked.begin(), parked.end());
  for (auto& [order, name] : parked) {
    auto it = m.reps.find(name);
    if (it == m.reps.end()) continue;
    Rep& r = *it->second;
    if (r.txn && r.txn->blocked && r.txn->kind == OpKind::replicate)
      start_replicate(r);
  }
}

// ----------------------------------------------------- progress / complete

void Registry::progress(const std::string& model, const std::string& replica,
                        std::uint32_t shard, std::uint64_t items, bool seed,
                        VersionId seed_version) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (r && seed) r = find_seed(*r);
  if (r && seed && seed_version && r->offload_v != seed_version) return;
  if (!r || r->life != Life::replicating || shard >= r->num_shards) return;
  auto& sx = r->shards[shard];
  if (items > sx.progress) sx.progress = items;
}

void Registry::complete(const std::string& model, const std::string& replica,
                        std::uint32_t shard, Status outcome, bool seed,
                        VersionId seed_version) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (r && seed) r = find_seed(*r);
  if (r && seed && seed_version && r->offload_v != seed_version) return;
  if (!r || r->life != Life::replicating || shard >= r->num_shards) return;
  if (!ok(outcome)) {
    trace("shard_failed", {{"model", model}, {"replica", r->name},
                           {"shard", n2s(shard)}, {"status", status_name(outcome)}});
    if (r->kind == Kind::offload && r->seed) {
      void_replication(*r, "seed_failed");
      release_offload(*r);
    } else {
      void_replication(*r, status_name(outcome));
    }
    cv_.notify_all();
    return;
  }
  r->shards[shard].complete = true;
  trace("shard_complete", {{"model", model}, {"replica", r->name}, {"shard", n2s(shard)}});
  if (r->complete_all()) finish_replication(*r);
  cv_.notify_all();
}

void Registry::finish_replication(Rep& r) {
  std::string consumed_seed;  // the owner consumed its own seed buffer
  if (Rep* src = find(r.model, r.source);
      src && src->kind == Kind::offload && src->seed && src->owner == r.name)
    consumed_seed = src->name;
  release_source(r);
  r.life = Life::published;
  r.visible = true;
  bool was_seeding = r.seeding;
  r.seeding = false;
  trace("replica_complete", {{"model", r.model}, {"replica", r.name},
                             {"v", n2s(*r.version)}, {"seeded", was_seeding ? "1" : "0"}});
  if (!consumed_seed.empty()) {
    if (Rep* sd = find(r.model, consumed_seed)) {
      trace("seed_consumed", {{"model", r.model}, {"replica", r.name}});
      release_offload(*sd);
    }
  }
  wake_blocked(r.model);
  eval_offload_releases(r.model);
}

void Registry::release_source(Rep& r) {
  if (r.source.empty()) return;
  Rep* src = find(r.model, r.source);
  r.source.clear();
  if (!src) return;
  if (src->serving > 0) src->serving--;
  check_drain(*src);
}

void Registry::check_drain(Rep& src) {
  if (src.serving > 0) return;
  if (src.kind == Kind::offload && src.releasing) return finish_offload_release(src);
  try_settle(src);
  if (src.life == Life::failed && !src.txn) {
    // nothing else to do; failed records linger until re-opened
  }
}

void Registry::void_replication(Rep& r, const std::string& reason) {
  if (r.life != Life::replicating) return;
  std::optional<VersionId> v = r.version;
  release_source(r);
  r.life = Life::registered;
  r.version.reset();
  r.seeding = false;
  for (auto& s : r.shards) s = {};
  trace("replica_voided", {{"model", r.model}, {"replica", r.name}, {"reason", reason}});
  if (v) prune_version(ms(r.model), *v);
}

void Registry::fail_replica(Rep& r, const std::string& reason) {
  if (r.life == Life::failed) return;
  std::optional<VersionId> v = r.version;
  trace("replica_failed", {{"model", r.model}, {"replica", r.name},
                           {"reason", reason}, {"was", life_name(r.life)}});
  release_source(r);
  r.life = Life::failed;
  r.visible = false;
  r.seeding = false;
  r.serving = 0;
  if (r.txn) finish_op(r, Status::group_aborted);
  if (v) prune_version(ms(r.model), *v);
}

void Registry::prune_version(ModelState& m, VersionId v) {
  for (const auto& [name, r] : m.reps)
    if (r->life != Life::failed && r->version == v) return;
  m.versions.erase(v);
}

// --------------------------------------------------------------- retention

Status Registry::set_retention(const std::string& model, const std::string& replica,
                               const std::set<std::uint64_t>& lags) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (!r || r->kind != Kind::worker) return Status::not_found;
  r->retain = lags;
  return Status::ok;
}

Status Registry::set_offload_seed(const std::string& model, const std::string& replica, bool on) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (!r || r->kind != Kind::worker) return Status::not_found;
  r->offload_seed = on;
  return Status::ok;
}

Registry::Rep* Registry::find_seed(const Rep& owner) {
  // the owner's live seed buffer: at most one not already draining
  for (auto& [name, r] : ms(owner.model).reps)
    if (r->kind == Kind::offload && r->seed && r->owner == owner.name && !r->releasing)
      return r.get();
  return nullptr;
}

std::set<VersionId> Registry::retained_versions(ModelState& m) {
  std::set<VersionId> out;
  if (!m.max_published) return out;
  const VersionId max = *m.max_published;
  for (const auto& [name, r] : m.reps)
    for (auto lag : r->retain)
      if (lag <= max) out.insert(max - lag);
  return out;
}

bool Registry::needs_offload(ModelState& m, const Rep& r, VersionId v) {
  if (r.kind != Kind::worker || !retained_versions(m).count(v)) return false;
  for (const auto& [name, other] : m.reps) {
    if (other.get() == &r) continue;
    if (other->visible && other->life == Life::published && other->version == v &&
        other->complete_all())
      return false;  // another durable copy exists
  }
  return true;
}

void Registry::request_offload(Rep& r, Txn& t, VersionId v) {
  t.offload_needed = true;
  t.offload_v = v;
  t.offload_endpoints.assign(r.num_shards, "");
  trace("offload_first", {{"model", r.model}, {"replica", r.name}, {"v", n2s(v)}});
  r.last.done = false;
  r.last.offload_first = v;
}

Status Registry::offload_confirm(const std::string& model, const std::string& replica,
                                 std::uint32_t shard, VersionId version, bool ok,
                                 const std::string& endpoint) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (!r) return Status::not_found;
  if (!r->txn || !r->txn->offload_needed || r->txn->offload_v != version ||
      shard >= r->num_shards)
    return Status::invalid_state;
  Txn& t = *r->txn;
  if (t.offload_done) return Status::ok;
  if (!ok) {
    // Host memory unavailable: the op fails, the replica stays published and
    // visible; nothing was given up (server_core.cpp:1404-1421).
    trace("offload_failed", {{"model", model}, {"replica", replica}, {"v", n2s(version)}});
    if (t.was_visible && r->life == Life::published) r->visible = true;
    if (!t.source.empty()) {
      Rep* s = find(model, t.source);
      if (s && s->serving > 0) {
        s->serving--;
        check_drain(*s);
      }
    }
    finish_op(*r, Status::offload_failed);
    cv_.notify_all();
    return Status::ok;
  }
  t.offload_confirmed.insert(shard);
  t.offload_endpoints[shard] = endpoint;
  trace("offload_confirmed", {{"model", model}, {"replica", replica}, {"shard", n2s(shard)},
                              {"v", n2s(version)}});
  if (t.offload_confirmed.size() == r->num_shards) {
    t.offload_done = true;
    r->last.offload_first.reset();
    create_offload_replica(*r, version, t.offload_endpoints);
    try_settle(*r);
  }
  cv_.notify_all();
  return Status::ok;
}

void Registry::create_offload_replica(Rep& owner, VersionId v,
                                      const std::vector<std::string>& endpoints) {
  auto& m = ms(owner.model);
  const std::string name = owner.name + "+offload@" + n2s(v);
  auto it = m.reps.find(name);
  if (it != m.reps.end()) {
    // mid-drain toward release when it became needed again: keep it
    Rep& old = *it->second;
    old.releasing = false;
    old.visible = true;
    old.endpoints = endpoints;
    trace("offload_reused", {{"model", owner.model}, {"replica", name}});
    wake_blocked(owner.model);
    return;
  }
  auto rec = std::make_unique<Rep>();
  rec->kind = Kind::offload;
  rec->owner = owner.name;
  rec->model = owner.model;
  rec->name = name;
  rec->dc = owner.dc;
  rec->layout = owner.layout;
  rec->num_shards = owner.num_shards;
  rec->endpoints = endpoints;
  rec->life = Life::published;
  rec->visible = true;
  rec->version = v;
  rec->offload_v = v;
  rec->shards.assign(owner.num_shards, ShardState{0, true});
  m.reps.emplace(name, std::move(rec));
  trace("offload_replica", {{"model", owner.model}, {"replica", name}, {"v", n2s(v)},
                            {"purpose", "retention"}});
  wake_blocked(owner.model);
}

void Registry::eval_offload_releases(const std::string& model) {
  auto& m = ms(model);
  const auto retained = retained_versions(m);
  std::vector<Rep*> drop;
  for (auto& [name, r] : m.reps) {
    // retention buffers only: a seed is released when its owner consumes it
    if (r->kind != Kind::offload || r->seed || r->releasing || r->life != Life::published) continue;
    const VersionId v = *r->version;
    bool replaced = false;
    for (const auto& [oname, other] : m.reps)
      if (other->kind == Kind::worker && other->visible && other->life == Life::published &&
          other->version == v && other->complete_all())
        replaced = true;
    if (replaced || !retained.count(v)) drop.push_back(r.get());
  }
  for (Rep* r : drop) release_offload(*r);
}

void Registry::release_offload(Rep& off) {
  if (off.releasing) return;
  off.releasing = true;
  off.visible = false;
  trace("offload_release_start", {{"model", off.model}, {"replica", off.name},
                                  {"v", n2s(off.offload_v)},
                                  {"serving", n2s(off.serving)}});
  if (off.serving == 0) finish_offload_release(off);
}

void Registry::finish_offload_release(Rep& off) {
  const std::string model = off.model, name = off.name;
  releases_[model].push_back({off.owner, off.offload_v, off.seed});
  trace("offload_released", {{"model", model}, {"replica", name}});
  auto& m = ms(model);
  const VersionId v = off.offload_v;
  m.reps.erase(name);
  prune_version(m, v);
}

std::vector<OffloadRelease> Registry::take_releases(const std::string& model,
                                                    const std::string& owner) {
  std::lock_guard lk(mu_);
  std::vector<OffloadRelease> out, keep;
  for (auto& d : releases_[model]) (d.owner == owner ? out : keep).push_back(d);
  releases_[model] = std::move(keep);
  return out;
}

Result<Assignment> Registry::failure_report(const std::string& model,
                                            const std::string& replica,
                                            std::uint32_t shard,
                                            const std::string& failed,
                                            int reason) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (!r) return Status::not_found;
  trace("failure_report", {{"model", model}, {"replica", replica},
                           {"shard", n2s(shard)}, {"failed", failed},
                           {"reason", reason == 0 ? "timeout" : "checksum"}});
  if (r->life != Life::replicating) return Status::invalid_state;
  auto& m = ms(model);
  // A timeout is evidence the peer is gone; checksum corruption is not.
  if (reason == 0 && failed == r->source) {
    Rep* f = find(model, failed);
    if (f && f->life != Life::failed) fail_replica(*f, "reported_timeout");
  }
  if (r->life != Life::replicating) return Status::invalid_state;
  VersionId v = *r->version;
  if (r->source == failed || r->source.empty()) {
    if (reason == 1 && !r->source.empty()) {
      Rep* s = find(model, r->source);
      if (s && s->serving > 0) s->serving--;
    }
    r->source.clear();
    Rep* src = pick_source(m, v, *r);
    if (!src) {
      trace("reassign_failed", {{"model", model}, {"replica", replica}, {"v", n2s(v)}});
      void_replication(*r, "no_source");
      cv_.notify_all();
      return Status::version_unavailable;
    }
    r->source = src->name;
    src->serving++;
    src->last_assigned = ++tick_;
    if (src->dc != r->dc) r->seeding = true;
    trace("reassign", {{"model", model}, {"replica", replica}, {"v", n2s(v)},
                       {"src", src->name}});
  }
  Rep* s = find(model, r->source);
  if (!s) return Status::version_unavailable;
  Assignment a = make_assignment(m, *s, v, shard, *r);
  a.seeding = r->seeding;
  cv_.notify_all();
  return a;
}

// ---------------------------------------------------------------- queries

Result<Assignment> Registry::locate(const std::string& model, const std::string& replica,
                                   const VersionSpec& spec, std::uint32_t shard) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (!r) return Status::not_found;
  if (shard >= r->num_shards) return Status::invalid_argument;
  auto& m = ms(model);
  auto target = resolve_version(spec, available(m, r->dc));
  if (!target) return Status::version_unavailable;
  if (!servable(m, *target, *r)) return Status::invalid_argument;
  Rep* src = pick_source(m, *target, *r);
  if (!src) return Status::version_unavailable;
  return make_assignment(m, *src, *target, shard, *r);
}

Result<Assignment> Registry::current_assignment(const std::string& model,
                                                const std::string& replica,
                                                std::uint32_t shard) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (!r) return Status::not_found;
  if (r->life != Life::replicating || !r->version || shard >= r->num_shards)
    return Status::invalid_state;
  Rep* s = find(model, r->source);
  if (!s) return Status::version_unavailable;
  Assignment a = make_assignment(ms(model), *s, *r->version, shard, *r);
  a.seeding = r->seeding;
  return a;
}

OpOutcome Registry::op_result(const std::string& model, const std::string& replica) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (!r) return {true, Status::not_found, std::nullopt, false, {}};
  return r->last;
}

OpOutcome Registry::wait_op(const std::string& model, const std::string& replica,
                            double timeout_s) {
  std::unique_lock lk(mu_);
  auto deadline = std::chrono::steady_clock::now() +
                  std::chrono::duration<double>(timeout_s);
  for (;;) {
    Rep* r = find(model, replica);
    if (!r) return {true, Status::not_found, std::nullopt, false, {}};
    if (r->last.done) return r->last;
    if (cv_.wait_until(lk, deadline) == std::cv_status::timeout) {
      r = find(model, replica);
      if (r && r->last.done) return r->last;
      return {false, Status::timeout, std::nullopt, false, {}};
    }
  }
}

std::map<VersionId, std::set<std::string>> Registry::listing(const std::string& model) {
  std::lock_guard lk(mu_);
  std::map<VersionId, std::set<std::string>> out;
  auto mit = models_.find(model);
  if (mit == models_.end()) return out;
  for (const auto& [name, r] : mit->second.reps)
    if (r->visible && r->life == Life::published && r->version && r->complete_all())
      out[*r->version].insert(name);
  return out;
}

std::optional<ReplicaView> Registry::view(const std::string& model,
                                          const std::string& replica) {
  std::lock_guard lk(mu_);
  Rep* r = find(model, replica);
  if (!r) return std::nullopt;
  ReplicaView v;
  v.kind = r->kind == Kind::offload ? "offload" : "worker";
  v.lifecycle = life_name(r->life);
  v.version = r->version;
  v.serving = r->serving;
  v.visible = r->visible;
  v.seeding = r->seeding;
  v.source = r->source;
  std::uint64_t mp = ~0ull;
  for (const auto& s : r->shards) mp = std::min(mp, s.progress);
  v.min_progress = r->shards.empty() ? 0 : mp;
  return v;
}

std::vector<TraceLine> Registry::trace() {
  std::lock_guard lk(mu_);
  return trace_;
}

std::string Registry::trace_text() {
  std::lock_guard lk(mu_);
  std::string out;
  for (const auto& t : trace_) {
    out += t.format();
    out += '\n';
  }
  return out;
}

}  // namespace rsb
