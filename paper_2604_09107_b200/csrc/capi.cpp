// extern "C" boundary of libros_b200.so (declared in include/ros_b200.h).
#include "../../include/ros_b200.h"

#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <set>
#include <vector>

#include "client.hpp"
#include "device.hpp"
#include "registry.hpp"
#include "stream.hpp"

struct rs_cluster {
  rsb::Registry reg;
  rsb::ServeRegistry serves;
  std::unique_ptr<rsb::StreamServer> stream;  // off-box data plane (rs_cluster_listen)
  explicit rs_cluster(rsb::Registry::Config c) : reg(c) {}
};

struct rs_handle {
  rs_cluster* cluster = nullptr;
  std::unique_ptr<rsb::Client> client;
  std::vector<std::uint32_t> pending;  // split-phase fill: shards still to land
};

namespace {

int st(rsb::Status s) { return static_cast<int>(s); }

int put_bytes(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (buf && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
  else if (buf && cap < s.size()) return st(rsb::Status::invalid_argument);
  return 0;
}

void fill_assignment(const rsb::Assignment& a, rs_assignment* out) {
  std::memset(out, 0, sizeof(*out));
  out->version = a.version;
  std::strncpy(out->source_replica, a.source_replica.c_str(), sizeof(out->source_replica) - 1);
  std::strncpy(out->source_endpoint, a.source_endpoint.c_str(), sizeof(out->source_endpoint) - 1);
  out->source_complete = a.source_complete;
  out->cross_dc = a.cross_dc;
  out->seeding = a.seeding;
  out->local_seed_consume = a.local_seed_consume;
}

rsb::ClientConfig to_cfg(const rs_config* c) {
  rsb::ClientConfig cfg;
  if (!c) return cfg;
  if (c->chunk_bytes) cfg.chunk_bytes = c->chunk_bytes;
  if (c->tiny_threshold) cfg.limits.tiny_threshold = c->tiny_threshold;
  if (c->group_target) cfg.limits.group_target = c->group_target;
  cfg.pipeline = c->pipeline != 0;
  cfg.checksum_retries = c->checksum_retries;
  if (c->pull_timeout_s > 0) cfg.pull_timeout_s = c->pull_timeout_s;
  if (c->datacenter[0]) cfg.dc = std::string(c->datacenter, strnlen(c->datacenter, 32));
  if (c->reshard_align) cfg.reshard_align = c->reshard_align;
  cfg.grid_sms = c->grid_sms;
  cfg.early_publish = c->early_publish != 0;
  cfg.offload_seed = c->offload_seed != 0;
  return cfg;
}

bool parse_spec(const char* spec, rsb::VersionSpec* out) {
  if (!spec) return false;
  auto r = rsb::VersionSpec::parse(spec);
  if (!r) return false;
  *out = *r;
  return true;
}

// Runs `fn` with the device that owns `ptr` current (kernels must launch on
// the device whose memory they touch).
template <class F>
int on_ptr_device(const void* ptr, F fn) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess || a.type != cudaMemoryTypeDevice) {
    cudaGetLastError();
    return st(rsb::Status::invalid_argument);
  }
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != a.device) cudaSetDevice(a.device);
  cudaError_t e = fn();
  if (prev != a.device) cudaSetDevice(prev);
  return e == cudaSuccess ? 0 : st(rsb::Status::transfer_failed);
}

}  // namespace

extern "C" {

int rs_abi_version(void) { return RS_ABI_VERSION; }

const char* rs_status_name(int status) {
  return rsb::status_name(static_cast<rsb::Status>(status));
}

void rs_config_default(rs_config* cfg) {
  std::memset(cfg, 0, sizeof(*cfg));
  rsb::ClientConfig d;
  cfg->chunk_bytes = d.chunk_bytes;
  cfg->tiny_threshold = d.limits.tiny_threshold;
  cfg->group_target = d.limits.group_target;
  cfg->pipeline = d.pipeline;
  cfg->checksum_retries = d.checksum_retries;
  cfg->pull_timeout_s = d.pull_timeout_s;
  std::strncpy(cfg->datacenter, d.dc.c_str(), sizeof(cfg->datacenter) - 1);
  cfg->reshard_align = d.reshard_align;
  cfg->grid_sms = d.grid_sms;
  cfg->early_publish = d.early_publish ? 1 : 0;
  cfg->offload_seed = d.offload_seed ? 1 : 0;
}

int rs_cluster_create(int pipeline, int smart_skipping, rs_cluster** out) {
  if (!out) return st(rsb::Status::invalid_argument);
  rsb::Registry::Config c;
  c.pipeline = pipeline != 0;
  c.smart_skipping = smart_skipping != 0;
  *out = new rs_cluster(c);
  return 0;
}

void rs_cluster_destroy(rs_cluster* c) { delete c; }

int rs_cluster_trace(rs_cluster* c, char* buf, size_t cap, size_t* len) {
  if (!c) return st(rsb::Status::invalid_argument);
  return put_bytes(c->reg.trace_text(), buf, cap, len);
}

int rs_cluster_listing(rs_cluster* c, const char* model, char* buf, size_t cap, size_t* len) {
  if (!c || !model) return st(rsb::Status::invalid_argument);
  std::string out;
  for (const auto& [v, reps] : c->reg.listing(model)) {
    if (!out.empty()) out += ';';
    out += std::to_string(v) + ':';
    bool first = true;
    for (const auto& r : reps) {
      if (!first) out += ',';
      out += r;
      first = false;
    }
  }
  return put_bytes(out, buf, cap, len);
}

int rs_cluster_view(rs_cluster* c, const char* model, const char* replica, char* lifecycle,
                    uint64_t* version, uint32_t* serving, int* visible) {
  if (!c || !model || !replica) return st(rsb::Status::invalid_argument);
  auto v = c->reg.view(model, replica);
  if (!v) return st(rsb::Status::not_found);
  if (lifecycle) std::strncpy(lifecycle, v->lifecycle.c_str(), 15), lifecycle[15] = 0;
  if (version) *version = v->version.value_or(0);
  if (serving) *serving = v->serving;
  if (visible) *visible = v->visible;
  return 0;
}

int rs_cluster_seeding(rs_cluster* c, const char* model, const char* replica, int* seeding) {
  if (!c || !model || !replica || !seeding) return st(rsb::Status::invalid_argument);
  auto v = c->reg.view(model, replica);
  if (!v) return st(rsb::Status::not_found);
  *seeding = v->seeding;
  return 0;
}

int rs_cluster_progress(rs_cluster* c, const char* model, const char* replica,
                        uint64_t* min_progress) {
  if (!c || !model || !replica || !min_progress) return st(rsb::Status::invalid_argument);
  auto v = c->reg.view(model, replica);
  if (!v) return st(rsb::Status::not_found);
  *min_progress = v->min_progress;
  return 0;
}

int rs_cluster_source(rs_cluster* c, const char* model, const char* replica, char* buf,
                      size_t cap, size_t* len) {
  if (!c || !model || !replica) return st(rsb::Status::invalid_argument);
  auto v = c->reg.view(model, replica);
  if (!v) return st(rsb::Status::not_found);
  return put_bytes(v->source, buf, cap, len);
}

int rs_cluster_set_silent(rs_cluster* c, const char* model, const char* replica, int silent) {
  if (!c || !model || !replica) return st(rsb::Status::invalid_argument);
  c->serves.set_silent(model, replica, silent != 0);
  return 0;
}

// ------------------------------------------------------------ ClientCore

int rs_open(rs_cluster* c, const char* model, const char* replica, uint32_t num_shards,
            const rs_config* cfg, rs_handle** out) {
  if (!c || !model || !replica || !out || num_shards == 0 || !*model || !*replica)
    return st(rsb::Status::invalid_argument);
  auto* h = new rs_handle;
  h->cluster = c;
  h->client = std::make_unique<rsb::Client>(&c->reg, &c->serves, model, replica, num_shards,
                                            to_cfg(cfg));
  *out = h;
  return 0;
}

int rs_register(rs_handle* h, uint32_t shard, const char* name, void* dev_ptr, uint64_t bytes) {
  if (!h || !name) return st(rsb::Status::invalid_argument);
  return st(h->client->register_tensor(shard, name, dev_ptr, bytes));
}

int rs_register_slice(rs_handle* h, uint32_t shard, const char* name, void* dev_ptr,
                      uint64_t bytes, uint64_t rows, uint64_t row_bytes, uint64_t r0, uint64_t nr,
                      uint64_t c0, uint64_t nc) {
  if (!h || !name || rows == 0) return st(rsb::Status::invalid_argument);
  rsb::Geometry g{rows, row_bytes, r0, nr, c0, nc};
  return st(h->client->register_tensor(shard, name, dev_ptr, bytes, g));
}

int rs_register_cast(rs_handle* h, uint32_t shard, const char* name, void* dev_ptr,
                     uint64_t bytes, uint64_t rows, uint64_t row_bytes, uint64_t r0, uint64_t nr,
                     uint64_t c0, uint64_t nc) {
  if (!h || !name) return st(rsb::Status::invalid_argument);
  rsb::Geometry g{rows, row_bytes, r0, nr, c0, nc};
  if (rows == 0) g = {};
  return st(h->client->register_tensor(shard, name, dev_ptr, bytes, g, true));
}

uint32_t rs_chunk_len_for(uint64_t row_bytes, uint64_t nc, uint64_t chunk_bytes, uint32_t align) {
  rsb::Geometry g{1, row_bytes, 0, 1, 0, nc};
  if (row_bytes == 0) g.rows = 0;
  return rsb::chunk_len_for(g, chunk_bytes, align);
}

int rs_shard_local(rs_handle* h, uint32_t shard) {
  return h && h->client->is_local(shard) ? 1 : 0;
}

int rs_shard_hash(rs_handle* h, uint32_t shard, uint64_t* hash, int* geometry, int* cast) {
  if (!h || shard >= h->client->num_shards()) return st(rsb::Status::invalid_argument);
  const auto sh = h->client->shard_hash(shard);
  if (hash) *hash = sh.hash;
  if (geometry) *geometry = sh.geometry ? 1 : 0;
  if (cast) *cast = sh.cast ? 1 : 0;
  return 0;
}

int rs_combine_layout_key(uint32_t n, const uint64_t* hashes, const int* geometry, const int* cast,
                          char* buf, size_t cap, size_t* len) {
  if (n && (!hashes || !geometry || !cast)) return st(rsb::Status::invalid_argument);
  std::vector<rsb::Client::ShardHash> hs(n);
  for (uint32_t i = 0; i < n; ++i) hs[i] = {hashes[i], geometry[i] != 0, cast[i] != 0};
  return put_bytes(rsb::Client::combine_layout_key(hs), buf, cap, len);
}

int rs_layout_key(rs_handle* h, char* buf, size_t cap, size_t* len) {
  if (!h) return st(rsb::Status::invalid_argument);
  return put_bytes(h->client->layout_key(), buf, cap, len);
}

int rs_layout(rs_handle* h, uint32_t shard, char* buf, size_t cap, size_t* len) {
  if (!h) return st(rsb::Status::invalid_argument);
  auto m = h->client->layout_bytes(shard);
  if (!m) return st(m.status());
  return put_bytes(*m, buf, cap, len);
}

int rs_transfer_derived(rs_handle* h) {
  if (!h) return 0;
  std::vector<std::string> m, l;
  return h->client->derived_layout(&m, &l) ? 1 : 0;
}

int rs_set_endpoint(rs_handle* h, uint32_t shard, const char* endpoint) {
  if (!h || !endpoint || shard >= h->client->num_shards()) return st(rsb::Status::invalid_argument);
  h->client->set_shard_endpoint(shard, endpoint);
  return 0;
}

int rs_set_stream(rs_handle* h, uint32_t shard, void* cuda_stream) {
  if (!h || shard >= h->client->num_shards()) return st(rsb::Status::invalid_argument);
  h->client->set_stream(shard, static_cast<cudaStream_t>(cuda_stream));
  return 0;
}

int rs_publish_pending(rs_handle* h) { return h && h->client->publish_pending() ? 1 : 0; }

int rs_set_early_publish(rs_handle* h, int on) {
  if (!h) return st(rsb::Status::invalid_argument);
  h->client->set_early_publish(on != 0);
  return 0;
}

int rs_publish_finalize(rs_handle* h, double wait_s) {
  if (!h) return st(rsb::Status::invalid_argument);
  return st(h->client->finalize_publish(wait_s));
}

int rs_publish(rs_handle* h, uint64_t version) {
  if (!h) return st(rsb::Status::invalid_argument);
  return st(h->client->publish(version));
}

int rs_unpublish(rs_handle* h) {
  if (!h) return st(rsb::Status::invalid_argument);
  return st(h->client->unpublish());
}

int rs_replicate(rs_handle* h, const char* spec, double wait_s, uint64_t* out_version) {
  rsb::VersionSpec vs;
  if (!h || !parse_spec(spec, &vs)) return st(rsb::Status::invalid_argument);
  rsb::VersionId v = 0;
  auto s = h->client->replicate(vs, &v, wait_s > 0 ? wait_s : 0.0);
  if (out_version) *out_version = v;
  return st(s);
}

int rs_pull(rs_handle* h, const char* spec, double wait_s, uint64_t* out_version) {
  return rs_replicate(h, spec, wait_s, out_version);
}

int rs_release(rs_handle* h, uint64_t version) {
  if (!h) return st(rsb::Status::invalid_argument);
  h->client->release_lane(version);
  return 0;
}

int rs_serve_state(rs_handle* h, uint32_t shard, uint64_t** digests, uint32_t** watermarks,
                   uint32_t* epoch, uint32_t* n_batches) {
  if (!h) return st(rsb::Status::invalid_argument);
  std::uint64_t d = 0, f = 0;
  std::uint32_t e = 0, nb = 0;
  if (auto s = h->client->serve_tables(shard, &d, &f, &e, &nb); !rsb::ok(s)) return st(s);
  if (digests) *digests = reinterpret_cast<uint64_t*>(d);
  if (watermarks) *watermarks = reinterpret_cast<uint32_t*>(f);
  if (epoch) *epoch = e;
  if (n_batches) *n_batches = nb;
  return 0;
}

int rs_update(rs_handle* h, const char* spec, double wait_s, int* changed, uint64_t* out_version) {
  rsb::VersionSpec vs;
  if (!h || !parse_spec(spec, &vs)) return st(rsb::Status::invalid_argument);
  bool ch = false;
  rsb::VersionId v = 0;
  auto s = h->client->update(vs, &ch, &v, wait_s > 0 ? wait_s : 0.0);
  if (changed) *changed = ch;
  if (out_version) *out_version = v;
  return st(s);
}

int rs_close(rs_handle* h) {
  if (!h) return st(rsb::Status::invalid_argument);
  auto s = h->client->close();
  delete h;
  return st(s);
}

int rs_cluster_set_topology(rs_cluster* c, uint32_t n, const char* const* endpoints,
                            const int32_t* cost) {
  if (!c || (n && (!endpoints || !cost))) return st(rsb::Status::invalid_argument);
  auto m = std::make_shared<std::map<std::pair<std::string, std::string>, int>>();
  for (uint32_t i = 0; i < n; ++i) {
    if (!endpoints[i]) return st(rsb::Status::invalid_argument);
    for (uint32_t j = 0; j < n; ++j) (*m)[{endpoints[i], endpoints[j]}] = cost[std::size_t(i) * n + j];
  }
  if (n == 0) {
    c->reg.set_topology(nullptr);
    return 0;
  }
  c->reg.set_topology([m](const std::string& reader, const std::string& source) {
    auto it = m->find({reader, source});
    return it == m->end() ? 0 : it->second;
  });
  return 0;
}

int rs_locate(rs_cluster* c, const char* model, const char* replica, const char* spec,
              uint32_t shard, rs_assignment* out) {
  rsb::VersionSpec vs;
  if (!c || !model || !replica || !out || !parse_spec(spec, &vs))
    return st(rsb::Status::invalid_argument);
  auto r = c->reg.locate(model, replica, vs, shard);
  if (!r) return st(r.status());
  fill_assignment(*r, out);
  return 0;
}

int rs_current_version(rs_handle* h, uint64_t* out) {
  if (!h || !out) return st(rsb::Status::invalid_argument);
  auto v = h->client->current_version();
  if (!v) return st(rsb::Status::not_found);
  *out = *v;
  return 0;
}

int rs_is_published(rs_handle* h) { return h && h->client->is_published() ? 1 : 0; }

int rs_stats_get(rs_handle* h, rs_stats* out) {
  if (!h || !out) return st(rsb::Status::invalid_argument);
  const auto& s = h->client->stats();
  out->bytes_pulled = s.bytes_pulled;
  out->bytes_pulled_cross_dc = s.bytes_pulled_cross_dc;
  out->bytes_copied_local = s.bytes_copied_local;
  out->items_verified = s.items_verified;
  out->checksum_failures = s.checksum_failures;
  out->failure_reports = s.failure_reports;
  out->failovers = s.failovers;
  out->last_pull_ms = s.last_pull_ms;
  out->last_publish_ms = s.last_publish_ms;
  out->last_pull_bytes = s.last_pull_bytes;
  out->last_pull_launches = s.last_pull_launches;
  out->h2d_bytes = s.h2d_bytes;
  out->d2h_bytes = s.d2h_bytes;
  out->fill_max_ms = s.fill_max_ms;
  out->fill_sum_ms = s.fill_sum_ms;
  out->fill_bytes = s.fill_bytes;
  out->kernel_launches = s.kernel_launches;
  return 0;
}

int rs_manifest_now(rs_handle* h, uint32_t shard, char* buf, size_t cap, size_t* len) {
  if (!h) return st(rsb::Status::invalid_argument);
  auto m = h->client->held_manifest(shard);
  if (!m) return st(m.status());
  return put_bytes(*m, buf, cap, len);
}

int rs_manifest(rs_handle* h, uint32_t shard, char* buf, size_t cap, size_t* len) {
  if (!h) return st(rsb::Status::invalid_argument);
  auto m = h->client->manifest_bytes(shard);
  if (!m) return st(m.status());
  return put_bytes(*m, buf, cap, len);
}

int rs_chunk_digests(rs_handle* h, uint32_t shard, uint64_t* out, size_t cap, size_t* n) {
  if (!h) return st(rsb::Status::invalid_argument);
  std::vector<std::uint64_t> d;
  auto s = h->client->chunk_digests(shard, &d);
  if (!rsb::ok(s)) return st(s);
  if (n) *n = d.size();
  if (out) {
    if (cap < d.size()) return st(rsb::Status::invalid_argument);
    std::memcpy(out, d.data(), d.size() * 8);
  }
  return 0;
}

int rs_invalidate(rs_handle* h) {
  if (!h) return st(rsb::Status::invalid_argument);
  h->client->invalidate();
  return 0;
}

// ------------------------------------------------------------ split phase

namespace {
std::vector<std::string> blobs(uint32_t n, const char* const* p, const size_t* lens) {
  std::vector<std::string> out;
  if (!p || !lens) return out;
  for (uint32_t i = 0; i < n; ++i) out.emplace_back(p[i] ? std::string(p[i], lens[i]) : std::string());
  return out;
}
}  // namespace

int rs_server_open(rs_cluster* c, const char* model, const char* replica, uint32_t num_shards,
                   const char* datacenter, const char* const* endpoints, const char* layout_key,
                   const char* const* derived_manifests, const size_t* dm_lens,
                   const char* const* derived_layouts, const size_t* dl_lens) {
  if (!c || !model || !replica || !endpoints) return st(rsb::Status::invalid_argument);
  std::vector<std::string> eps;
  for (uint32_t i = 0; i < num_shards; ++i) eps.emplace_back(endpoints[i] ? endpoints[i] : "");
  return st(c->reg.open(model, replica, num_shards, datacenter ? datacenter : "dc0", eps,
                        layout_key ? layout_key : "",
                        blobs(num_shards, derived_manifests, dm_lens),
                        blobs(num_shards, derived_layouts, dl_lens)));
}

int rs_derived(rs_handle* h, uint32_t shard, int what, char* buf, size_t cap, size_t* len) {
  if (!h || shard >= h->client->num_shards()) return st(rsb::Status::invalid_argument);
  std::vector<std::string> m, l;
  if (auto s = h->client->derived_blobs(&m, &l); !rsb::ok(s)) return st(s);
  const std::string empty;
  const std::string& b = m.empty() ? empty : (what == 0 ? m[shard] : l[shard]);
  return put_bytes(b, buf, cap, len);
}

int rs_server_publish(rs_cluster* c, const char* model, const char* replica, uint64_t version,
                      uint32_t num_shards, const char* const* manifests, const size_t* lens,
                      const char* const* layouts, const size_t* layout_lens) {
  if (!c || !model || !replica || !manifests || !lens) return st(rsb::Status::invalid_argument);
  rsb::OpOutcome o;
  auto s = c->reg.publish(model, replica, version, blobs(num_shards, manifests, lens), &o,
                          blobs(num_shards, layouts, layout_lens));
  return st(rsb::ok(s) ? o.status : s);
}

int rs_server_publish_provisional(rs_cluster* c, const char* model, const char* replica,
                                  uint64_t version, uint32_t num_shards,
                                  const char* const* manifests, const size_t* lens,
                                  const char* const* layouts, const size_t* layout_lens) {
  if (!c || !model || !replica || !manifests || !lens) return st(rsb::Status::invalid_argument);
  rsb::OpOutcome o;
  auto s = c->reg.publish(model, replica, version, blobs(num_shards, manifests, lens), &o,
                          blobs(num_shards, layouts, layout_lens), true);
  return st(rsb::ok(s) ? o.status : s);
}

int rs_server_finalize(rs_cluster* c, const char* model, const char* replica, uint64_t version,
                       uint32_t num_shards, const char* const* manifests, const size_t* lens) {
  if (!c || !model || !replica || !manifests || !lens) return st(rsb::Status::invalid_argument);
  return st(c->reg.finalize_manifests(model, replica, version, blobs(num_shards, manifests, lens)));
}

int rs_server_add_layout(rs_cluster* c, const char* model, uint64_t version, const char* layout_key,
                         uint32_t num_shards, const char* const* manifests, const size_t* lens,
                         const char* const* layouts, const size_t* layout_lens) {
  if (!c || !model || !layout_key || !manifests || !lens) return st(rsb::Status::invalid_argument);
  return st(c->reg.add_layout(model, version, layout_key, blobs(num_shards, manifests, lens),
                              blobs(num_shards, layouts, layout_lens)));
}

int rs_server_unpublish(rs_cluster* c, const char* model, const char* replica) {
  if (!c || !model || !replica) return st(rsb::Status::invalid_argument);
  return st(c->reg.unpublish(model, replica, nullptr));
}

int rs_server_replicate(rs_cluster* c, const char* model, const char* replica, const char* spec) {
  rsb::VersionSpec vs;
  if (!c || !model || !replica || !parse_spec(spec, &vs)) return st(rsb::Status::invalid_argument);
  return st(c->reg.replicate(model, replica, vs, nullptr));
}

int rs_server_update(rs_cluster* c, const char* model, const char* replica, const char* spec,
                     int has_current, uint64_t current) {
  rsb::VersionSpec vs;
  if (!c || !model || !replica || !parse_spec(spec, &vs)) return st(rsb::Status::invalid_argument);
  std::optional<rsb::VersionId> cur;
  if (has_current) cur = current;
  return st(c->reg.update(model, replica, vs, cur, nullptr));
}

int rs_server_result(rs_cluster* c, const char* model, const char* replica, int* done, int* status,
                     uint64_t* version, int* changed) {
  if (!c || !model || !replica) return st(rsb::Status::invalid_argument);
  auto o = c->reg.op_result(model, replica);
  if (done) *done = o.done;
  if (status) *status = st(o.status);
  if (version) *version = o.version.value_or(0);
  if (changed) *changed = o.changed;
  return 0;
}

int rs_server_complete(rs_cluster* c, const char* model, const char* replica, uint32_t shard,
                       int outcome) {
  if (!c || !model || !replica) return st(rsb::Status::invalid_argument);
  c->reg.complete(model, replica, shard, static_cast<rsb::Status>(outcome));
  return 0;
}

int rs_server_set_offload_seed(rs_cluster* c, const char* model, const char* replica, int on) {
  if (!c || !model || !replica) return st(rsb::Status::invalid_argument);
  return st(c->reg.set_offload_seed(model, replica, on != 0));
}

int rs_server_assignment(rs_cluster* c, const char* model, const char* replica, uint32_t shard,
                         rs_assignment* out) {
  if (!c || !model || !replica || !out) return st(rsb::Status::invalid_argument);
  auto o = c->reg.op_result(model, replica);
  if (!o.done || shard >= o.assignments.size()) return st(rsb::Status::not_found);
  fill_assignment(o.assignments[shard], out);
  return 0;
}

int rs_server_seed_start(rs_cluster* c, const char* model, const char* replica, uint32_t shard,
                         rs_assignment* out) {
  if (!c || !model || !replica) return 0;
  auto o = c->reg.op_result(model, replica);
  if (!o.done || !o.seed || shard >= o.seed->assignments.size()) return 0;
  if (out) fill_assignment(o.seed->assignments[shard], out);
  return 1;
}

int rs_server_seed_progress(rs_cluster* c, const char* model, const char* replica, uint32_t shard,
                            uint64_t items, uint64_t version) {
  if (!c || !model || !replica) return st(rsb::Status::invalid_argument);
  c->reg.progress(model, replica, shard, items, true, version);
  return 0;
}

int rs_server_seed_complete(rs_cluster* c, const char* model, const char* replica, uint32_t shard,
                            int outcome, uint64_t version) {
  if (!c || !model || !replica) return st(rsb::Status::invalid_argument);
  c->reg.complete(model, replica, shard, static_cast<rsb::Status>(outcome), true, version);
  return 0;
}

int rs_seed_lanes(rs_handle* h, uint64_t* versions, size_t cap, size_t* n) {
  if (!h) return st(rsb::Status::invalid_argument);
  h->client->join_seed();
  auto vs = h->client->seed_lanes();
  if (n) *n = vs.size();
  if (versions)
    for (size_t i = 0; i < vs.size() && i < cap; ++i) versions[i] = vs[i];
  return 0;
}

int rs_seed_fill(rs_handle* h) {
  if (!h) return st(rsb::Status::invalid_argument);
  auto& cl = *h->client;
  auto o = h->cluster->reg.op_result(cl.model(), cl.replica());
  if (!o.done || !o.seed) return st(rsb::Status::not_found);
  cl.set_seed_report(false);
  return st(cl.start_seed(*o.seed));
}

int rs_seed_status(rs_handle* h, uint32_t shard) {
  if (!h) return st(rsb::Status::invalid_argument);
  return st(h->client->seed_status(shard));
}

int rs_seed_export(rs_handle* h, uint32_t shard, uint64_t version, void* buf, size_t cap,
                   size_t* len) {
  if (!h) return st(rsb::Status::invalid_argument);
  auto r = h->client->export_seed(shard, version);
  if (!r) return st(r.status());
  return put_bytes(*r, static_cast<char*>(buf), cap, len);
}

int rs_seed_wait(rs_handle* h) {
  if (!h) return st(rsb::Status::invalid_argument);
  h->client->join_seed();
  return 0;
}

int rs_server_failure_report(rs_cluster* c, const char* model, const char* replica,
                             uint32_t shard, const char* failed_replica, int reason) {
  if (!c || !model || !replica || !failed_replica) return st(rsb::Status::invalid_argument);
  auto r = c->reg.failure_report(model, replica, shard, failed_replica, reason);
  return st(r.status());
}

int rs_server_close(rs_cluster* c, const char* model, const char* replica) {
  if (!c || !model || !replica) return st(rsb::Status::invalid_argument);
  return st(c->reg.close(model, replica));
}

int rs_prepare_publish(rs_handle* h, uint64_t version) {
  if (!h) return st(rsb::Status::invalid_argument);
  std::vector<std::string> ms;
  return st(h->client->prepare_publish(version, &ms));
}

int rs_commit_publish(rs_handle* h, uint64_t version, int status) {
  if (!h) return st(rsb::Status::invalid_argument);
  h->client->commit_publish(version, static_cast<rsb::Status>(status));
  return 0;
}

int rs_transfer_bind(rs_handle* h, uint64_t version) {
  if (!h) return st(rsb::Status::invalid_argument);
  auto& cl = *h->client;
  std::vector<rsb::Assignment> as(cl.num_shards());
  for (std::uint32_t i = 0; i < cl.num_shards(); ++i) {
    if (!cl.is_local(i)) continue;  // bound by the process that holds it
    auto a = h->cluster->reg.current_assignment(cl.model(), cl.replica(), i);
    if (!a) return st(a.status());
    as[i] = std::move(*a);
  }
  auto s = cl.bind_all(as, version);
  h->pending.clear();
  if (rsb::ok(s))
    for (std::uint32_t i = 0; i < cl.num_shards(); ++i)
      if (cl.is_local(i)) h->pending.push_back(i);
  return st(s);
}

int rs_transfer_launch(rs_handle* h) {
  if (!h) return st(rsb::Status::invalid_argument);
  auto& cl = *h->client;
  std::vector<rsb::Assignment> as(cl.num_shards());
  for (std::uint32_t i : h->pending) {
    auto a = h->cluster->reg.current_assignment(cl.model(), cl.replica(), i);
    if (!a) return st(a.status());
    as[i] = std::move(*a);
  }
  cl.launch_shards(as, h->pending);
  return 0;
}

int rs_transfer_progress(rs_handle* h, uint32_t shard, uint32_t* batches_done, uint32_t* n_batches) {
  if (!h || !batches_done || !n_batches) return st(rsb::Status::invalid_argument);
  return st(h->client->progress(shard, batches_done, n_batches));
}

int rs_transfer_assignment(rs_handle* h, uint32_t shard, rs_assignment* out) {
  if (!h || !out || shard >= h->client->num_shards()) return st(rsb::Status::invalid_argument);
  const rsb::Assignment* a = h->client->launched_assignment(shard);
  if (!a) return st(rsb::Status::not_found);
  fill_assignment(*a, out);
  return 0;
}

int rs_transfer_wait(rs_handle* h, int* statuses, int* reasons) {
  if (!h) return st(rsb::Status::invalid_argument);
  auto& cl = *h->client;
  auto res = cl.wait_shards(h->pending);
  std::vector<std::uint32_t> still;
  int worst = 0;
  for (std::uint32_t i = 0; i < cl.num_shards(); ++i) {
    int s = st(res[i].status);
    if (statuses) statuses[i] = s;
    if (reasons) reasons[i] = res[i].reason;
    bool was_pending = false;
    for (auto p : h->pending) was_pending |= p == i;
    if (was_pending && s != 0) {
      still.push_back(i);
      worst = s;
    }
  }
  h->pending = std::move(still);
  return worst;
}

int rs_transfer_fill(rs_handle* h, int* statuses, int* reasons) {
  if (int rc = rs_transfer_launch(h); rc != 0) return rc;
  return rs_transfer_wait(h, statuses, reasons);
}

int rs_transfer_finish(rs_handle* h, uint64_t version, int good) {
  if (!h) return st(rsb::Status::invalid_argument);
  h->client->finish_transfers(version, good != 0);
  return 0;
}

int rs_serve_export(rs_handle* h, uint32_t shard, void* buf, size_t cap, size_t* len) {
  if (!h) return st(rsb::Status::invalid_argument);
  auto b = h->client->export_serve(shard);
  if (!b) return st(b.status());
  return put_bytes(*b, static_cast<char*>(buf), cap, len);
}

int rs_serve_import(rs_cluster* c, const void* blob, size_t len) {
  if (!c || !blob) return st(rsb::Status::invalid_argument);
  return st(c->serves.import_state(std::string(static_cast<const char*>(blob), len)));
}

// ------------------------------------------------------- retention offload

int rs_connect(rs_handle* h) {
  if (!h) return st(rsb::Status::invalid_argument);
  return st(h->client->open());
}

int rs_set_retention(rs_handle* h, const uint64_t* lags, size_t n) {
  if (!h || (n && !lags)) return st(rsb::Status::invalid_argument);
  h->client->set_retention(std::set<std::uint64_t>(lags, lags + n));
  return 0;
}

int rs_offload_lanes(rs_handle* h, uint64_t version) {
  if (!h) return st(rsb::Status::invalid_argument);
  std::vector<std::string> eps;
  return st(h->client->make_retention_lanes(version, &eps));
}

int rs_lane_export(rs_handle* h, uint32_t shard, uint64_t version, void* buf, size_t cap,
                   size_t* len) {
  if (!h) return st(rsb::Status::invalid_argument);
  auto b = h->client->export_lane(shard, version);
  if (!b) return st(b.status());
  return put_bytes(*b, static_cast<char*>(buf), cap, len);
}

int rs_offload_release(rs_handle* h, uint64_t version) {
  if (!h) return st(rsb::Status::invalid_argument);
  h->client->release_lane(version);
  return 0;
}

int rs_poll(rs_handle* h) {
  if (!h) return st(rsb::Status::invalid_argument);
  h->client->apply_releases();
  return 0;
}

int rs_lanes(rs_handle* h, uint64_t* versions, size_t cap, size_t* n) {
  if (!h) return st(rsb::Status::invalid_argument);
  auto vs = h->client->lanes();
  if (n) *n = vs.size();
  if (versions)
    for (size_t i = 0; i < vs.size() && i < cap; ++i) versions[i] = vs[i];
  return 0;
}

int rs_server_set_retention(rs_cluster* c, const char* model, const char* replica,
                            const uint64_t* lags, size_t n) {
  if (!c || !model || !replica || (n && !lags)) return st(rsb::Status::invalid_argument);
  return st(c->reg.set_retention(model, replica, std::set<std::uint64_t>(lags, lags + n)));
}

int rs_server_offload_pending(rs_cluster* c, const char* model, const char* replica,
                              uint64_t* version) {
  if (!c || !model || !replica) return 0;
  auto o = c->reg.op_result(model, replica);
  if (o.done || !o.offload_first) return 0;
  if (version) *version = *o.offload_first;
  return 1;
}

int rs_server_offload_confirm(rs_cluster* c, const char* model, const char* replica,
                              uint32_t shard, uint64_t version, int ok, const char* endpoint) {
  if (!c || !model || !replica) return st(rsb::Status::invalid_argument);
  return st(c->reg.offload_confirm(model, replica, shard, version, ok != 0,
                                   endpoint ? endpoint : ""));
}

int rs_server_take_releases(rs_cluster* c, const char* model, const char* owner,
                            uint64_t* versions, size_t cap, size_t* n) {
  if (!c || !model || !owner) return st(rsb::Status::invalid_argument);
  auto rs = c->reg.take_releases(model, owner);
  if (n) *n = rs.size();
  if (versions)
    for (size_t i = 0; i < rs.size() && i < cap; ++i) versions[i] = rs[i].version;
  return 0;
}

int rs_cluster_listen(rs_cluster* c, const char* host, int port, int* bound_port) {
  if (!c || !host) return st(rsb::Status::invalid_argument);
  if (!c->stream) c->stream = std::make_unique<rsb::StreamServer>(&c->serves);
  auto r = c->stream->start(host, port);
  if (!r) return st(r.status());
  if (bound_port) *bound_port = *r;
  return 0;
}

int rs_cluster_kind(rs_cluster* c, const char* model, const char* replica, char* buf, size_t cap,
                    size_t* len) {
  if (!c || !model || !replica) return st(rsb::Status::invalid_argument);
  auto v = c->reg.view(model, replica);
  if (!v) return st(rsb::Status::not_found);
  return put_bytes(v->kind, buf, cap, len);
}

// ------------------------------------------------------- device primitives

int rs_digest_spans(const uint64_t* dev_ptrs, const uint64_t* lens, int n, uint64_t* out,
                    int device) {
  if (n < 0 || (n > 0 && (!dev_ptrs || !lens || !out))) return st(rsb::Status::invalid_argument);
  if (n == 0) return 0;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  rsb::DevBuf t;
  int rc = 0;
  if (!rsb::ok(t.alloc(device, 3 * std::size_t(n) * 8))) rc = st(rsb::Status::transfer_failed);
  auto* d = static_cast<std::uint64_t*>(t.p);
  if (!rc && (cudaMemcpy(d, dev_ptrs, n * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
              cudaMemcpy(d + n, lens, n * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
              rsb::dev::launch_span_digests(d, d + n, d + 2 * n, n, nullptr) != cudaSuccess ||
              cudaMemcpy(out, d + 2 * n, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess))
    rc = st(rsb::Status::transfer_failed);
  cudaSetDevice(prev);
  return rc;
}

int rs_synth_bf16(void* dev_dst, uint64_t n_elems, uint64_t seed, uint64_t first_elem,
                  void* cuda_stream) {
  if (!n_elems) return 0;
  if (!dev_dst) return st(rsb::Status::invalid_argument);
  return on_ptr_device(dev_dst, [&] {
    return rsb::dev::launch_synth_bf16(static_cast<std::uint16_t*>(dev_dst), n_elems, seed,
                                       first_elem, static_cast<cudaStream_t>(cuda_stream));
  });
}

int rs_bf16_to_e4m3(const void* dev_src, void* dev_dst, uint64_t n_elems, void* cuda_stream) {
  if (!n_elems) return 0;
  if (!dev_src || !dev_dst) return st(rsb::Status::invalid_argument);
  return on_ptr_device(dev_dst, [&] {
    return rsb::dev::launch_bf16_to_e4m3(static_cast<const std::uint16_t*>(dev_src),
                                         static_cast<std::uint8_t*>(dev_dst), n_elems,
                                         static_cast<cudaStream_t>(cuda_stream));
  });
}

int rs_pull_spans(const uint64_t* src_ptrs, const uint64_t* dst_ptrs, const uint64_t* lens,
                  int n_items, uint64_t chunk_bytes, const uint64_t* expect_dev,
                  uint64_t* out_digests_dev, int device, void* cuda_stream, int* kernel_code,
                  float* kernel_ms) {
  if (n_items < 0 || chunk_bytes == 0 || chunk_bytes % 16 || chunk_bytes > (1u << 30))
    return st(rsb::Status::invalid_argument);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  auto stream = static_cast<cudaStream_t>(cuda_stream);
  // spans in a peer GPU's memory (a pull from it, or a push into it)
  std::set<int> peers;
  for (int i = 0; i < n_items; ++i)
    for (const uint64_t* p : {src_ptrs, dst_ptrs}) {
      if (!p || !p[i]) continue;
      cudaPointerAttributes a{};
      if (cudaPointerGetAttributes(&a, reinterpret_cast<void*>(p[i])) == cudaSuccess &&
          a.type == cudaMemoryTypeDevice && a.device != device)
        peers.insert(a.device);
      cudaGetLastError();
    }
  for (int o : peers)
    if (!rsb::ok(rsb::enable_peer(device, o))) {
      cudaSetDevice(prev);
      return st(rsb::Status::not_serving);
    }
  const bool remote = !peers.empty();
  // Item i's chunks start at a multiple of 32 (batch aligned, as in
  // ChunkMap::uniform); indices in between are holes of expect/out tables.
  std::vector<rsb::dev::ItemDesc> descs(n_items);
  std::uint32_t chunk = 0;
  for (int i = 0; i < n_items; ++i) {
    descs[i] = {};
    descs[i].src = src_ptrs[i];
    descs[i].dst = dst_ptrs ? dst_ptrs[i] : 0;
    descs[i].len = lens[i];
    descs[i].chunk0 = chunk;
    descs[i].chunk_len = static_cast<std::uint32_t>(chunk_bytes);
    descs[i].src_chunk0 = chunk;
    descs[i].q = descs[i].m = 1;
    const auto n = static_cast<std::uint32_t>((lens[i] + chunk_bytes - 1) / chunk_bytes);
    chunk += (n + rsb::dev::kBatchChunks - 1) / rsb::dev::kBatchChunks * rsb::dev::kBatchChunks;
  }
  rsb::dev::PlanUpload plan;
  int rc = 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  rsb::dev::PullStatus ps{};
  rsb::dev::PullParams p{};
  const rsb::dev::SrcDesc sdesc{expect_dev, nullptr, 0, 0};
  const bool debug = std::getenv("RSB_DEBUG") != nullptr;
  auto failed = [&](cudaError_t e, const char* what) {
    if (e == cudaSuccess) return false;
    if (debug) std::fprintf(stderr, "[rsb] rs_pull_spans: %s: %s\n", what, cudaGetErrorString(e));
    return true;
  };
  if (failed(rsb::dev::upload_pull_plan(device, stream, descs.data(), static_cast<std::uint32_t>(n_items),
                                        &sdesc, 1, chunk, &plan, &p), "plan upload"))
    rc = st(rsb::Status::transfer_failed);
  if (!rc) {
    p.remote = remote ? 1u : 0u;
    p.dst_digests = out_digests_dev;
    p.timeout_ns = 4000000000ull;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    if (failed(cudaEventRecord(e0, stream), "event") ||
        failed(rsb::dev::launch_pull(p, rsb::dev::pull_grid(device), stream), "launch") ||
        failed(cudaEventRecord(e1, stream), "event") ||
        failed(cudaMemcpyAsync(&ps, p.status, sizeof(ps), cudaMemcpyDeviceToHost, stream), "status copy") ||
        failed(cudaStreamSynchronize(stream), "kernel"))
      rc = st(rsb::Status::transfer_failed);
    float ms = 0;
    if (!rc) cudaEventElapsedTime(&ms, e0, e1);
    if (kernel_ms) *kernel_ms = ms;
    if (kernel_code) *kernel_code = static_cast<int>(ps.code);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  rsb::dev::free_pull_plan(device, &plan);
  cudaSetDevice(prev);
  return rc;
}

}  // extern "C"
