// refstore/b200_transport.hpp -- level B integration: the
// reference's own ClientCore / ServerCore stay, and only the data plane's
// byte mover changes.  B200Transport is a refstore::DataTransport
// (transport.hpp:127-140) whose async_pull moves the bytes with the B200
// path's device copy (rs_pull_spans: the sm_100a TMA pull kernel) instead of
// MemNetwork's memcpy (transport_mem.cpp:170-201).
//
// Everything around the copy is the reference's: the safe prefix is the
// reference's compute_slice (transport.cpp:32-49) over the source's
// PeerServeState, the stream offset -> item span walk is copy_slice_locked's
// (transport.cpp:51-69), and the control plane and the long-poll queries go
// through the wrapped MemNetwork.  Registered regions must be reachable by
// both the GPU (the copy) and the CPU (the reference still digests items on
// the host in TransferTask::verify_ready / build_publish_payload), e.g.
// cudaMallocManaged memory.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "refstore/transport.hpp"
#include "refstore/transport_mem.hpp"
#include "ros_b200.h"

namespace refstore {

class B200Transport : public DataTransport {
 public:
  B200Transport(MemNetwork* net, int device) : net_(net), device_(device) {}

  // Same registration as MemNetwork::register_data (the endpoint a client
  // advertises -> its ServeRegistry); the MemNetwork keeps serving queries.
  void register_data(const std::string& endpoint, ServeRegistry* serves) {
    {
      std::lock_guard lk(m_);
      data_[endpoint] = serves;
    }
    net_->register_data(endpoint, serves);
  }

  void async_pull(const std::string& endpoint, const PullSpec& spec, PullDest dest,
                  Executor* exec, std::function<void(PullResult)> done) override {
    std::shared_ptr<PeerServeState> st;
    {
      std::lock_guard lk(m_);
      auto it = data_.find(endpoint);
      if (it != data_.end()) st = it->second->find(ServeRegistry::key(spec.model, spec.replica, spec.shard));
    }
    PullResult r;
    if (!st) {
      r.status = Status::not_serving;
      exec->post([done = std::move(done), r] { done(r); });
      return;
    }
    ServeSlice s = compute_slice(*st, spec.version, spec.offset, spec.max_bytes);
    r.status = s.status;
    r.source_progress = s.progress;
    r.source_complete = s.complete;
    r.bytes = s.bytes;
    if (ok(s.status) && s.bytes > 0 && !dest.empty()) {
      std::lock_guard lk(st->m);
      // [offset, offset + bytes) of the source's item stream against the
      // ordered destination spans: one (src, dst, len) copy per overlap.
      std::vector<std::uint64_t> srcs, dsts, lens;
      std::uint64_t off = spec.offset, left = s.bytes;
      std::size_t idx = std::upper_bound(st->item_ends.begin(), st->item_ends.end(), off) -
                        st->item_ends.begin();
      std::size_t di = 0;
      std::uint64_t in_dest = 0;
      while (left && idx < st->item_spans.size() && di < dest.size()) {
        const std::uint64_t item_start = idx == 0 ? 0 : st->item_ends[idx - 1];
        const std::uint64_t in_item = off - item_start;
        const auto span = st->item_spans[idx];
        const std::uint64_t take = std::min({left, span.size() - in_item, dest[di].size() - in_dest});
        srcs.push_back(reinterpret_cast<std::uint64_t>(span.data() + in_item));
        dsts.push_back(reinterpret_cast<std::uint64_t>(dest[di].data() + in_dest));
        lens.push_back(take);
        off += take;
        left -= take;
        in_dest += take;
        if (in_item + take == span.size()) ++idx;
        if (in_dest == dest[di].size()) {
          ++di;
          in_dest = 0;
        }
      }
      int code = 0;
      float ms = 0;
      const int rc = rs_pull_spans(srcs.data(), dsts.data(), lens.data(), static_cast<int>(srcs.size()),
                                   4096, nullptr, nullptr, device_, nullptr, &code, &ms);
      if (rc != 0 || code != 0) r.status = Status::transfer_failed;
      pulls_.fetch_add(1);
      device_bytes_.fetch_add(s.bytes - left);
    }
    if (ok(r.status) && spec.activity) spec.activity->fetch_add(1);
    exec->post([done = std::move(done), r] { done(r); });
  }

  void async_query(const std::string& endpoint, const QuerySpec& spec, Executor* exec,
                   std::function<void(QueryResult)> done) override {
    net_->async_query(endpoint, spec, exec, std::move(done));
  }

  std::uint64_t device_pulls() const { return pulls_.load(); }
  std::uint64_t device_bytes() const { return device_bytes_.load(); }

 private:
  MemNetwork* net_;
  int device_;
  std::mutex m_;
  std::map<std::string, ServeRegistry*> data_;
  std::atomic<std::uint64_t> pulls_{0}, device_bytes_{0};
};

}  // namespace refstore
