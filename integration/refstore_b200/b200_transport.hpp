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
#include <cstring>
#include <cstdint>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include <cuda_runtime.h>

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

  // MemNetwork::set_data_silent (transport_mem.hpp:43-46): a silent
  // endpoint swallows pulls and queries without a reply (a crashed peer).
  void set_data_silent(const std::string& endpoint, bool silent) {
    {
      std::lock_guard lk(m_);
      if (silent) silent_.insert(endpoint);
      else silent_.erase(endpoint);
    }
    net_->set_data_silent(endpoint, silent);
  }

  void async_pull(const std::string& endpoint, const PullSpec& spec, PullDest dest,
                  Executor* exec, std::function<void(PullResult)> done) override {
    std::shared_ptr<PeerServeState> st;
    {
      std::lock_guard lk(m_);
      if (silent_.count(endpoint)) return;  // nothing ever comes back
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
      // Registered regions (device or managed memory) move on the GPU.  The
      // reference's packed-group staging lives on the host heap (pageable,
      // Payload::group_bufs), which the GPU cannot address: those few small
      // spans are copied on the host, exactly as MemNetwork would.
      auto gpu_addressable = [](std::uint64_t p) {
        cudaPointerAttributes a{};
        const bool ok = cudaPointerGetAttributes(&a, reinterpret_cast<void*>(p)) == cudaSuccess &&
                        (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged);
        cudaGetLastError();
        return ok;
      };
      std::vector<std::uint64_t> ks, kd, kl;
      for (std::size_t k = 0; k < srcs.size(); ++k) {
        if (gpu_addressable(srcs[k]) && gpu_addressable(dsts[k])) {
          ks.push_back(srcs[k]);
          kd.push_back(dsts[k]);
          kl.push_back(lens[k]);
        } else {
          cudaDeviceSynchronize();  // managed pages the GPU may still hold
          std::memcpy(reinterpret_cast<void*>(dsts[k]), reinterpret_cast<const void*>(srcs[k]), lens[k]);
          host_bytes_.fetch_add(lens[k]);
        }
      }
      if (!ks.empty()) {
        // managed regions migrate to the pulling GPU first, so the kernel's
        // bulk-tensor copies touch resident pages (the reference's host-side
        // digest faults them back afterwards)
        for (std::size_t k = 0; k < ks.size(); ++k)
          for (std::uint64_t p : {ks[k], kd[k]}) {
            cudaPointerAttributes a{};
            if (cudaPointerGetAttributes(&a, reinterpret_cast<void*>(p)) == cudaSuccess &&
                a.type == cudaMemoryTypeManaged)
              cudaMemPrefetchAsync(reinterpret_cast<void*>(p), kl[k], device_, nullptr);
            cudaGetLastError();
          }
        cudaStreamSynchronize(nullptr);
        int code = 0;
        float ms = 0;
        const int rc = rs_pull_spans(ks.data(), kd.data(), kl.data(), static_cast<int>(ks.size()), 4096,
                                     nullptr, nullptr, device_, nullptr, &code, &ms);
        if (rc != 0 || code != 0) {
          r.status = Status::transfer_failed;
          last_error_.store((static_cast<std::uint64_t>(rc) << 32) | static_cast<std::uint32_t>(code));
        }
        for (auto l : kl) device_bytes_.fetch_add(l);
      }
      pulls_.fetch_add(1);
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
  std::uint64_t host_bytes() const { return host_bytes_.load(); }  // group staging on the host
  // (rs_pull_spans status << 32 | kernel code) of the last failed pull, 0: none
  std::uint64_t last_error() const { return last_error_.load(); }

 private:
  MemNetwork* net_;
  int device_;
  std::mutex m_;
  std::map<std::string, ServeRegistry*> data_;
  std::set<std::string> silent_;
  std::atomic<std::uint64_t> pulls_{0}, device_bytes_{0}, host_bytes_{0}, last_error_{0};
};

}  // namespace refstore
