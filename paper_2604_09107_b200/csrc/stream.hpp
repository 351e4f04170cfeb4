// Off-box data plane: serve states over TCP.
//
// The reference's stream transport (transport_stream.hpp:36-76, the RSDP
// wire) moves pull windows between hosts.  Here a process runs one
// StreamServer; a reader whose assigned source endpoint is "tcp:host:port"
// opens a few connections (RSB_TCP_STREAMS, default 4), names the serve
// state (model|replica|shard), version and its stripe on each, and receives
// the source's chunk map and chunk-digest table (first connection) followed
// by the payload in frames of watermark batches, frame k on connection k % n (the server D2H-copies each batch from the
// source's device memory into pinned staging once the source has verified
// it, so a chasing chain works across the wire too).  The reader lands the
// stream into pinned, device-mapped host memory and raises a host watermark
// per batch; the SAME pull kernel then lands and verifies it into the
// reader's regions, chasing those host watermarks -- network receive, PCIe
// and the kernel overlap batch by batch.
#pragma once

#include <atomic>
#include <chrono>
#include <cstdint>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "client.hpp"

namespace rsb {

// rsdp.cpp: serves one connection speaking the reference's data wire (RSDP,
// transport_stream.hpp:36-76) from this process's serve states; `first4`
// are the header bytes the caller already read.  Closes fd.
void serve_rsdp(int fd, ServeRegistry* serves, const std::uint8_t first4[4]);

class StreamServer {
 public:
  explicit StreamServer(ServeRegistry* serves);
  ~StreamServer();
  // Listen on host:port (port 0: any free port); returns the bound port.
  Result<int> start(const std::string& host, int port);
  void stop();
  int port() const { return port_; }

 private:
  void accept_loop();
  void serve_conn(int fd);

  // Per-connection D2H staging, created at start() and reused: pinned
  // allocation and release synchronize the device, and a reader's persistent
  // pull kernel on that device may be waiting for this very stream.
  struct Slot {
    void* stage[2] = {nullptr, nullptr};
    std::size_t bytes = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
  };
  Slot* take_slot();
  void give_slot(Slot* s);

  ServeRegistry* serves_;
  std::vector<std::unique_ptr<Slot>> slots_;
  std::vector<Slot*> free_slots_;
  std::mutex slots_mu_;
  int listen_fd_ = -1;
  int port_ = 0;
  std::atomic<bool> stop_{false};
  std::thread acceptor_;
  std::vector<std::thread> conns_;
  std::mutex conns_mu_;
};

// A source reached over TCP: the received stream in pinned host memory.
class StreamSource {
 public:
  StreamSource() = default;
  ~StreamSource();
  StreamSource(const StreamSource&) = delete;
  StreamSource& operator=(const StreamSource&) = delete;
  // Connect to "tcp:host:port", request `key` at `version`, read the header
  // (chunk map + digests) and start receiving in the background.
  // `pool` holds pinned buffers from earlier fills (pinning fresh host
  // memory is slow): taken when large enough, handed back by release().
  Status open(const std::string& endpoint, const std::string& key, VersionId version,
              double timeout_s, std::vector<std::unique_ptr<HostBuf>>* pool = nullptr);
  void release(std::vector<std::unique_ptr<HostBuf>>* pool);
  // The view the pull kernel reads: host item pointers, digests, watermarks
  // (flags == 1 once a batch arrived).
  const SourceView& view() const { return view_; }
  // Waits for the receiver; ok when every batch arrived.  kernel_ok false:
  // the pull kernel failed, so the sockets are shut instead of drained.
  Status finish(bool kernel_ok = true);
  std::uint64_t bytes_received() const { return received_.load(); }
  // watermarks raised so far, and the first batch still missing
  std::pair<std::uint32_t, std::uint32_t> flag_summary() const;

 private:
  void receive_loop(int fd);
  void abort_all();
  static bool valid_header(const ChunkMap& cm, const std::vector<std::uint64_t>& lens);

  // one connection per stripe of the stream's frames (frame k on k % n);
  // the first also carries the header
  std::vector<int> fds_;
  std::unique_ptr<HostBuf> data_, tables_;
  SourceView view_;
  std::vector<std::uint64_t> item_off_;  // byte offset of each item in data_
  std::vector<std::uint64_t> item_len_;  // bytes of each item (validated header)
  std::vector<std::thread> rx_;
  std::atomic<int> rx_status_{0};  // first failure of any connection
  std::atomic<std::uint64_t> received_{0};
};

}  // namespace rsb
