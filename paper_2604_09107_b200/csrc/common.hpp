// Shared host-side vocabulary of the B200 ROS read path.
#pragma once

#include <cstdint>
#include <optional>
#include <set>
#include <string>
#include <string_view>
#include <utility>
#include <variant>

namespace rsb {

using VersionId = std::uint64_t;

// Wire-visible status codes; values are identical to refstore::Status
// (/root/reference/proj/include/refstore/types.hpp:22-41) so the C ABI's int
// returns mean the same thing to a caller of either implementation.
enum class Status : std::uint8_t {
  ok = 0,
  invalid_argument = 1,
  invalid_state = 2,
  already_exists = 3,
  not_found = 4,
  version_regression = 5,
  manifest_conflict = 6,
  mutability_violation = 7,
  version_unavailable = 8,
  group_aborted = 9,
  server_unavailable = 10,
  transfer_failed = 11,
  checksum_mismatch = 12,
  not_serving = 13,
  timeout = 14,
  offload_failed = 15,
  protocol_error = 16,
  closed = 17,
};

const char* status_name(Status s);
inline bool ok(Status s) { return s == Status::ok; }

template <typename T>
class Result {
 public:
  Result(T v) : v_(std::move(v)) {}
  Result(Status s) : v_(s) {}
  bool has_value() const { return v_.index() == 0; }
  explicit operator bool() const { return has_value(); }
  Status status() const { return has_value() ? Status::ok : std::get<1>(v_); }
  T& operator*() { return std::get<0>(v_); }
  const T& operator*() const { return std::get<0>(v_); }
  T* operator->() { return &std::get<0>(v_); }
  const T* operator->() const { return &std::get<0>(v_); }

 private:
  std::variant<T, Status> v_;
};

// "17" | "latest" | "latest-k"  (reference types.hpp:72-93, types.cpp:31-66).
struct VersionSpec {
  bool absolute = false;
  std::uint64_t value = 0;  // version (absolute) or lag (relative)
  static Result<VersionSpec> parse(std::string_view text);
  std::string to_string() const;
};

// absolute(v): v if available; latest(k): the (k+1)-th largest available.
std::optional<VersionId> resolve_version(const VersionSpec& spec,
                                         const std::set<VersionId>& avail);

}  // namespace rsb
