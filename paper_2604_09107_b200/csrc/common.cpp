#include "common.hpp"

#include <charconv>
#include <iterator>

namespace rsb {

const char* status_name(Status s) {
  static const char* const kNames[] = {
      "ok",                 "invalid_argument",    "invalid_state",
      "already_exists",     "not_found",           "version_regression",
      "manifest_conflict",  "mutability_violation", "version_unavailable",
      "group_aborted",      "server_unavailable",  "transfer_failed",
      "checksum_mismatch",  "not_serving",         "timeout",
      "offload_failed",     "protocol_error",      "closed"};
  auto i = static_cast<unsigned>(s);
  return i < std::size(kNames) ? kNames[i] : "unknown";
}

namespace {
bool parse_u64(std::string_view t, std::uint64_t& out) {
  if (t.empty()) return false;
  auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), out);
  return ec == std::errc() && p == t.data() + t.size();
}
}  // namespace

Result<VersionSpec> VersionSpec::parse(std::string_view text) {
  VersionSpec s;
  constexpr std::string_view kLatest = "latest";
  if (text == kLatest) return s;
  if (text.size() > kLatest.size() + 1 && text.substr(0, kLatest.size() + 1) == "latest-") {
    if (!parse_u64(text.substr(kLatest.size() + 1), s.value))
      return Status::invalid_argument;
    return s;
  }
  s.absolute = true;
  if (!parse_u64(text, s.value)) return Status::invalid_argument;
  return s;
}

std::string VersionSpec::to_string() const {
  if (absolute) return std::to_string(value);
  return value == 0 ? "latest" : "latest-" + std::to_string(value);
}

std::optional<VersionId> resolve_version(const VersionSpec& spec,
                                         const std::set<VersionId>& avail) {
  if (avail.empty()) return std::nullopt;
  if (spec.absolute)
    return avail.count(spec.value) ? std::optional<VersionId>(spec.value)
                                   : std::nullopt;
  if (spec.value >= avail.size()) return std::nullopt;
  return *std::next(avail.rbegin(), static_cast<long>(spec.value));
}

}  // namespace rsb
