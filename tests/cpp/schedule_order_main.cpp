// Host-side check of the pull schedule (pullplan.cpp schedule_order): reads
// cases from stdin, prints each case's order.  Built and driven by
// tests/test_schedule_order.py; no GPU needed.
//   case:  n_batches n_segments, then per segment: chunk0 chunk_len len link_class
#include <cstdio>
#include <vector>

#include "device.hpp"

int main() {
  unsigned nb = 0, n = 0;
  while (std::scanf("%u %u", &nb, &n) == 2) {
    std::vector<rsb::dev::ItemDesc> items(n);
    for (auto& d : items) {
      unsigned long long len = 0;
      unsigned cl = 0;
      std::scanf("%u %u %llu %u", &d.chunk0, &cl, &len, &d.pad);
      d.chunk_len = cl;
      d.len = len;
    }
    std::vector<std::uint32_t> bseg(nb);
    for (std::uint32_t b = 0, sg = 0; b < nb; ++b) {
      while (sg + 1 < n && items[sg + 1].chunk0 <= b * rsb::dev::kBatchChunks) ++sg;
      bseg[b] = sg;
    }
    const auto order = rsb::dev::schedule_order(items.data(), n, bseg);
    std::printf("%zu", order.size());
    for (auto b : order) std::printf(" %u", b);
    std::printf("\n");
  }
  return 0;
}
