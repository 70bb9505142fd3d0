// Placement of managed allocations in the shim's reserved virtual range, in
// 2 MiB blocks (internal header; unit-tested by tests/cpp/test_units.cpp).
//
// Bump order by default: every allocation goes after the previous one, so
// range order equals allocation order, which is the registry's chunk order,
// which is the order the planner evicts a victim's blocks in
// (proj/src/planner.cpp:47-76). A victim's evicted blocks then empty its
// virtual slabs one after another, and at most the boundary slab stays partly
// resident. First fit (reusing freed holes) scatters that order and leaves
// many partly resident slabs, each holding a whole physical slab
// (DESIGN.md §10). The 1 TiB range is not reused in bump mode.
// Allocations of at least half a slab start on a slab boundary.
#pragma once

#include <cstdint>
#include <iterator>
#include <map>

namespace nixie::shim {

class RangeAlloc {
 public:
  void reset(std::uint64_t blocks, bool first_fit = false) {
    free_.clear();
    if (blocks) free_[0] = blocks;
    first_fit_ = first_fit;
  }

  bool take(std::uint64_t n, std::uint64_t slab_blocks, std::uint64_t& start) {
    if (n == 0) return false;
    const std::uint64_t align = slab_blocks && n >= slab_blocks / 2 ? slab_blocks : 1;
    // bump mode: only the last run (the untouched tail of the range)
    auto first = first_fit_ || free_.empty() ? free_.begin() : std::prev(free_.end());
    for (auto it = first; it != free_.end(); ++it) {
      const std::uint64_t s0 = (it->first + align - 1) / align * align;
      if (s0 + n > it->first + it->second) continue;
      const std::uint64_t run_start = it->first, run_len = it->second;
      free_.erase(it);
      if (s0 > run_start) free_[run_start] = s0 - run_start;
      if (s0 + n < run_start + run_len) free_[s0 + n] = run_start + run_len - (s0 + n);
      start = s0;
      return true;
    }
    return false;
  }

  void give(std::uint64_t start, std::uint64_t n) {
    if (!first_fit_) return;  // bump mode never reuses a range
    auto next = free_.lower_bound(start);
    if (next != free_.end() && start + n == next->first) {
      n += next->second;
      next = free_.erase(next);
    }
    if (next != free_.begin()) {
      auto prev = std::prev(next);
      if (prev->first + prev->second == start) {
        prev->second += n;
        return;
      }
    }
    free_[start] = n;
  }

  const std::map<std::uint64_t, std::uint64_t>& runs() const { return free_; }

 private:
  std::map<std::uint64_t, std::uint64_t> free_;  // start -> length
  bool first_fit_ = false;
};

}  // namespace nixie::shim
