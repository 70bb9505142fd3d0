// Placement of managed allocations in the shim's reserved virtual range, in
// 2 MiB blocks (internal header; unit-tested by tests/cpp/test_units.cpp).
//
// Why placement matters: a virtual slab holds a whole physical slab while any
// of its blocks is resident, so the blocks a victim gives up
// at a switch should empty whole slabs. The planner evicts a victim's chunks
// largest footprint first, ties by ascending chunk id, each chunk's blocks in
// order (proj/src/planner.cpp:47-76). In a model that is every 96 MiB weight
// of every layer, then every 32 MiB one, ...; packed in allocation order
// those are interleaved, and a partial eviction leaves every slab of the
// model partly resident.
//
// Default (lanes): allocations smaller than a slab get a lane per exact size,
// a slab-aligned span of the range filled in allocation order (= chunk id
// order). Equal footprints are evicted in exactly that order, so a victim's
// evicted blocks empty each lane's slabs one after another and only the
// boundary slab of the lane being evicted stays partly resident. Single
// blocks and allocations of a slab or more bump through the common part of
// the range (slab-aligned from half a slab up). Freed ranges are not reused;
// the range is 1 TiB.
// NIXIE_SHIM_FIRST_FIT=1: one first-fit free list that reuses freed holes
// (scatters the eviction order; kept for comparison).
#pragma once

#include <cstdint>
#include <iterator>
#include <map>

namespace nixie::shim {

class RangeAlloc {
 public:
  void reset(std::uint64_t blocks, bool first_fit = false) {
    free_.clear();
    lanes_.clear();
    if (blocks) free_[0] = blocks;
    blocks_ = blocks;
    first_fit_ = first_fit;
  }

  bool take(std::uint64_t n, std::uint64_t slab_blocks, std::uint64_t& start) {
    if (n == 0) return false;
    if (!first_fit_ && slab_blocks && n >= kLaneMin && n < slab_blocks && take_lane(n, slab_blocks, start))
      return true;
    const std::uint64_t align = slab_blocks && n >= slab_blocks / 2 ? slab_blocks : 1;
    return carve(n, align, start);
  }

  void give(std::uint64_t start, std::uint64_t n) {
    if (!first_fit_) return;  // lanes / bump never reuse a range
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
  std::size_t lanes() const { return lanes_.size(); }

  static constexpr std::uint64_t kLaneMin = 2;  // single blocks share the common bump

 private:
  struct Lane {
    std::uint64_t cur, end;
  };

  // Takes n blocks aligned to `align`: first fit over the free runs, or the
  // tail run only (bump) when lanes are on.
  bool carve(std::uint64_t n, std::uint64_t align, std::uint64_t& start) {
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

  bool take_lane(std::uint64_t n, std::uint64_t sb, std::uint64_t& start) {
    auto it = lanes_.find(n);
    if (it == lanes_.end() || it->second.cur + n > it->second.end) {
      // a new span for this size: 1/64 of the range (16 GiB of 1 TiB), at
      // least 8 slabs, while three quarters of the range stay common
      std::uint64_t span = blocks_ / 64;
      if (span < 8 * sb) span = 8 * sb;
      span = (span + sb - 1) / sb * sb;
      if (free_.empty()) return false;
      const auto tail = std::prev(free_.end());
      if (tail->second < span + blocks_ / 4) return false;
      std::uint64_t s0 = 0;
      if (!carve(span, sb, s0)) return false;
      it = lanes_.insert_or_assign(n, Lane{s0, s0 + span}).first;
    }
    start = it->second.cur;
    it->second.cur += n;
    return true;
  }

  std::map<std::uint64_t, std::uint64_t> free_;  // start -> length
  std::map<std::uint64_t, Lane> lanes_;          // allocation size -> its current span
  std::uint64_t blocks_ = 0;
  bool first_fit_ = false;
};

}  // namespace nixie::shim
