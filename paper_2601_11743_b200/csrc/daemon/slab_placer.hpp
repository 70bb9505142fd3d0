// SlabPlacer: GPU frame placement of the interposer daemon (internal header,
// unit-tested by tests/cpp/test_units.cpp).
#pragma once

#include <cstdint>
#include <algorithm>
#include <deque>
#include <functional>
#include <map>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "nixie/swap_engine.hpp"
#include "nixie_ipc.hpp"

namespace nixie::b200 {

// GPU frame placement for the interposer: each application's virtual
// slab (slab_blocks blocks of its shim's range) is backed by one whole
// physical slab while any of its blocks is on the GPU, at the block's slot.
// The registry still charges 2 MiB per resident block against the budget;
// the arena holds `slack` extra slabs for slabs that are partly resident
// (an eviction boundary inside a slab, or small allocations sharing one).
class SlabPlacer final : public FramePlacer {
 public:
  using Key = std::pair<AppId, std::uint32_t>;  // (app, vslab)

  SlabPlacer(std::uint32_t slabs, std::uint32_t slab_blocks)
      : sb_(slab_blocks), base_(slabs), is_free_(slabs, 1), gen_(slabs, 1), nfree_(slabs) {
    for (std::uint32_t p = 0; p < slabs; ++p) free_.push_back(p);
  }

  // Blocks first .. first+n-1 (about to be created by MemState::allocate, in
  // order) sit at range blocks va_block .. of `app`.
  void expect(BlockId first, std::uint64_t n, AppId app, std::uint64_t va_block) {
    if (app_.size() < first + n) {
      app_.resize(first + n);
      vpos_.resize(first + n);
    }
    for (std::uint64_t k = 0; k < n; ++k) {
      app_[first + k] = app;
      vpos_[first + k] = va_block + k;
    }
  }

  std::uint32_t acquire(BlockId b) override {
    if (b >= app_.size()) throw InvariantViolation("slab placer: block " + std::to_string(b) + " has no virtual placement");
    Slab& s = slabs_[key(b)];
    if (s.phys == ipc::kNoFrame) {
      if (nfree_ == 0) {
        // Partly resident slabs (eviction boundaries, allocations sharing a
        // slab) can use up the slack: the arena grows by one slab.
        if (!grow_)
          throw InvariantViolation("slab placer: every physical slab is in use (partly resident slabs: " +
                                   std::to_string(partial()) + ")");
        const std::uint32_t p = grow_();
        if (is_free_.size() <= p) {
          is_free_.resize(p + 1, 0);
          gen_.resize(p + 1, 0);
        }
        ++gen_[p];
        dropped_.erase(p);
        is_free_[p] = 1;
        free_.push_back(p);
        ++nfree_;
        ++grown_;
      }
      // Affinity: the slab this vslab had last time, if it is free, is still
      // mapped in the app (stale mappings are kept), so no remap is needed.
      if (s.pref != ipc::kNoFrame && is_free_[s.pref]) {
        s.phys = s.pref;
      } else {
        while (!is_free_[free_.front()]) free_.pop_front();  // lazily deleted entries
        s.phys = free_.front();
        free_.pop_front();
      }
      is_free_[s.phys] = 0;
      --nfree_;
      s.pref = s.phys;
    }
    if (s.count++ == 0) assigned_.push_back(key(b));
    return s.phys * sb_ + static_cast<std::uint32_t>(vpos_[b] % sb_);
  }

  void release(BlockId b, std::uint32_t frame) override {
    const Key k = key(b);
    Slab& s = slabs_[k];
    if (s.count == 0 || frame / sb_ != s.phys) throw InvariantViolation("slab placer: release of an unplaced block");
    if (--s.count == 0) {
      free_.push_back(s.phys);
      is_free_[s.phys] = 1;
      ++nfree_;
      s.phys = ipc::kNoFrame;
      released_.push_back(k);
    }
  }

  // vslabs that got a physical slab since the last call.
  std::vector<Key> take_assigned() { return std::exchange(assigned_, {}); }

  // vslabs that lost their physical slab since the last call.
  std::vector<Key> take_released() { return std::exchange(released_, {}); }

  // Every backed vslab of `app`.
  std::vector<ipc::SlabMap> backed(AppId app) const {
    std::vector<ipc::SlabMap> out;
    for (auto it = slabs_.lower_bound(Key{app, 0}); it != slabs_.end() && it->first.first == app; ++it)
      if (it->second.phys != ipc::kNoFrame) out.push_back(ipc::SlabMap{it->first.second, it->second.phys});
    return out;
  }

  ipc::SlabMap map_of(AppId app, std::uint32_t vslab) const {
    auto it = slabs_.find(Key{app, vslab});
    return ipc::SlabMap{vslab, it == slabs_.end() ? ipc::kNoFrame : it->second.phys};
  }

  std::uint64_t partial() const {
    std::uint64_t n = 0;
    for (const auto& kv : slabs_) n += kv.second.phys != ipc::kNoFrame && kv.second.count < sb_;
    return n;
  }
  std::size_t free_slabs() const { return nfree_; }
  std::size_t slabs() const { return is_free_.size(); }  // slots (dropped ones included)
  std::uint32_t gen(std::uint32_t p) const { return gen_[p]; }
  std::uint32_t base() const { return base_; }  // slabs created at start, never dropped
  std::size_t live_slabs() const { return is_free_.size() - dropped_.size(); }
  bool dropped(std::uint32_t p) const { return gen_[p] == 0 || dropped_.count(p) != 0; }

  // Free grown slabs beyond `keep_free` free ones, taken out of the pool to
  // be dropped (highest index first); vslabs still (stale-)mapped to them are
  // marked unmapped (the shims unmap them on Drop).
  std::vector<std::uint32_t> take_droppable(std::size_t keep_free) {
    std::vector<std::uint32_t> out;
    for (std::uint32_t p = static_cast<std::uint32_t>(is_free_.size()); p-- > base_ && nfree_ > keep_free;) {
      if (!is_free_[p]) continue;
      is_free_[p] = 0;
      --nfree_;
      dropped_.insert(p);
      out.push_back(p);
    }
    if (!out.empty())
      for (auto& kv : slabs_)
        for (std::uint32_t p : out)
          if (kv.second.mapped == p) kv.second.mapped = ipc::kNoFrame;
    return out;
  }
  // A dropped slot handed out again by grow() is live again.
  void revive(std::uint32_t p) { dropped_.erase(p); }
  std::uint32_t grown() const { return grown_; }
  // Called when no slab is free; returns the index of a new one.
  void set_grow(std::function<std::uint32_t()> g) { grow_ = std::move(g); }

  // What the app's shim has mapped at a vslab (as far as the daemon told it).
  std::uint32_t mapped(const Key& k) const {
    auto it = slabs_.find(k);
    return it == slabs_.end() ? ipc::kNoFrame : it->second.mapped;
  }
  void set_mapped(const Key& k, std::uint32_t phys) { slabs_[k].mapped = phys; }
  // Slab-aligned victim choice (PlannerConfig::gpu_victims): per victim app,
  // in the planner's app order, its GPU-resident blocks grouped by virtual
  // slab, fewest resident first, whole groups until `want` bytes are covered;
  // only the last group is split. Same bytes and app order as the reference
  // planner, but an eviction frees whole physical slabs instead of leaving
  // every slab the largest chunks touch partly resident.
  std::vector<BlockId> slab_victims(const MemState& st, const std::vector<AppId>& order, Bytes want) const {
    std::vector<BlockId> out;
    const std::uint64_t need = block_count_for(want);
    for (AppId app : order) {
      std::map<std::uint32_t, std::vector<BlockId>> by_vslab;
      for (ChunkId c : st.chunks_of(app))
        for (BlockId b : st.chunk(c).blocks) {
          const Location& loc = st.block(b).loc;
          if (!loc.is_resident() || loc.tier != TierId::Gpu) continue;
          if (b >= app_.size()) throw InvariantViolation("slab placer: block " + std::to_string(b) + " has no virtual placement");
          by_vslab[key(b).second].push_back(b);
        }
      std::vector<std::vector<BlockId>*> groups;
      for (auto& kv : by_vslab) groups.push_back(&kv.second);
      std::stable_sort(groups.begin(), groups.end(), [](auto* a, auto* b) { return a->size() < b->size(); });
      for (auto* g : groups) {
        std::sort(g->begin(), g->end(), [&](BlockId a, BlockId b) { return vpos_[a] < vpos_[b]; });
        for (BlockId b : *g) {
          out.push_back(b);
          if (out.size() >= need) return out;
        }
      }
    }
    return out;
  }

  std::uint32_t vslab_of(BlockId b) const { return key(b).second; }

  // After a Grant: the shim maps exactly the backed vslabs and unmaps the rest.
  void granted(AppId app) {
    for (auto it = slabs_.lower_bound(Key{app, 0}); it != slabs_.end() && it->first.first == app; ++it)
      it->second.mapped = it->second.phys;
  }

 private:
  struct Slab {
    std::uint32_t phys = ipc::kNoFrame;
    std::uint32_t count = 0;               // blocks placed in it
    std::uint32_t pref = ipc::kNoFrame;    // the physical slab it had last
    std::uint32_t mapped = ipc::kNoFrame;  // what the shim maps there now
  };
  Key key(BlockId b) const { return Key{app_[b], static_cast<std::uint32_t>(vpos_[b] / sb_)}; }

  std::uint32_t sb_;  // blocks per slab

  std::vector<AppId> app_;
  std::vector<std::uint64_t> vpos_;
  std::map<Key, Slab> slabs_;
  std::deque<std::uint32_t> free_;  // FIFO with lazily deleted entries (is_free_)
  std::uint32_t base_;           // slabs created at start (never dropped)
  std::vector<char> is_free_;
  std::vector<std::uint32_t> gen_;
  std::set<std::uint32_t> dropped_;
  std::size_t nfree_ = 0;
  std::function<std::uint32_t()> grow_;
  std::uint32_t grown_ = 0;
  std::vector<Key> released_;
  std::vector<Key> assigned_;
};

}  // namespace nixie::b200
