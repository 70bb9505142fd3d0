// Global migration planner (include/nixie/planner.hpp).
//
// The arithmetic is a restatement of reference proj/src/planner.cpp:111-216
// and must stay bit-identical to it (plan dumps are compared byte for byte
// against oracle/_ref). The code is organised as a small staged planner:
//   1. collect fetches and the byte tallies they imply        (ref :129-144)
//   2. pinned headroom: window + transit lane, demotions       (ref :148-171)
//   3. paged allotment with a transit lane toward disk         (ref :173-196)
//   4. victim blocks in victim order, destination by budget    (ref :198-211)
//   5. canonical ordering                                      (ref :213-214)
#include <algorithm>
#include <sstream>

#include "nixie/planner.hpp"

namespace nixie {

const char* move_kind_name(MoveKind k) {
  switch (k) {
    case MoveKind::FetchForIncoming: return "fetch";
    case MoveKind::EvictFromGpu: return "evict";
    case MoveKind::Demote: return "demote";
    case MoveKind::PrefetchToPinned: return "prefetch";
  }
  return "?";
}

std::string MigrationPlan::dump() const {
  std::ostringstream os;
  for (const Move& m : moves)
    os << m.block << ' ' << tier_name(m.src) << ' ' << tier_name(m.dst) << ' ' << m.tier_distance() << ' '
       << move_kind_name(m.kind) << '\n';
  return os.str();
}

namespace {

constexpr Bytes kB = kBlockBytes;

Bytes floor_block(Bytes v) { return v - v % kB; }
Bytes ceil_block(Bytes v) { return block_count_for(v) * kB; }

// Free bytes under min(capacity, budget); kUnbounded if both are unbounded,
// 0 (not an exception) if the budget is already exceeded. ref :29-34
Bytes free_under_budget(const TierState& t, Bytes budget) {
  const Bytes limit = t.unbounded() ? budget : std::min(t.capacity, budget);
  if (limit == kUnbounded) return kUnbounded;
  const Bytes committed = t.used + t.reserved + t.window_reserved;
  return committed < limit ? limit - committed : 0;
}

// Hinted apps first (duplicates kept, as in ref :37-44), then every other app
// that owns chunks, ascending; `skip` never appears.
std::vector<AppId> eviction_order(const MemState& st, const std::vector<AppId>& hint, AppId skip) {
  std::vector<AppId> order;
  order.reserve(hint.size() + 4);
  for (AppId a : hint)
    if (a != skip) order.push_back(a);
  for (AppId a : st.apps())
    if (a != skip && std::find(order.begin(), order.end(), a) == order.end()) order.push_back(a);
  return order;
}

// An app's chunks, largest footprint first, ties by ascending id. ref :47-56
std::vector<ChunkId> chunks_largest_first(const MemState& st, AppId app) {
  std::vector<ChunkId> cs = st.chunks_of(app);
  std::stable_sort(cs.begin(), cs.end(), [&](ChunkId a, ChunkId b) {
    const Bytes fa = st.chunk(a).footprint(), fb = st.chunk(b).footprint();
    return fa != fb ? fa > fb : a < b;
  });
  return cs;
}

// Resident blocks on `tier` in victim order until `want` bytes are covered
// (possibly fewer if the tier runs dry). ref :60-76
std::vector<BlockId> victims_on(const MemState& st, const std::vector<AppId>& order, TierId tier, Bytes want) {
  std::vector<BlockId> picked;
  if (want == 0) return picked;
  const std::uint64_t need = block_count_for(want);
  for (AppId app : order)
    for (ChunkId c : chunks_largest_first(st, app))
      for (BlockId b : st.chunk(c).blocks) {
        const Location& loc = st.block(b).loc;
        if (!loc.is_resident() || loc.tier != tier) continue;
        picked.push_back(b);
        if (picked.size() >= need) return picked;
      }
  return picked;
}

// Distance-major, then kind, then block id. ref :78-85
bool canonical_before(const Move& a, const Move& b) {
  const int da = a.tier_distance(), db = b.tier_distance();
  if (da != db) return da > db;
  if (a.kind != b.kind) return static_cast<int>(a.kind) < static_cast<int>(b.kind);
  return a.block < b.block;
}

struct FetchTally {
  Bytes from_pinned = 0;  // departures that will free pinned space
  Bytes from_below = 0;   // must transit pinned on the way up
  Bytes from_paged = 0;   // departures that will free paged space
};

class SwitchPlanner {
 public:
  SwitchPlanner(AppId incoming, const MemState& st, const PlannerConfig& cfg) : in_(incoming), st_(st), cfg_(cfg) {}

  MigrationPlan run() {
    plan_.incoming_app = in_;
    check_preconditions();
    collect_fetches();
    const TierState& gpu = st_.tier(TierId::Gpu);
    const Bytes gpu_free = gpu.unbounded() ? kUnbounded : free_under_budget(gpu, kUnbounded);
    plan_.bytes_out = plan_.bytes_in > gpu_free ? plan_.bytes_in - gpu_free : 0;
    order_ = eviction_order(st_, cfg_.eviction_policy.victim_order, in_);
    size_pinned();
    size_paged();
    assign_victims();
    plan_.moves.insert(plan_.moves.end(), demotes_.begin(), demotes_.end());
    std::sort(plan_.moves.begin(), plan_.moves.end(), canonical_before);
    return std::move(plan_);
  }

 private:
  void check_preconditions() {
    if (st_.chunks_of(in_).empty()) throw SimError(Err::UnknownApp, "app " + std::to_string(in_));
    const TierState& gpu = st_.tier(TierId::Gpu);
    const Bytes fp = st_.app_footprint(in_);
    if (!gpu.unbounded() && fp > gpu.capacity)
      throw SimError(Err::AppTooLarge, "footprint " + format_bytes(fp) + " exceeds GPU " + format_bytes(gpu.capacity));
  }

  void collect_fetches() {
    for (ChunkId c : st_.chunks_of(in_))
      for (BlockId b : st_.chunk(c).blocks) {
        const Location& loc = st_.block(b).loc;
        if (!loc.is_resident()) throw SimError(Err::InvalidState, "plan requested with block in flight");
        if (loc.tier == TierId::Gpu) continue;
        plan_.moves.push_back(Move{b, loc.tier, TierId::Gpu, MoveKind::FetchForIncoming});
        plan_.bytes_in += kB;
        if (loc.tier == TierId::PinnedHost) tally_.from_pinned += kB;
        if (loc.tier == TierId::PagedHost) tally_.from_paged += kB;
        if (tier_depth(loc.tier) > tier_depth(TierId::PinnedHost)) tally_.from_below += kB;
      }
  }

  // Pinned keeps `window + transit lane` clear; demote cold pinned residents
  // when the projected free space cannot cover that headroom.
  void size_pinned() {
    const Bytes window = plan_.bytes_out > 0 ? cfg_.streaming_window : 0;
    const Bytes lane = tally_.from_below > 0 ? std::min(tally_.from_below, cfg_.streaming_window) : 0;
    const Bytes headroom = window + lane;
    const Bytes free_now = free_under_budget(st_.tier(TierId::PinnedHost), cfg_.pinned_budget);
    Bytes projected = free_now == kUnbounded ? kUnbounded : free_now + tally_.from_pinned;

    if (projected != kUnbounded && projected < headroom) {
      for (BlockId b : victims_on(st_, order_, TierId::PinnedHost, ceil_block(headroom - projected)))
        demotes_.push_back(Move{b, TierId::PinnedHost, TierId::PagedHost, MoveKind::Demote});
      projected += demotes_.size() * kB;
    }
    if (projected == kUnbounded)
      keep_pinned_ = plan_.bytes_out;
    else
      keep_pinned_ = std::min(plan_.bytes_out, projected > headroom ? projected - headroom : Bytes{0});
    keep_pinned_ = floor_block(keep_pinned_);
  }

  // What pinned cannot keep goes to paged, minus a transit lane toward disk
  // when paged overflows too; the remainder spills to disk.
  void size_paged() {
    const Bytes demoted = demotes_.size() * kB;
    Bytes room = free_under_budget(st_.tier(TierId::PagedHost), kUnbounded);
    if (room != kUnbounded) {
      room += tally_.from_paged;
      room = room > demoted ? room - demoted : 0;
    }
    const Bytes rest = plan_.bytes_out - keep_pinned_;
    if (room == kUnbounded) {
      keep_paged_ = rest;
    } else {
      keep_paged_ = std::min(rest, room);
      if (rest > keep_paged_) {
        const Bytes transit = std::min(rest - keep_paged_, cfg_.streaming_window);
        keep_paged_ = keep_paged_ > transit ? keep_paged_ - transit : 0;
      }
    }
    keep_paged_ = floor_block(keep_paged_);
    const Bytes spill = rest - keep_paged_;
    if (spill > 0 && st_.tier(TierId::Disk).capacity < spill)
      throw SimError(Err::CapacityExceeded, "hierarchy cannot absorb " + format_bytes(spill));
  }

  void assign_victims() {
    Bytes placed = 0;
    const std::vector<BlockId> picked = cfg_.gpu_victims && plan_.bytes_out
                                            ? cfg_.gpu_victims(st_, order_, plan_.bytes_out)
                                            : victims_on(st_, order_, TierId::Gpu, plan_.bytes_out);
    for (BlockId b : picked) {
      TierId dst = TierId::Disk;
      if (placed < keep_pinned_)
        dst = TierId::PinnedHost;
      else if (placed < keep_pinned_ + keep_paged_)
        dst = TierId::PagedHost;
      plan_.moves.push_back(Move{b, TierId::Gpu, dst, MoveKind::EvictFromGpu});
      placed += kB;
    }
    if (placed < plan_.bytes_out)
      throw SimError(Err::InsufficientEvictable, "only " + format_bytes(placed) + " evictable");
  }

  AppId in_;
  const MemState& st_;
  const PlannerConfig& cfg_;
  MigrationPlan plan_;
  FetchTally tally_;
  std::vector<AppId> order_;
  std::vector<Move> demotes_;
  Bytes keep_pinned_ = 0;
  Bytes keep_paged_ = 0;
};

}  // namespace

MigrationPlan plan_switch(AppId incoming, const MemState& state, const PlannerConfig& cfg) {
  return SwitchPlanner(incoming, state, cfg).run();
}

// reference planner.cpp:89-109
std::vector<ChunkId> select_evictions(Bytes bytes_needed, const MemState& state, const std::vector<AppId>& sched_hint) {
  std::vector<ChunkId> picked;
  if (bytes_needed == 0) return picked;
  Bytes got = 0;
  for (AppId app : eviction_order(state, sched_hint, kNoApp))
    for (ChunkId c : chunks_largest_first(state, app)) {
      Bytes on_gpu = 0;
      for (BlockId b : state.chunk(c).blocks) {
        const Location& loc = state.block(b).loc;
        if (loc.is_resident() && loc.tier == TierId::Gpu) on_gpu += kB;
      }
      if (on_gpu == 0) continue;
      picked.push_back(c);
      got += on_gpu;
      if (got >= bytes_needed) return picked;
    }
  throw SimError(Err::InsufficientEvictable, "need " + format_bytes(bytes_needed) + ", evictable " + format_bytes(got));
}

// reference planner.cpp:218-242
MigrationPlan plan_prefetch(AppId next, const MemState& state, const PlannerConfig& cfg) {
  MigrationPlan plan;
  plan.incoming_app = next;
  Bytes budget = free_under_budget(state.tier(TierId::PinnedHost), cfg.pinned_budget);
  if (budget != kUnbounded) {
    budget = budget > cfg.streaming_window ? budget - cfg.streaming_window : 0;
    budget = floor_block(budget);
  }
  if (budget == 0) return plan;

  Bytes planned = 0;
  auto room_for_one = [&] { return budget == kUnbounded || planned + kB <= budget; };
  for (ChunkId c : state.chunks_of(next)) {
    for (BlockId b : state.chunk(c).blocks) {
      const Location& loc = state.block(b).loc;
      if (!loc.is_resident() || tier_depth(loc.tier) <= tier_depth(TierId::PinnedHost)) continue;
      if (!room_for_one()) break;
      plan.moves.push_back(Move{b, loc.tier, TierId::PinnedHost, MoveKind::PrefetchToPinned});
      planned += kB;
    }
    if (!room_for_one()) break;
  }
  std::sort(plan.moves.begin(), plan.moves.end(), canonical_before);
  return plan;
}

}  // namespace nixie
