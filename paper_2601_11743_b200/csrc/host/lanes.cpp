// Lane state machine (see lanes.hpp for the semantics and the reference
// anchors in proj/src/transfer.cpp).
#include "lanes.hpp"

namespace nixie::detail {

LaneSet::LaneSet(MemState& mem, const HardwareConfig& hw) : mem_(mem) {
  for (int l = 0; l < kLinkCount; ++l) duplex_[l] = hw.links[l].duplex;
}

void LaneSet::set_limit(int lane, int legs) { lanes_[lane].limit = legs < 1 ? 1 : legs; }

int LaneSet::lane_of(TierId from, TierId to) const {
  const int link = std::min(tier_depth(from), tier_depth(to));
  if (duplex_[link] == Duplex::HalfDuplex) return 2 * link;
  return 2 * link + (tier_depth(to) < tier_depth(from) ? 0 : 1);
}

TierId LaneSet::next_hop(const MoveState& ms) {
  const int here = tier_depth(ms.at), goal = tier_depth(ms.move.dst);
  return tier_at_depth(goal > here ? here + 1 : here - 1);
}

// ref transfer.cpp:53-80
void LaneSet::begin(const MigrationPlan& plan, const PlannerConfig& cfg, bool gate_evictions, AppId window_owner,
                    LaneSink* sink) {
  if (active()) throw SimError(Err::InvalidState, "orchestrator already executing a plan");
  if (on_link_ != 0) throw SimError(Err::InvalidState, "legs of a cancelled plan are still on a link");
  sink_ = sink;
  moves_.clear();
  moves_.reserve(plan.moves.size());
  window_wanted_ = false;
  window_size_ = cfg.streaming_window;
  for (const Move& m : plan.moves) {
    moves_.push_back(MoveState{m, m.src, false});
    if (m.kind == MoveKind::EvictFromGpu) window_wanted_ = window_size_ > 0;
  }
  remaining_ = moves_.size();
  gate_open_ = !gate_evictions;
  window_owner_ = window_owner;
  if (remaining_ == 0) {  // empty plan: completes now, no legs, no window
    sink_->plan_finished();
    return;
  }
  try_reserve_window();
  // While the plan is loaded, a lane starts at most its first leg, exactly
  // when the reference would (pump on every push, plan order). Extra legs
  // are only considered once every lane's queue is known, so a lane cannot
  // grab space another lane's first leg needs (see startable_extra).
  loading_ = true;
  for (std::size_t i = 0; i < moves_.size(); ++i) enqueue(i);
  loading_ = false;
  pump_all();
  check_progress();
}

void LaneSet::enqueue(std::size_t mi) {
  const MoveState& ms = moves_[mi];
  const TierId hop = next_hop(ms);
  const int lane = lane_of(ms.at, hop);
  const int dir = tier_depth(hop) < tier_depth(ms.at) ? 0 : 1;
  lanes_[lane].q[dir].push_back(Entry{mi, seq_++});
  pump(lane);
}

bool LaneSet::gated(const MoveState& ms) const {
  return !gate_open_ && ms.move.kind == MoveKind::EvictFromGpu && ms.at == TierId::Gpu;
}

// ref transfer.cpp:131-143
bool LaneSet::startable(const MoveState& ms, TierId hop, bool* use_window) const {
  *use_window = false;
  if (gated(ms)) return false;
  const TierState& dst = mem_.tier(hop);
  if (dst.unbounded() || dst.free_bytes() >= kBlockBytes) return true;
  if (hop != TierId::PinnedHost || ms.move.kind != MoveKind::EvictFromGpu || !window_held_) return false;
  const auto& win = mem_.window();
  if (win && win->owner == mem_.block(ms.move.block).app && dst.window_reserved >= kBlockBytes) {
    *use_window = true;
    return true;
  }
  return false;
}

// An extra leg (its lane already has one in flight) must leave one free block
// of its destination tier for every other lane whose head targets that tier
// and that has nothing in flight: with a single leg per lane the reference
// never lets one lane take another lane's only slot, and greedy concurrency
// would (e.g. paged->pinned fetches filling a small pinned tier before any
// eviction can land there, while the fetched blocks wait for GPU frames only
// those evictions free).
bool LaneSet::extra_leaves_room(int lane, TierId hop, bool use_window) const {
  if (use_window) return true;  // drawn from the owner's window, not ordinary space
  const TierState& t = mem_.tier(hop);
  if (t.unbounded()) return true;
  std::uint64_t others = 0;
  for (int l = 0; l < kLaneCount; ++l) {
    if (l == lane) continue;
    for (const auto& q : lanes_[l].q)
      if (!q.empty() && next_hop(moves_[q.front().mi]) == hop) {
        ++others;
        break;
      }
  }
  return t.free_bytes() >= (others + 1) * kBlockBytes;
}

// Head-of-direction pump; see lanes.hpp for why it equals ref :145-171.
void LaneSet::pump(int lane, int cap) {
  Lane& L = lanes_[lane];
  while (L.inflight < std::min(L.limit, cap) && !(loading_ && L.inflight > 0)) {
    int first = 0;
    if (L.q[0].empty() || (!L.q[1].empty() && L.q[1].front().seq < L.q[0].front().seq)) first = 1;
    int pick = -1;
    bool use_window = false;
    for (int k = 0; k < 2 && pick < 0; ++k) {
      const int dir = k == 0 ? first : 1 - first;
      if (L.q[dir].empty()) continue;
      const MoveState& ms = moves_[L.q[dir].front().mi];
      const TierId hop = next_hop(ms);
      if (startable(ms, hop, &use_window) && (L.inflight == 0 || extra_leaves_room(lane, hop, use_window))) pick = dir;
    }
    if (pick < 0) return;
    const std::size_t mi = L.q[pick].front().mi;
    L.q[pick].pop_front();
    MoveState& ms = moves_[mi];
    const TierId hop = next_hop(ms);
    mem_.begin_move(ms.move.block, hop, use_window);
    ++L.inflight;
    ++on_link_;
    sink_->leg_started(lane, mi, ms.at, hop, use_window);
  }
}

void LaneSet::pump_all() {
  if (fetch_first_) {
    // Every lane's first leg in the reference's lane order (the one-leg
    // decisions), then the extra legs: toward the GPU first.
    for (int lane = 0; lane < kLaneCount; ++lane) pump(lane, 1);
    for (int dir = 0; dir < 2; ++dir)
      for (int lane = dir; lane < kLaneCount; lane += 2) pump(lane);
    return;
  }
  for (int lane = 0; lane < kLaneCount; ++lane) pump(lane);
}

void LaneSet::release_slot(int lane) {
  --lanes_[lane].inflight;
  pump(lane);
}

// ref transfer.cpp:197-225
void LaneSet::commit(std::size_t mi, TierId hop) {
  MoveState& ms = moves_[mi];
  mem_.commit_move(ms.move.block, hop);
  ms.at = hop;
  --on_link_;
  if (ms.at == ms.move.dst) {
    ms.done = true;
    --remaining_;
  } else {
    enqueue(mi);
  }
  try_reserve_window();
  pump_all();
  if (remaining_ == 0) {
    finish();
    return;
  }
  check_progress();
}

void LaneSet::finish_hop(int lane, std::size_t mi, TierId hop) {
  --lanes_[lane].inflight;
  commit(mi, hop);
}

void LaneSet::finish() {
  if (window_held_) {
    mem_.release_window();
    window_held_ = false;
  }
  sink_->plan_finished();
}

// ref transfer.cpp:82-87
void LaneSet::open_eviction_gate() {
  if (gate_open_) return;
  gate_open_ = true;
  pump_all();
  check_progress();
}

// ref transfer.cpp:89-111
void LaneSet::cancel_pending() {
  const bool was_active = remaining_ > 0;
  for (Lane& L : lanes_)
    for (auto& q : L.q) {
      for (const Entry& e : q)
        if (!moves_[e.mi].done) {
          moves_[e.mi].done = true;  // the block stays where its last committed hop left it
          --remaining_;
        }
      q.clear();
    }
  if (was_active && remaining_ == 0) finish();
}

// ref transfer.cpp:227-233
void LaneSet::try_reserve_window() {
  if (!window_wanted_ || window_held_) return;
  const TierState& pinned = mem_.tier(TierId::PinnedHost);
  if (!pinned.unbounded() && pinned.free_bytes() < window_size_) return;
  mem_.reserve_window(TierId::PinnedHost, window_size_, window_owner_);
  window_held_ = true;
}

// ref transfer.cpp:235-248
void LaneSet::check_progress() const {
  if (remaining_ == 0 || on_link_ > 0) return;
  bool pending = false;
  for (const Lane& L : lanes_)
    for (const auto& q : L.q)
      for (const Entry& e : q) {
        pending = true;
        if (gated(moves_[e.mi])) return;  // waiting on the kernel-drain gate is progress
      }
  if (pending) throw InvariantViolation("transfer deadlock: stalled legs with idle links" + describe());
}

std::string LaneSet::describe() const {
  std::string s = " [";
  for (int d = 0; d < kTierCount; ++d) {
    const TierState& t = mem_.tier(tier_at_depth(d));
    if (t.unbounded()) continue;
    s += std::string(tier_name(t.tier)) + " cap=" + std::to_string(t.capacity / kBlockBytes) +
         " used=" + std::to_string(t.used / kBlockBytes) + " rsv=" + std::to_string(t.reserved / kBlockBytes) +
         " win=" + std::to_string(t.window_reserved / kBlockBytes) + "; ";
  }
  for (int l = 0; l < kLaneCount; ++l) {
    const Lane& L = lanes_[l];
    if (L.q[0].empty() && L.q[1].empty() && L.inflight == 0) continue;
    s += "lane" + std::to_string(l) + " inflight=" + std::to_string(L.inflight) + " queued=" +
         std::to_string(L.q[0].size() + L.q[1].size());
    for (const auto& q : L.q)
      if (!q.empty()) {
        const MoveState& ms = moves_[q.front().mi];
        s += " head=blk" + std::to_string(ms.move.block) + "(" + tier_name(ms.at) + "->" + tier_name(next_hop(ms)) + ")";
      }
    s += "; ";
  }
  return s + "]";
}

}  // namespace nixie::detail
