// Lane state machine shared by the modeled Orchestrator and the CUDA
// SwapEngine (internal header).
//
// Semantics follow reference proj/src/transfer.cpp:53-248:
//   * lane = 2*link + (up ? 0 : 1); a half-duplex link shares lane 2*link
//     (lane_index, ref :39-45); multi-tier moves go one adjacent hop at a time
//     (next_hop, ref :47-51);
//   * per lane and direction the queue is FIFO; a leg starts iff the eviction
//     gate lets it (ref :126-129) and its destination has a free block or the
//     streaming window admits an owner's eviction (ref :131-143);
//   * a commit applies MemState::commit_move, enqueues the next hop, retries
//     the lazy window reservation and pumps every lane (ref :197-225);
//   * nothing on any link with legs pending and none gated is a deadlock
//     (ref :235-248).
// Two deliberate differences, neither observable in decisions:
//   * pump() looks only at the head of each direction's deque. The reference
//     scans the whole lane deque every time (O(n) per pump, O(n^2) per switch
//     when the GPU is full: 152 ms of host time at 16 GiB);
//     because a stalled head blocks its whole direction, the first startable
//     leg of a direction can only be its head, so the decisions are the same.
//   * a lane may carry up to `limit` legs at once (the reference: 1). The
//     start order per lane is still the FIFO order, so per-lane leg sequences
//     match the reference; only timing-dependent details (window use of a
//     given leg, cross-lane interleaving) can differ.
#pragma once

#include <array>
#include <cstdint>
#include <deque>
#include <vector>

#include "nixie/transfer.hpp"

namespace nixie::detail {

inline constexpr int kLaneCount = 2 * kLinkCount;

// Backend callbacks.
class LaneSink {
 public:
  virtual ~LaneSink() = default;
  // MemState::begin_move(block, to, use_window) has been applied.
  virtual void leg_started(int lane, std::size_t move_index, TierId from, TierId to, bool use_window) = 0;
  // Every move committed (or was cancelled); the window is released.
  virtual void plan_finished() = 0;
};

class LaneSet {
 public:
  LaneSet(MemState& mem, const HardwareConfig& hw);

  void set_limit(int lane, int legs);
  // Concurrent lanes only: after a commit, start every lane's first leg in
  // lane order (as the reference would, transfer.cpp:217-221), then the
  // extra legs of the lanes toward the GPU (0, 2, 4) before the others. In
  // plain lane order, with many legs per lane, the evictions into the pinned
  // tier (lane 1) take every slot that frees, and the fetches' first hop into
  // it (lane 2) starves until they are done: the two halves of a two-hop
  // switch run one after the other. Per-lane FIFO order, and so the
  // decisions, are the same either way.
  void set_fetch_first(bool on) { fetch_first_ = on; }
  int limit(int lane) const { return lanes_[lane].limit; }

  void begin(const MigrationPlan& plan, const PlannerConfig& cfg, bool gate_evictions, AppId window_owner,
             LaneSink* sink);
  // A lane slot is free again (link occupancy ended); pumps that lane.
  void release_slot(int lane);
  // The hop of move `mi` to `hop` has landed: commit, enqueue the next hop,
  // pump everything, detect completion / deadlock.
  void commit(std::size_t mi, TierId hop);
  // Real executors: the copy of a hop finished, so its lane slot frees and
  // the hop commits in one step.
  void finish_hop(int lane, std::size_t mi, TierId hop);
  void open_eviction_gate();
  void cancel_pending();

  bool active() const { return remaining_ > 0; }
  bool quiesced() const { return on_link_ == 0; }
  int legs_on_link() const { return on_link_; }
  int in_flight(int lane) const { return lanes_[lane].inflight; }
  std::size_t queued(int lane) const { return lanes_[lane].q[0].size() + lanes_[lane].q[1].size(); }

  const Move& move(std::size_t mi) const { return moves_[mi].move; }
  TierId at(std::size_t mi) const { return moves_[mi].at; }
  TierId hop_of(std::size_t mi) const { return next_hop(moves_[mi]); }
  std::size_t move_count() const { return moves_.size(); }
  int lane_of(TierId from, TierId to) const;
  bool window_held() const { return window_held_; }
  std::string describe() const;  // tiers + lane heads, for deadlock reports

 private:
  struct MoveState {
    Move move;
    TierId at;
    bool done = false;
  };
  struct Entry {
    std::size_t mi;
    std::uint64_t seq;
  };
  struct Lane {
    std::deque<Entry> q[2];  // [0] up (toward GPU), [1] down
    int inflight = 0;
    int limit = 1;
  };

  static TierId next_hop(const MoveState& ms);
  void enqueue(std::size_t mi);
  void pump(int lane, int cap = 1 << 30);  // starts legs while fewer than min(limit, cap) are in flight
  void pump_all();
  bool gated(const MoveState& ms) const;
  bool startable(const MoveState& ms, TierId hop, bool* use_window) const;
  bool extra_leaves_room(int lane, TierId hop, bool use_window) const;
  void try_reserve_window();
  void check_progress() const;
  void finish();

  MemState& mem_;
  std::array<Duplex, kLinkCount> duplex_{};
  std::vector<MoveState> moves_;
  std::array<Lane, kLaneCount> lanes_{};
  LaneSink* sink_ = nullptr;
  std::size_t remaining_ = 0;
  int on_link_ = 0;
  std::uint64_t seq_ = 0;
  bool gate_open_ = true;
  bool loading_ = false;  // begin(): first legs only
  bool fetch_first_ = false;
  bool window_wanted_ = false;
  bool window_held_ = false;
  Bytes window_size_ = 0;
  AppId window_owner_ = kNoApp;
};

}  // namespace nixie::detail
