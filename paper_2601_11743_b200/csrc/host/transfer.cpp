// Modeled executor (parity mode) over the shared lane state machine, plus
// the throughput metric and the one-shot execute() wrapper.
// Reference: proj/src/transfer.cpp.
#include <algorithm>

#include "lanes.hpp"
#include "nixie/transfer.hpp"

namespace nixie {

// reference transfer.cpp:7-28
ThroughputSample aggregate_throughput(const std::vector<TransferRecord>& log, Seconds t0, Seconds t1) {
  ThroughputSample out;
  if (!(t1 > t0)) return out;
  double up = 0, down = 0;
  for (const TransferRecord& r : log) {
    const bool pcie = (r.src == TierId::Gpu && r.dst == TierId::PinnedHost) ||
                      (r.src == TierId::PinnedHost && r.dst == TierId::Gpu);
    if (!pcie || !(r.end > r.start)) continue;
    const Seconds overlap = std::min(r.end, t1) - std::max(r.start, t0);
    if (overlap <= 0) continue;
    const double share = static_cast<double>(r.bytes) * overlap / (r.end - r.start);
    (r.dst == TierId::Gpu ? up : down) += share;
  }
  const Seconds span = t1 - t0;
  out.to_gpu = up / span;
  out.from_gpu = down / span;
  out.bidirectional = (up + down) / span;
  return out;
}

WindowHandle reserve_streaming_window(MemState& mem, TierId tier, Bytes size, AppId owner) {
  mem.reserve_window(tier, size, owner);
  return WindowHandle{tier, size, owner};
}

// Link model: a leg occupies its lane for kBlockBytes / bw, its commit lands
// dispatch_overhead later (ref transfer.cpp:173-195).
class Orchestrator::ModelLinks final : public detail::LaneSink {
 public:
  ModelLinks(const HardwareConfig& hw, EventQueue& q, std::vector<TransferRecord>* log) : hw_(hw), q_(q), log_(log) {}

  void bind(detail::LaneSet* lanes) { lanes_ = lanes; }
  void set_callback(std::function<void(Seconds)> cb) { cb_ = std::move(cb); }

  void leg_started(int lane, std::size_t mi, TierId from, TierId to, bool) override {
    const int link = std::min(tier_depth(from), tier_depth(to));
    const bool up = tier_depth(to) < tier_depth(from);
    const Bandwidth bw = up ? hw_.links[link].up_bw : hw_.links[link].down_bw;
    const Seconds started = q_.now();
    q_.after(static_cast<Seconds>(kBlockBytes) / bw, [this, lane, mi, from, to, started] {
      if (log_) log_->push_back(TransferRecord{started, q_.now(), lanes_->move(mi).block, from, to, kBlockBytes});
      lanes_->release_slot(lane);
      q_.after(hw_.dispatch_overhead, [this, mi, to] { lanes_->commit(mi, to); });
    });
  }

  void plan_finished() override {
    if (!cb_) return;
    auto cb = std::move(cb_);
    cb_ = nullptr;
    const Seconds t = q_.now();
    q_.at(t, [cb, t] { cb(t); });
  }

 private:
  HardwareConfig hw_;
  EventQueue& q_;
  std::vector<TransferRecord>* log_;
  detail::LaneSet* lanes_ = nullptr;
  std::function<void(Seconds)> cb_;
};

Orchestrator::Orchestrator(MemState& mem, const HardwareConfig& hw, EventQueue& queue, std::vector<TransferRecord>* log)
    : links_(std::make_unique<ModelLinks>(hw, queue, log)), lanes_(std::make_unique<detail::LaneSet>(mem, hw)) {
  links_->bind(lanes_.get());
}

Orchestrator::~Orchestrator() = default;

void Orchestrator::begin_plan(const MigrationPlan& plan, const PlannerConfig& cfg, bool gate_evictions,
                              AppId window_owner, std::function<void(Seconds)> on_complete) {
  if (lanes_->active()) throw SimError(Err::InvalidState, "orchestrator already executing a plan");
  links_->set_callback(std::move(on_complete));
  lanes_->begin(plan, cfg, gate_evictions, window_owner, links_.get());
}

void Orchestrator::open_eviction_gate() { lanes_->open_eviction_gate(); }
void Orchestrator::cancel_pending() { lanes_->cancel_pending(); }
bool Orchestrator::active() const { return lanes_->active(); }
bool Orchestrator::quiesced() const { return lanes_->quiesced(); }

void Orchestrator::set_lane_concurrency(int legs_per_lane) {
  for (int lane = 0; lane < detail::kLaneCount; ++lane) lanes_->set_limit(lane, legs_per_lane);
  lanes_->set_fetch_first(legs_per_lane > 1);
}

// reference transfer.cpp:250-271
ExecResult execute(const MigrationPlan& plan, MemState& mem, const HardwareConfig& hw, const PlannerConfig& cfg,
                   Seconds start) {
  ExecResult res;
  EventQueue q;
  Orchestrator orch(mem, hw, q, &res.events);
  AppId owner = kNoApp;
  auto ev = std::find_if(plan.moves.begin(), plan.moves.end(),
                         [](const Move& m) { return m.kind == MoveKind::EvictFromGpu; });
  if (ev != plan.moves.end()) owner = mem.block(ev->block).app;
  bool finished = false;
  q.at(start, [&] {
    orch.begin_plan(plan, cfg, /*gate_evictions=*/false, owner, [&](Seconds t) {
      res.completion = t;
      finished = true;
    });
  });
  q.run_all();
  if (!finished) throw InvariantViolation("plan did not complete");
  return res;
}

}  // namespace nixie
