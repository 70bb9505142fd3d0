// nixie-b200 — minimal workload driver: the `context_switch` subset of the
// reference spec's workload-sim (absent from the reference
// code), used to produce the swap + schedule trace that the parity contract
// compares.
//
// Scenario text (one directive per line, '#' comments):
//   capacity <gpu|pinned|paged|disk> <bytes|unbounded>
//   link <0|1|2> <up bw> <down bw> <full|half>
//   dispatch <seconds>
//   window <bytes>            budget <bytes|unbounded>
//   app <id> <size> <gpu|pinned|paged>
//   switch <time> <app> <busy seconds>
//
// Each `switch` at virtual time t: now = max(t, previous completion);
// enqueue_request(app); infer_all(now); next = select_next(now); the current
// grant holder gets add_execution(busy) and on_grant_end(now); the planner
// uses victim_hint() as the victim order; plan_switch; execute from `now`;
// clear_request(next); on_grant_start(next, completion); audit().
//
// Trace lines (all deterministic except where noted):
//   S k app <id> in <bytes> out <bytes> moves <n>     switch header
//   P k <block> <src> <dst> <distance> <kind>        plan dump
//   L k <lane> <block> <src> <dst>                   per-lane leg sequence
//   R k <app> <gpu> <pinned> <paged> <disk>          resident bytes per tier after the switch
//   B k <fnv64 of (block, tier) over all live blocks>
//   E <app> <event> <level>                          scheduler log, time-free
//   T k <start> <completion>                         virtual-clock only
//   G <time> <app> <event> <level> <t> <i> <p> <q>   scheduler log rows, virtual-clock only
#pragma once

#include <array>
#include <functional>
#include <string>
#include <vector>

#include "nixie/mem_model.hpp"
#include "nixie/mlfq.hpp"
#include "nixie/planner.hpp"
#include "nixie/transfer.hpp"

namespace nixie {

struct ScenarioApp {
  AppId id = 0;
  Bytes size = 0;
  TierId tier = TierId::PagedHost;
};

struct ScenarioSwitch {
  Seconds time = 0;
  AppId app = 0;
  Seconds busy = 0;
};

struct Scenario {
  HardwareConfig hw;
  PlannerConfig planner;
  MlfqConfig mlfq;
  std::vector<ScenarioApp> apps;
  std::vector<ScenarioSwitch> switches;
};

Scenario parse_scenario(const std::string& text);  // ParseError / InvalidScenario

// How a planned switch gets executed. The model executor is
// nixie::execute on the virtual clock; the CUDA engine supplies a real one.
struct SwitchRunner {
  std::function<MemState&()> mem;
  // Runs `plan` starting at `now`; returns the completion time and fills the
  // per-lane leg sequences (6 lanes, start order).
  std::function<Seconds(const MigrationPlan&, const PlannerConfig&, Seconds now,
                        std::array<std::vector<std::array<std::uint64_t, 3>>, 6>& lanes)>
      run;
  bool virtual_clock = true;
  std::function<void(std::size_t k, AppId incoming, std::string& trace)> after_switch;  // optional extra lines
};

// Drives the scenario; the registry must already hold the scenario's apps.
std::string drive_scenario(const Scenario& sc, SwitchRunner& runner);

// Model-mode convenience: builds MemState from the scenario and runs it on
// the virtual clock with reference-identical link timing.
// legs_per_lane > 1 runs the lanes with the CUDA engine's concurrency
// (Orchestrator::set_lane_concurrency); times then differ from the
// reference, decisions must not.
std::string run_scenario_model(const Scenario& sc, int legs_per_lane = 1);

// Lane of a single hop (full-duplex layout, reference transfer.cpp:39-45).
int lane_for(TierId from, TierId to);

}  // namespace nixie
