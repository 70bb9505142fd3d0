// Minimal workload driver (include/nixie/scenario.hpp).
#include "nixie/scenario.hpp"

#include <algorithm>
#include <cinttypes>
#include <cstdarg>
#include <cstdio>
#include <sstream>

namespace nixie {

namespace {

std::string fmt(const char* f, ...) __attribute__((format(printf, 1, 2)));
std::string fmt(const char* f, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, f);
  std::vsnprintf(buf, sizeof(buf), f, ap);
  va_end(ap);
  return buf;
}

Seconds parse_seconds(const std::string& s, int line) {
  try {
    std::size_t pos = 0;
    const double v = std::stod(s, &pos);
    if (pos != s.size()) throw std::invalid_argument(s);
    return v;
  } catch (const std::exception&) {
    throw SimError(Err::ParseError, "line " + std::to_string(line) + ": bad number '" + s + "'");
  }
}

std::uint64_t fnv1a(std::uint64_t h, const void* p, std::size_t n) {
  const auto* b = static_cast<const unsigned char*>(p);
  for (std::size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

}  // namespace

int lane_for(TierId from, TierId to) {
  const int link = std::min(tier_depth(from), tier_depth(to));
  return 2 * link + (tier_depth(to) < tier_depth(from) ? 0 : 1);
}

Scenario parse_scenario(const std::string& text) {
  Scenario sc;
  sc.hw.tier_capacity[3] = kUnbounded;
  std::istringstream in(text);
  std::string raw;
  int line = 0;
  while (std::getline(in, raw)) {
    ++line;
    if (auto h = raw.find('#'); h != std::string::npos) raw.resize(h);
    std::istringstream ls(raw);
    std::vector<std::string> tok;
    for (std::string t; ls >> t;) tok.push_back(t);
    if (tok.empty()) continue;
    const std::string& op = tok[0];
    auto need = [&](std::size_t n) {
      if (tok.size() != n) throw SimError(Err::ParseError, "line " + std::to_string(line) + ": '" + op + "' expects " + std::to_string(n - 1) + " fields");
    };
    if (op == "capacity") {
      need(3);
      sc.hw.tier_capacity[tier_depth(parse_tier(tok[1]))] = parse_bytes(tok[2]);
    } else if (op == "link") {
      need(5);
      const int l = static_cast<int>(parse_seconds(tok[1], line));
      if (l < 0 || l >= kLinkCount) throw SimError(Err::ParseError, "line " + std::to_string(line) + ": bad link");
      sc.hw.links[l].up_bw = parse_bandwidth(tok[2]);
      sc.hw.links[l].down_bw = parse_bandwidth(tok[3]);
      sc.hw.links[l].duplex = tok[4] == "half" ? Duplex::HalfDuplex : Duplex::FullDuplex;
    } else if (op == "dispatch") {
      need(2);
      sc.hw.dispatch_overhead = parse_seconds(tok[1], line);
    } else if (op == "window") {
      need(2);
      sc.planner.streaming_window = parse_bytes(tok[1]);
    } else if (op == "budget") {
      need(2);
      sc.planner.pinned_budget = parse_bytes(tok[1]);
    } else if (op == "app") {
      need(4);
      sc.apps.push_back(ScenarioApp{static_cast<AppId>(parse_seconds(tok[1], line)), parse_bytes(tok[2]), parse_tier(tok[3])});
    } else if (op == "switch") {
      need(4);
      sc.switches.push_back(
          ScenarioSwitch{parse_seconds(tok[1], line), static_cast<AppId>(parse_seconds(tok[2], line)), parse_seconds(tok[3], line)});
    } else {
      throw SimError(Err::ParseError, "line " + std::to_string(line) + ": unknown directive '" + op + "'");
    }
  }
  if (sc.apps.empty()) throw SimError(Err::InvalidScenario, "scenario has no apps");
  return sc;
}

std::string drive_scenario(const Scenario& sc, SwitchRunner& runner) {
  MemState& mem = runner.mem();
  MlfqScheduler sched(sc.mlfq);
  sched.set_logging(true);
  for (const ScenarioApp& a : sc.apps) sched.register_app(a.id, 0.0);

  std::string out;
  PlannerConfig cfg = sc.planner;
  Seconds now = 0;
  std::optional<AppId> running;
  Seconds running_busy = 0;
  for (std::size_t k = 0; k < sc.switches.size(); ++k) {
    const ScenarioSwitch& sw = sc.switches[k];
    now = std::max(now, sw.time);
    sched.enqueue_request(sw.app, now);
    sched.infer_all(now);
    const std::optional<AppId> next = sched.select_next(now);
    if (!next) throw SimError(Err::InvalidScenario, "switch " + std::to_string(k) + ": nothing selectable");
    if (running) {
      sched.add_execution(*running, running_busy);
      sched.on_grant_end(*running, now);
    }
    cfg.eviction_policy.victim_order = sched.victim_hint();
    const MigrationPlan plan = plan_switch(*next, mem, cfg);
    out += fmt("S %zu app %u in %" PRIu64 " out %" PRIu64 " moves %zu\n", k, *next, plan.bytes_in, plan.bytes_out,
               plan.moves.size());
    {
      std::istringstream d(plan.dump());
      for (std::string l; std::getline(d, l);) out += fmt("P %zu ", k) + l + "\n";
    }
    std::array<std::vector<std::array<std::uint64_t, 3>>, 6> lanes;
    const Seconds start = now;
    const Seconds done = runner.run(plan, cfg, now, lanes);
    for (int lane = 0; lane < 6; ++lane)
      for (const auto& leg : lanes[lane])
        out += fmt("L %zu %d %" PRIu64 " %s %s\n", k, lane, leg[0], tier_name(static_cast<TierId>(leg[1])),
                   tier_name(static_cast<TierId>(leg[2])));
    sched.clear_request(*next);
    sched.on_grant_start(*next, done);
    running = *next;
    running_busy = sw.busy;
    now = done;
    mem.audit();
    std::vector<BlockId> live;
    for (AppId a : mem.apps()) {
      out += fmt("R %zu %u", k, a);
      for (int d = 0; d < kTierCount; ++d) out += fmt(" %" PRIu64, mem.app_bytes_resident(a, tier_at_depth(d)));
      out += "\n";
      for (ChunkId c : mem.chunks_of(a))
        for (BlockId b : mem.chunk(c).blocks) live.push_back(b);
    }
    std::sort(live.begin(), live.end());
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (BlockId b : live) {
      const std::uint64_t id = b;
      const auto t = static_cast<std::uint8_t>(mem.block(b).loc.tier);
      h = fnv1a(h, &id, sizeof(id));
      h = fnv1a(h, &t, sizeof(t));
    }
    out += fmt("B %zu %016" PRIx64 "\n", k, h);
    if (runner.virtual_clock) out += fmt("T %zu %.17g %.17g\n", k, start, done);
    if (runner.after_switch) runner.after_switch(k, *next, out);
  }
  for (const SchedLogRow& r : sched.log()) out += fmt("E %u %s %d\n", r.app, r.event.c_str(), r.level);
  if (runner.virtual_clock)
    for (const SchedLogRow& r : sched.log())
      out += fmt("G %.17g %u %s %d %.17g %.17g %.17g %.17g\n", r.time, r.app, r.event.c_str(), r.level, r.exec_at_level,
                 r.idle_for, r.since_level_change, r.pending_for);
  return out;
}

namespace {
// execute() with a lane-concurrency override (reference transfer.cpp:250-271).
ExecResult execute_lanes(const MigrationPlan& plan, MemState& mem, const HardwareConfig& hw, const PlannerConfig& cfg,
                         Seconds start, int legs_per_lane) {
  if (legs_per_lane <= 1) return execute(plan, mem, hw, cfg, start);
  ExecResult res;
  EventQueue q;
  Orchestrator orch(mem, hw, q, &res.events);
  orch.set_lane_concurrency(legs_per_lane);
  AppId owner = kNoApp;
  for (const Move& m : plan.moves)
    if (m.kind == MoveKind::EvictFromGpu) {
      owner = mem.block(m.block).app;
      break;
    }
  bool finished = false;
  q.at(start, [&] {
    orch.begin_plan(plan, cfg, false, owner, [&](Seconds t) {
      res.completion = t;
      finished = true;
    });
  });
  q.run_all();
  if (!finished) throw InvariantViolation("plan did not complete");
  // With several legs per lane, records land in completion order; restore
  // per-lane start order.
  std::stable_sort(res.events.begin(), res.events.end(),
                   [](const TransferRecord& a, const TransferRecord& b) { return a.start < b.start; });
  return res;
}
}  // namespace

std::string run_scenario_model(const Scenario& sc, int legs_per_lane) {
  MemState mem;
  sc.hw.apply_to(mem);
  for (const ScenarioApp& a : sc.apps) mem.allocate(a.id, a.size, a.tier);
  SwitchRunner runner;
  runner.mem = [&]() -> MemState& { return mem; };
  runner.run = [&](const MigrationPlan& plan, const PlannerConfig& cfg, Seconds now,
                   std::array<std::vector<std::array<std::uint64_t, 3>>, 6>& lanes) {
    ExecResult r = execute_lanes(plan, mem, sc.hw, cfg, now, legs_per_lane);
    // Records are logged at occupancy end; per lane that is start order.
    for (const TransferRecord& t : r.events)
      lanes[lane_for(t.src, t.dst)].push_back(
          {t.block, static_cast<std::uint64_t>(t.src), static_cast<std::uint64_t>(t.dst)});
    return r.completion;
  };
  runner.virtual_clock = true;
  return drive_scenario(sc, runner);
}

}  // namespace nixie
