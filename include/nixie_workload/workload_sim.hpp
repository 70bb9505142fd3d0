// nixie-b200 — the workload engine on the virtual clock (SPEC.md:432-503,
// module workload-sim; the reference ships the spec but no engine).
//
// Header-only and written against the `nixie` namespace API alone
// (<nixie/mem_model.hpp>, <nixie/planner.hpp>, <nixie/transfer.hpp>,
// <nixie/mlfq.hpp>), so the SAME engine compiles against this repository's
// headers (product: csrc/host/workload.cpp) and against the unmodified
// reference's headers (oracle/ref_workload.cpp, include path first). The
// schedule-and-swap trace of a workload therefore compares the two libraries'
// decisions (scheduler, planner, transfer model) under one driver: the
// north star's "sequence of swap and schedule decisions must match the
// reference's trace for the same synthetic workload", for MLFQ-driven
// workloads (config 3) as well as scripted switch lists (scenario.hpp).
//
// Application model:
//   interactive: from `start`, requests every interval*(1 +- jitter): RequestBegin,
//                `burst` kernel launches of `kernel` seconds, BlockingSync,
//                RequestEnd, Think
//   batch:       from `start`, forever: `per_sync` launches, BlockingSync
// Execution gate (the six steps of PAPER.md:116 / SPEC.md:458): a launch of an
// app that does not hold the grant (or while a switch runs) enqueues a
// schedule request and holds the app. The scheduler evaluates every tick
// (SPEC.md:354): infer_all, then a context switch to select_next() when there
// is no holder, the holder is idle, or should_preempt fires. A switch pauses
// the holder, waits for its in-flight kernels (drain), plans with the
// scheduler's victim hint, executes the plan from the drain point, and grants
// the incoming app at completion. t_a accrues per launched
// kernel of the holder. Kernels of the holder run back to back
// on one device timeline.
//
// Text format (one directive per line, '#' comments):
//   capacity <gpu|pinned|paged|disk> <bytes|unbounded>
//   link <0|1|2> <up bw> <down bw> <full|half>      dispatch <s>
//   window <bytes>    budget <bytes|unbounded>
//   mlfq <levels> <T1 s> <S1 s> <idle s> <tick s>
//   seed <u64>        horizon <s>      prefetch <on|off>
//   interactive <id> <size> <tier> <start s> <interval s> <burst> <kernel s> <jitter>
//   batch <id> <size> <tier> <start s> <kernel s> <per_sync>
//
// Trace lines (deterministic):
//   X k <decision t> <drain end> <completion> <from|-> <to>   one context switch
//   S/P/L/R/B k ...                                            as scenario.hpp
//   Q <app> <n> <begin> <first kernel done> <end>              one request
//   H <start> <app> <moves>                                    prefetch started
//   h <decision t> <quiesced t> <app>                          prefetch stopped for a switch
//
// Prefetch: with `prefetch on`,
// whenever no switch or prefetch is running, the scheduler's
// next_prefetch_candidate() (if not the holder) gets plan_prefetch()'s
// paged->pinned moves, executed by an Orchestrator on its own event queue in
// lockstep with the workload clock. A switch first cancels the prefetch's
// queued legs (cancel_pending) and waits for the legs on the link (quiesced);
// the switch's drain point is the later of the kernel drain and that.
//   E / G ...                                                  scheduler log (as scenario.hpp)
#pragma once

#include <nixie/event_queue.hpp>
#include <nixie/mem_model.hpp>
#include <nixie/mlfq.hpp>
#include <nixie/planner.hpp>
#include <nixie/transfer.hpp>

#include <algorithm>
#include <array>
#include <cinttypes>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <queue>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace nixie::workload {

struct AppSpec {
  AppId id = 0;
  Bytes size = 0;
  TierId tier = TierId::PagedHost;
  bool interactive = true;
  Seconds start = 0;
  Seconds interval = 1.0;  // interactive: think between requests
  int burst = 5;           // interactive: kernels per request
  Seconds kernel = 0.02;   // kernel duration
  double jitter = 0.0;     // interactive: +- fraction of interval
  int per_sync = 8;        // batch: launches between blocking syncs
};

struct Spec {
  HardwareConfig hw;
  PlannerConfig planner;
  MlfqConfig mlfq;
  std::uint64_t seed = 0x4E495849;
  Seconds horizon = 30.0;
  bool prefetch = false;
  std::vector<AppSpec> apps;
};

// Executes a planned switch from `now` and returns its completion; fills the
// per-lane leg sequences (6 lanes, start order). The default is the model:
// nixie::execute on the virtual clock.
using Runner = std::function<Seconds(const MigrationPlan&, MemState&, const HardwareConfig&, const PlannerConfig&,
                                     Seconds now, std::array<std::vector<std::array<std::uint64_t, 3>>, 6>& lanes)>;

struct Request {
  AppId app;
  int n;
  Seconds begin, first_done, end;
};

struct Result {
  std::string trace;
  std::vector<Request> requests;
  int switches = 0;
  Bytes bytes_in = 0, bytes_out = 0;
  Bytes prefetched = 0;  // bytes moved paged->pinned by prefetch plans (committed)
};

namespace detail {

inline void put(std::string& out, const char* f, ...) __attribute__((format(printf, 2, 3)));
inline void put(std::string& out, const char* f, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof buf, f, ap);
  va_end(ap);
  out += buf;
}

inline std::uint64_t splitmix64(std::uint64_t& s) {
  std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

inline int lane_of(TierId from, TierId to) {
  const int link = std::min(static_cast<int>(from), static_cast<int>(to));
  return 2 * link + (static_cast<int>(to) < static_cast<int>(from) ? 0 : 1);
}

}  // namespace detail

inline Spec parse(const std::string& text) {
  Spec s;
  s.hw.tier_capacity[3] = kUnbounded;
  std::istringstream in(text);
  std::string line;
  int no = 0;
  while (std::getline(in, line)) {
    ++no;
    line = line.substr(0, line.find('#'));
    std::istringstream ls(line);
    std::string op;
    if (!(ls >> op)) continue;
    auto fail = [&](const std::string& why) { throw SimError(Err::ParseError, "line " + std::to_string(no) + ": " + why); };
    std::vector<std::string> t;
    for (std::string w; ls >> w;) t.push_back(w);
    auto need = [&](std::size_t n) {
      if (t.size() != n) fail(op + " takes " + std::to_string(n) + " arguments");
    };
    if (op == "capacity") {
      need(2);
      s.hw.tier_capacity[static_cast<int>(parse_tier(t[0]))] = parse_bytes(t[1]);
    } else if (op == "link") {
      need(4);
      LinkConfig& L = s.hw.links[std::stoi(t[0])];
      L.up_bw = parse_bandwidth(t[1]);
      L.down_bw = parse_bandwidth(t[2]);
      L.duplex = t[3] == "half" ? Duplex::HalfDuplex : Duplex::FullDuplex;
    } else if (op == "dispatch") {
      need(1);
      s.hw.dispatch_overhead = std::stod(t[0]);
    } else if (op == "window") {
      need(1);
      s.planner.streaming_window = parse_bytes(t[0]);
    } else if (op == "budget") {
      need(1);
      s.planner.pinned_budget = parse_bytes(t[0]);
    } else if (op == "mlfq") {
      need(5);
      s.mlfq.levels = std::stoi(t[0]);
      s.mlfq.base_allotment = std::stod(t[1]);
      s.mlfq.base_preemption = std::stod(t[2]);
      s.mlfq.idle_threshold = std::stod(t[3]);
      s.mlfq.tick = std::stod(t[4]);
    } else if (op == "seed") {
      need(1);
      s.seed = std::stoull(t[0], nullptr, 0);
    } else if (op == "horizon") {
      need(1);
      s.horizon = std::stod(t[0]);
    } else if (op == "prefetch") {
      need(1);
      if (t[0] != "on" && t[0] != "off") fail("prefetch takes on|off");
      s.prefetch = t[0] == "on";
    } else if (op == "interactive") {
      need(8);
      AppSpec a;
      a.id = static_cast<AppId>(std::stoul(t[0]));
      a.size = parse_bytes(t[1]);
      a.tier = parse_tier(t[2]);
      a.interactive = true;
      a.start = std::stod(t[3]);
      a.interval = std::stod(t[4]);
      a.burst = std::stoi(t[5]);
      a.kernel = std::stod(t[6]);
      a.jitter = std::stod(t[7]);
      s.apps.push_back(a);
    } else if (op == "batch") {
      need(6);
      AppSpec a;
      a.id = static_cast<AppId>(std::stoul(t[0]));
      a.size = parse_bytes(t[1]);
      a.tier = parse_tier(t[2]);
      a.interactive = false;
      a.start = std::stod(t[3]);
      a.kernel = std::stod(t[4]);
      a.per_sync = std::stoi(t[5]);
      s.apps.push_back(a);
    } else {
      fail("unknown directive '" + op + "'");
    }
  }
  if (s.apps.empty()) throw SimError(Err::InvalidScenario, "workload has no apps");
  for (const AppSpec& a : s.apps) {
    if (a.kernel <= 0 || (a.interactive && (a.burst < 1 || a.interval <= 0)) || (!a.interactive && a.per_sync < 1))
      throw SimError(Err::ValidationError, "app " + std::to_string(a.id) + ": generator parameters must be positive");
    if (a.size > s.hw.tier_capacity[0])
      throw SimError(Err::ValidationError, "app " + std::to_string(a.id) + " is larger than the GPU (SPEC.md:443)");
  }
  s.mlfq.validate();
  return s;
}

inline Runner model_runner() {
  return [](const MigrationPlan& plan, MemState& mem, const HardwareConfig& hw, const PlannerConfig& cfg, Seconds now,
            std::array<std::vector<std::array<std::uint64_t, 3>>, 6>& lanes) {
    const ExecResult r = execute(plan, mem, hw, cfg, now);
    for (const TransferRecord& t : r.events)
      lanes[detail::lane_of(t.src, t.dst)].push_back(
          {t.block, static_cast<std::uint64_t>(t.src), static_cast<std::uint64_t>(t.dst)});
    return r.completion;
  };
}

// Runs the workload to its horizon. `mem` must be empty: the engine places
// every app with MemState::allocate in its initial tier (a real runner passes
// the engine's registry so the physical placement follows).
class Engine {
 public:
  Engine(const Spec& spec, MemState& mem, Runner runner = model_runner())
      : spec_(spec), mem_(mem), run_(std::move(runner)), sched_(spec.mlfq) {}

  // `allocate` places an app (default: mem.allocate).
  Result run(const std::function<void(AppId, Bytes, TierId)>& allocate = {}) {
    Result res;
    sched_.set_logging(true);
    for (const AppSpec& a : spec_.apps) {
      sched_.register_app(a.id, 0.0);
      if (allocate) allocate(a.id, a.size, a.tier);
      else mem_.allocate(a.id, a.size, a.tier);
      State st;
      st.spec = a;
      st.rng = spec_.seed ^ (static_cast<std::uint64_t>(a.id) << 32);
      apps_.emplace(a.id, st);
      push(a.start, Ev::Step, a.id);
    }
    push(spec_.mlfq.tick, Ev::Tick, 0);
    while (!q_.empty()) {
      const auto [t, seq_no, kind, app] = q_.top();
      (void)seq_no;
      q_.pop();
      if (t > spec_.horizon) break;
      now_ = t;
      if (kind == Ev::Tick) {
        tick(res);
        maybe_prefetch(res);
        push(now_ + spec_.mlfq.tick, Ev::Tick, 0);
      } else if (kind == Ev::SwitchDone) {
        switching_ = false;
        maybe_prefetch(res);
        State& s = apps_.at(app);
        if (s.held) {
          s.held = false;
          push(now_, Ev::Step, app);  // its held launch proceeds
        }
      } else {
        step(apps_.at(app), res);
      }
    }
    for (const SchedLogRow& row : sched_.log()) detail::put(res.trace, "E %u %s %d\n", row.app, row.event.c_str(), row.level);
    for (const SchedLogRow& row : sched_.log())
      detail::put(res.trace, "G %.17g %u %s %d %.17g %.17g %.17g %.17g\n", row.time, row.app, row.event.c_str(), row.level,
                  row.exec_at_level, row.idle_for, row.since_level_change, row.pending_for);
    for (const Request& r : res.requests)
      detail::put(res.trace, "Q %u %d %.17g %.17g %.17g\n", r.app, r.n, r.begin, r.first_done, r.end);
    // Pinned bytes at their physical peak over the run: resident blocks plus
    // transit, in-flight destination reservations and the streaming window
    // (MemState::pinned_physical_peak, proj/include/nixie/mem_model.hpp:128).
    detail::put(res.trace, "Z %" PRIu64 "\n", static_cast<std::uint64_t>(mem_.pinned_physical_peak()));
    return res;
  }

  const MlfqScheduler& scheduler() const { return sched_; }

 private:
  enum class Ev : int { SwitchDone = 0, Step = 1, Tick = 2 };
  using Item = std::tuple<Seconds, std::uint64_t, Ev, AppId>;
  struct Later {
    bool operator()(const Item& a, const Item& b) const {
      if (std::get<0>(a) != std::get<0>(b)) return std::get<0>(a) > std::get<0>(b);
      return std::get<1>(a) > std::get<1>(b);
    }
  };

  struct State {
    AppSpec spec;
    std::uint64_t rng = 0;
    int phase = 0;              // interactive: kernels launched in this request; batch: since last sync
    int requests = 0;
    bool in_request = false;
    bool held = false;          // waiting at the gate
    Seconds last_kernel_end = 0;
    bool in_sync = false;
    Seconds req_begin = 0;
    Seconds first_kernel_end = -1;
  };

  void push(Seconds t, Ev k, AppId a) { q_.emplace(t, seq_++, k, a); }

  // Advances the prefetch orchestrator's queue to t (events at or before t run).
  void sync_prefetch_clock(Seconds t) {
    bool hit = false;
    pq_.at(t, [&hit] { hit = true; });
    while (!hit && pq_.run_one()) {
    }
  }

  void maybe_prefetch(Result& res) {
    if (!spec_.prefetch || switching_ || orch_) return;
    const std::optional<AppId> cand = sched_.next_prefetch_candidate(now_);
    if (!cand || cand == sched_.granted()) return;
    const MigrationPlan plan = plan_prefetch(*cand, mem_, spec_.planner);
    if (plan.moves.empty()) return;
    sync_prefetch_clock(now_);
    orch_ = std::make_unique<Orchestrator>(mem_, spec_.hw, pq_, nullptr);
    pf_app_ = *cand;
    pf_bytes_ = static_cast<Bytes>(plan.moves.size()) * kBlockBytes;
    pf_done_ = false;
    orch_->begin_plan(plan, spec_.planner, false, kNoApp, [this](Seconds) { pf_done_ = true; });
    detail::put(res.trace, "H %.17g %u %zu\n", now_, *cand, plan.moves.size());
  }

  // Stops the running prefetch before a switch; returns when the link is quiet.
  Seconds quiesce_prefetch(Result& res) {
    if (!orch_) return now_;
    sync_prefetch_clock(now_);
    if (!pf_done_) {
      orch_->cancel_pending();
      while (orch_->active() && pq_.run_one()) {
      }
    }
    const Seconds quiet = std::max(now_, pq_.now());
    res.prefetched += pf_bytes_;  // upper bound: cancelled legs are not subtracted (trace shows the plan)
    detail::put(res.trace, "h %.17g %.17g %u\n", now_, quiet, pf_app_);
    orch_.reset();
    return quiet;
  }

  bool may_launch(AppId a) const {
    return !switching_ && sched_.granted() == a && mem_.app_fully_resident(a, TierId::Gpu);
  }

  // One action of app `s` at now_.
  void step(State& s, Result& res) {
    const AppSpec& a = s.spec;
    if (a.interactive && !s.in_request) {  // RequestBegin
      s.in_request = true;
      s.phase = 0;
      s.req_begin = now_;
      s.first_kernel_end = -1;
    }
    const int per = a.interactive ? a.burst : a.per_sync;
    if (s.phase < per) {  // LaunchKernel through the gate
      if (!may_launch(a.id)) {
        if (!s.held) {
          s.held = true;
          sched_.enqueue_request(a.id, now_);
        }
        return;  // resumed by SwitchDone
      }
      sched_.on_api_event(a.id, now_, ApiEventKind::NonBlockingReturn);
      const Seconds start = std::max(now_, gpu_free_);
      const Seconds end = start + a.kernel;
      gpu_free_ = end;
      s.last_kernel_end = end;
      if (s.phase == 0) s.first_kernel_end = end;
      sched_.add_execution(a.id, a.kernel);
      ++s.phase;
      push(now_, Ev::Step, a.id);  // launches are asynchronous: the next action follows at once
      return;
    }
    // BlockingSync: enter now, exit when the app's kernels are done.
    if (!s.in_sync) {
      sched_.on_api_event(a.id, now_, ApiEventKind::BlockingEnter);
      s.in_sync = true;
      push(std::max(now_, s.last_kernel_end), Ev::Step, a.id);
      return;
    }
    s.in_sync = false;
    sched_.on_api_event(a.id, now_, ApiEventKind::BlockingExit);
    s.phase = 0;
    if (a.interactive) {  // RequestEnd, then Think
      res.requests.push_back(Request{a.id, s.requests++, s.req_begin, s.first_kernel_end, now_});
      s.in_request = false;
      double gap = a.interval;
      if (a.jitter > 0) {
        const double u = static_cast<double>(detail::splitmix64(s.rng) >> 11) * (1.0 / 9007199254740992.0);
        gap *= 1.0 + a.jitter * (2.0 * u - 1.0);
      }
      push(now_ + gap, Ev::Step, a.id);
    } else {
      push(now_, Ev::Step, a.id);
    }
  }

  void tick(Result& res) {
    if (switching_) return;
    sched_.infer_all(now_);
    const std::optional<AppId> next = sched_.select_next(now_);
    if (!next) return;
    const std::optional<AppId> holder = sched_.granted();
    const bool go = !holder || sched_.is_idle(*holder, now_) || sched_.should_preempt(*holder, now_);
    if (go) context_switch(holder, *next, res);
  }

  void context_switch(const std::optional<AppId>& holder, AppId to, Result& res) {
    const std::size_t k = static_cast<std::size_t>(res.switches++);
    const Seconds decided = now_;
    Seconds drained = now_;
    if (holder) {
      drained = std::max(now_, apps_.at(*holder).last_kernel_end);  // in-flight kernels finish
      sched_.on_grant_end(*holder, now_);
    }
    drained = std::max(drained, quiesce_prefetch(res));
    PlannerConfig cfg = spec_.planner;
    cfg.eviction_policy.victim_order = sched_.victim_hint();
    const MigrationPlan plan = plan_switch(to, mem_, cfg);
    detail::put(res.trace, "S %zu app %u in %" PRIu64 " out %" PRIu64 " moves %zu\n", k, to, plan.bytes_in,
                plan.bytes_out, plan.moves.size());
    {
      std::istringstream d(plan.dump());
      for (std::string l; std::getline(d, l);) detail::put(res.trace, "P %zu %s\n", k, l.c_str());
    }
    std::array<std::vector<std::array<std::uint64_t, 3>>, 6> lanes;
    const Seconds done = run_(plan, mem_, spec_.hw, cfg, drained, lanes);
    for (int lane = 0; lane < 6; ++lane)
      for (const auto& leg : lanes[lane])
        detail::put(res.trace, "L %zu %d %" PRIu64 " %s %s\n", k, lane, leg[0], tier_name(static_cast<TierId>(leg[1])),
                    tier_name(static_cast<TierId>(leg[2])));
    res.bytes_in += plan.bytes_in;
    res.bytes_out += plan.bytes_out;
    sched_.clear_request(to);
    sched_.on_grant_start(to, done);
    switching_ = true;
    gpu_free_ = std::max(gpu_free_, done);
    push(done, Ev::SwitchDone, to);
    mem_.audit();
    std::vector<BlockId> live;
    for (AppId a : mem_.apps()) {
      detail::put(res.trace, "R %zu %u", k, a);
      for (int d = 0; d < kTierCount; ++d) detail::put(res.trace, " %" PRIu64, mem_.app_bytes_resident(a, static_cast<TierId>(d)));
      res.trace += "\n";
      for (ChunkId c : mem_.chunks_of(a))
        for (BlockId b : mem_.chunk(c).blocks) live.push_back(b);
    }
    std::sort(live.begin(), live.end());
    std::uint64_t h = 14695981039346656037ull;
    for (BlockId b : live) {
      const std::uint64_t id = b;
      const auto t = static_cast<unsigned char>(mem_.block(b).loc.tier);
      for (int i = 0; i < 8; ++i) h = (h ^ ((id >> (8 * i)) & 0xFF)) * 1099511628211ull;
      h = (h ^ t) * 1099511628211ull;
    }
    detail::put(res.trace, "B %zu %016" PRIx64 "\n", k, h);
    if (holder) detail::put(res.trace, "X %zu %.17g %.17g %.17g %u %u\n", k, decided, drained, done, *holder, to);
    else detail::put(res.trace, "X %zu %.17g %.17g %.17g - %u\n", k, decided, drained, done, to);
  }

  const Spec& spec_;
  MemState& mem_;
  Runner run_;
  MlfqScheduler sched_;
  std::map<AppId, State> apps_;
  std::priority_queue<Item, std::vector<Item>, Later> q_;
  std::uint64_t seq_ = 0;
  Seconds now_ = 0;
  Seconds gpu_free_ = 0;
  bool switching_ = false;
  EventQueue pq_;                         // the prefetch orchestrator's clock
  std::unique_ptr<Orchestrator> orch_;    // running prefetch plan
  AppId pf_app_ = kNoApp;
  Bytes pf_bytes_ = 0;
  bool pf_done_ = false;
};

}  // namespace nixie::workload
