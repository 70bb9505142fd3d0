// TEST INFRASTRUCTURE ONLY (oracle/). Linked against the UNMODIFIED
// reference library (oracle/_ref/libnixie_ref.a built from
// /root/reference/proj/src), never against the product.
//
// Independent scenario driver over the reference's public C++ API: it
// restates the context_switch step of the reference spec (
// the reference ships no engine) and prints the trace format documented in
// include/nixie/scenario.hpp, so the product's traces can be diffed against
// the reference's line by line. Reference calls used (file:line):
//   MlfqScheduler enqueue_request / infer_all / select_next / add_execution /
//     on_grant_end / victim_hint / clear_request / on_grant_start
//     (proj/src/mlfq.cpp:125-225)
//   plan_switch + MigrationPlan::dump (proj/src/planner.cpp:18-25, 111-216)
//   execute (proj/src/transfer.cpp:250-271), records per lane = the
//     occupancy log (transfer.cpp:188-195)
//   MemState::audit (proj/src/mem_model.cpp:274-325)
//
// Usage: ref_trace <scenario-file>   (or '-' for stdin)
//        ref_trace --bench <scenario-file> <switches>   time plan_switch+execute
#include <algorithm>
#include <chrono>
#include <cinttypes>
#include <cstdarg>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "nixie/mlfq.hpp"
#include "nixie/planner.hpp"
#include "nixie/transfer.hpp"

using namespace nixie;

namespace {

struct AppLine {
  AppId id;
  Bytes size;
  TierId tier;
};
struct SwitchLine {
  double t;
  AppId app;
  double busy;
};
struct Spec {
  HardwareConfig hw;
  PlannerConfig pc;
  std::vector<AppLine> apps;
  std::vector<SwitchLine> sw;
};

Spec read_spec(std::istream& in) {
  Spec s;
  s.hw.tier_capacity[3] = kUnbounded;
  std::string line;
  while (std::getline(in, line)) {
    line = line.substr(0, line.find('#'));
    std::istringstream ls(line);
    std::string op;
    if (!(ls >> op)) continue;
    std::string a, b, c, d;
    if (op == "capacity") {
      ls >> a >> b;
      s.hw.tier_capacity[static_cast<int>(parse_tier(a))] = parse_bytes(b);
    } else if (op == "link") {
      ls >> a >> b >> c >> d;
      LinkConfig& L = s.hw.links[std::stoi(a)];
      L.up_bw = parse_bandwidth(b);
      L.down_bw = parse_bandwidth(c);
      L.duplex = d == "half" ? Duplex::HalfDuplex : Duplex::FullDuplex;
    } else if (op == "dispatch") {
      ls >> a;
      s.hw.dispatch_overhead = std::stod(a);
    } else if (op == "window") {
      ls >> a;
      s.pc.streaming_window = parse_bytes(a);
    } else if (op == "budget") {
      ls >> a;
      s.pc.pinned_budget = parse_bytes(a);
    } else if (op == "app") {
      ls >> a >> b >> c;
      s.apps.push_back({static_cast<AppId>(std::stoul(a)), parse_bytes(b), parse_tier(c)});
    } else if (op == "switch") {
      ls >> a >> b >> c;
      s.sw.push_back({std::stod(a), static_cast<AppId>(std::stoul(b)), std::stod(c)});
    } else {
      throw std::runtime_error("unknown directive " + op);
    }
  }
  return s;
}

int lane_of(TierId from, TierId to) {
  int link = std::min(static_cast<int>(from), static_cast<int>(to));
  return 2 * link + (static_cast<int>(to) < static_cast<int>(from) ? 0 : 1);
}

void put(std::string& out, const char* f, ...) __attribute__((format(printf, 2, 3)));
void put(std::string& out, const char* f, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof buf, f, ap);
  va_end(ap);
  out += buf;
}

std::string run(const Spec& s) {
  MemState mem;
  s.hw.apply_to(mem);
  MlfqScheduler sched{MlfqConfig{}};
  sched.set_logging(true);
  for (const AppLine& a : s.apps) sched.register_app(a.id, 0.0);
  for (const AppLine& a : s.apps) mem.allocate(a.id, a.size, a.tier);

  std::string out;
  PlannerConfig pc = s.pc;
  double now = 0;
  bool have_runner = false;
  AppId runner = 0;
  double runner_busy = 0;
  for (std::size_t k = 0; k < s.sw.size(); ++k) {
    now = std::max(now, s.sw[k].t);
    sched.enqueue_request(s.sw[k].app, now);
    sched.infer_all(now);
    auto pick = sched.select_next(now);
    if (!pick) throw std::runtime_error("nothing selectable");
    if (have_runner) {
      sched.add_execution(runner, runner_busy);
      sched.on_grant_end(runner, now);
    }
    pc.eviction_policy.victim_order = sched.victim_hint();
    MigrationPlan plan = plan_switch(*pick, mem, pc);
    put(out, "S %zu app %u in %" PRIu64 " out %" PRIu64 " moves %zu\n", k, *pick, plan.bytes_in, plan.bytes_out,
        plan.moves.size());
    std::istringstream dump(plan.dump());
    for (std::string l; std::getline(dump, l);) put(out, "P %zu %s\n", k, l.c_str());
    const double start = now;
    ExecResult r = execute(plan, mem, s.hw, pc, now);
    std::map<int, std::vector<const TransferRecord*>> by_lane;
    for (const TransferRecord& t : r.events) by_lane[lane_of(t.src, t.dst)].push_back(&t);
    for (auto& [lane, recs] : by_lane)
      for (const TransferRecord* t : recs)
        put(out, "L %zu %d %" PRIu64 " %s %s\n", k, lane, t->block, tier_name(t->src), tier_name(t->dst));
    sched.clear_request(*pick);
    sched.on_grant_start(*pick, r.completion);
    have_runner = true;
    runner = *pick;
    runner_busy = s.sw[k].busy;
    now = r.completion;
    mem.audit();
    std::vector<BlockId> live;
    for (AppId a : mem.apps()) {
      put(out, "R %zu %u", k, a);
      for (int d = 0; d < kTierCount; ++d) put(out, " %" PRIu64, mem.app_bytes_resident(a, static_cast<TierId>(d)));
      out += "\n";
      for (ChunkId c : mem.chunks_of(a))
        for (BlockId b : mem.chunk(c).blocks) live.push_back(b);
    }
    std::sort(live.begin(), live.end());
    std::uint64_t h = 14695981039346656037ull;
    auto mix = [&h](const unsigned char* p, std::size_t n) {
      for (std::size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 1099511628211ull;
    };
    for (BlockId b : live) {
      std::uint64_t id = b;
      unsigned char t = static_cast<unsigned char>(mem.block(b).loc.tier);
      mix(reinterpret_cast<const unsigned char*>(&id), 8);
      mix(&t, 1);
    }
    put(out, "B %zu %016" PRIx64 "\n", k, h);
    put(out, "T %zu %.17g %.17g\n", k, start, r.completion);
  }
  for (const SchedLogRow& row : sched.log()) put(out, "E %u %s %d\n", row.app, row.event.c_str(), row.level);
  for (const SchedLogRow& row : sched.log())
    put(out, "G %.17g %u %s %d %.17g %.17g %.17g %.17g\n", row.time, row.app, row.event.c_str(), row.level,
        row.exec_at_level, row.idle_for, row.since_level_change, row.pending_for);
  return out;
}

// CPU-baseline timing: the reference control path (plan_switch + execute)
// for `n` round-robin switches of the scenario, after its own switch list
// has been replayed once as warm-up. Prints one line: seconds bytes.
int bench(const Spec& s, int n) {
  MemState mem;
  s.hw.apply_to(mem);
  for (const AppLine& a : s.apps) mem.allocate(a.id, a.size, a.tier);
  PlannerConfig pc = s.pc;
  std::vector<AppId> order;
  for (const auto& a : s.apps) order.push_back(a.id);
  std::size_t k = 0;
  auto one = [&](double* secs, Bytes* bytes) {
    const AppId next = order[k++ % order.size()];
    std::vector<AppId> victims;
    for (AppId a : order)
      if (a != next) victims.push_back(a);
    pc.eviction_policy.victim_order = victims;
    auto t0 = std::chrono::steady_clock::now();
    MigrationPlan plan = plan_switch(next, mem, pc);
    execute(plan, mem, s.hw, pc, 0);
    *secs += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *bytes += plan.bytes_in + plan.bytes_out;
  };
  double warm_s = 0, secs = 0;
  Bytes warm_b = 0, bytes = 0;
  for (std::size_t i = 0; i < 2 * order.size(); ++i) one(&warm_s, &warm_b);
  for (int i = 0; i < n; ++i) one(&secs, &bytes);
  std::printf("%.9f %" PRIu64 "\n", secs, bytes);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc >= 2 && std::string(argv[1]) == "--bench") {
      if (argc < 4) return 2;
      std::ifstream f(argv[2]);
      return bench(read_spec(f), std::stoi(argv[3]));
    }
    Spec s;
    if (argc < 2 || std::string(argv[1]) == "-") {
      s = read_spec(std::cin);
    } else {
      std::ifstream f(argv[1]);
      if (!f) {
        std::fprintf(stderr, "cannot open %s\n", argv[1]);
        return 2;
      }
      s = read_spec(f);
    }
    std::fputs(run(s).c_str(), stdout);
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_trace: %s\n", e.what());
    return 1;
  }
}
