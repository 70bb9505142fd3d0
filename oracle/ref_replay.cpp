// TEST INFRASTRUCTURE ONLY (oracle/). Linked against the UNMODIFIED
// reference library (oracle/_ref/libnixie_ref.a built from
// /root/reference/proj/src), never against the product.
//
// Replays the interposer daemon's registry + plan trace (nixied --trace,
// csrc/daemon/daemon.cpp trace_*) on the reference, switch by switch:
//   alloc APP BYTES TIER CHUNKS...  MemState::allocate (proj/src/mem_model.cpp:48-86);
//                                   the chunk ids must be the daemon's
//   free APP CHUNK                  MemState::free_chunk (mem_model.cpp:88-116)
//   prefetch K APP moves N           + its Q (dump) lines: the reference's
//                                    plan_prefetch(APP) on the same state
//                                    (planner.cpp:218-242) is printed as F lines
//   pcommit BLOCK                    a prefetch leg (paged -> pinned) that
//                                    committed: begin_move + commit_move
//                                    (mem_model.cpp:118-172)
//   plan K KIND APP in I out O victims V...   + its P (dump) and L (lane) lines
//       -> the reference's plan_switch(APP) on the same state with the same
//          victim order (proj/src/planner.cpp:111-216): printed as S/P/A lines;
//          then the DAEMON's plan (rebuilt from its P lines) runs through the
//          reference execute() (proj/src/transfer.cpp:250-271) so both
//          registries stay identical; its per-lane leg order is printed as L
//          lines (transfer.cpp:188-195 records) and MemState::audit() runs.
// Output per plan K:
//   S K APP IN OUT          the reference plan's totals
//   P K <dump line>         the reference plan (MigrationPlan::dump, planner.cpp:18-25)
//   A K ref|daemon APPS...  victim apps in order of their first eviction
//   L K LANE BLOCK SRC DST  reference execution of the daemon's plan
//   F K <dump line>         the reference's prefetch plan K
// With `victims reference` the daemon runs the planner unmodified, so its P
// and L lines must equal these; with `victims slab` (slab-aligned victim
// blocks) totals and victim app order must match while blocks may differ.
//
// Usage: ref_replay <trace-file>
#include <cinttypes>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "nixie/planner.hpp"
#include "nixie/transfer.hpp"

using namespace nixie;

namespace {

MoveKind parse_kind(const std::string& k) {
  if (k == "fetch") return MoveKind::FetchForIncoming;
  if (k == "evict") return MoveKind::EvictFromGpu;
  if (k == "demote") return MoveKind::Demote;
  if (k == "prefetch") return MoveKind::PrefetchToPinned;
  throw std::runtime_error("unknown move kind " + k);
}

int lane_of(TierId from, TierId to) {
  const int link = std::min(tier_depth(from), tier_depth(to));
  return 2 * link + (tier_depth(to) < tier_depth(from) ? 0 : 1);
}

std::vector<AppId> victim_apps(const MigrationPlan& plan, const MemState& mem) {
  std::vector<AppId> out;
  for (const Move& m : plan.moves) {
    if (m.kind != MoveKind::EvictFromGpu) continue;
    const AppId a = mem.block(m.block).app;
    bool seen = false;
    for (AppId x : out) seen = seen || x == a;
    if (!seen) out.push_back(a);
  }
  return out;
}

struct PendingPlan {
  bool open = false;
  std::uint64_t k = 0;
  AppId app = 0;
  Bytes in = 0, out = 0;
  std::vector<AppId> victims;
  MigrationPlan daemon;
};

class Replay {
 public:
  Replay() { hw_.tier_capacity[3] = kUnbounded; }

  void line(const std::string& raw) {
    std::istringstream ls(raw);
    std::string op;
    if (!(ls >> op)) return;
    if (op == "Q") return;  // the daemon's prefetch plan: compared by the test
    if (op == "P" || op == "L") {
      if (!cur_.open) throw std::runtime_error("P/L line outside a plan");
      if (op == "P") {
        std::uint64_t k;
        std::string blk, src, dst, dist, kind;
        ls >> k >> blk >> src >> dst >> dist >> kind;
        Move m;
        m.block = std::stoull(blk);
        m.src = parse_tier(src);
        m.dst = parse_tier(dst);
        m.kind = parse_kind(kind);
        cur_.daemon.moves.push_back(m);
      }
      return;  // the daemon's own L lines are compared by the test
    }
    flush();
    if (op == "capacity") {
      std::string t;
      Bytes v;
      ls >> t >> v;
      hw_.tier_capacity[tier_depth(parse_tier(t))] = v;
      hw_.apply_to(mem_);
    } else if (op == "window") {
      ls >> pc_.streaming_window;
    } else if (op == "budget") {
      ls >> pc_.pinned_budget;
    } else if (op == "victims") {
      ls >> mode_;
    } else if (op == "alloc") {
      unsigned app;
      Bytes bytes;
      std::string tier;
      ls >> app >> bytes >> tier;
      const std::vector<ChunkId> got = mem_.allocate(static_cast<AppId>(app), bytes, parse_tier(tier));
      std::vector<ChunkId> want;
      for (unsigned c; ls >> c;) want.push_back(static_cast<ChunkId>(c));
      if (got != want) throw std::runtime_error("alloc: reference chunk ids differ from the daemon's");
    } else if (op == "free") {
      unsigned app, chunk;
      ls >> app >> chunk;
      mem_.free_chunk(static_cast<AppId>(app), static_cast<ChunkId>(chunk));
    } else if (op == "prefetch") {
      std::uint64_t k;
      unsigned app;
      ls >> k >> app;
      const MigrationPlan ref = plan_prefetch(static_cast<AppId>(app), mem_, pc_);
      std::istringstream dump(ref.dump());
      for (std::string l; std::getline(dump, l);) std::printf("F %" PRIu64 " %s\n", k, l.c_str());
    } else if (op == "pcommit") {
      std::uint64_t b;
      ls >> b;
      mem_.begin_move(static_cast<BlockId>(b), TierId::PinnedHost, false);
      mem_.commit_move(static_cast<BlockId>(b), TierId::PinnedHost);
    } else if (op == "plan") {
      std::string kind, tok;
      unsigned app;
      cur_ = PendingPlan{};
      cur_.open = true;
      ls >> cur_.k >> kind >> app >> tok >> cur_.in >> tok >> cur_.out >> tok;
      cur_.app = static_cast<AppId>(app);
      for (unsigned v; ls >> v;) cur_.victims.push_back(static_cast<AppId>(v));
    } else {
      throw std::runtime_error("unknown trace line: " + raw);
    }
  }

  // The reference's plan on the pre-switch state, then the daemon's plan
  // executed by the reference.
  void flush() {
    if (!cur_.open) return;
    cur_.open = false;
    PlannerConfig pc = pc_;
    pc.eviction_policy.victim_order = cur_.victims;
    const MigrationPlan ref = plan_switch(cur_.app, mem_, pc);
    std::printf("S %" PRIu64 " %u %" PRIu64 " %" PRIu64 "\n", cur_.k, cur_.app, ref.bytes_in, ref.bytes_out);
    std::istringstream dump(ref.dump());
    for (std::string l; std::getline(dump, l);) std::printf("P %" PRIu64 " %s\n", cur_.k, l.c_str());
    auto print_apps = [&](const char* who, const std::vector<AppId>& v) {
      std::printf("A %" PRIu64 " %s", cur_.k, who);
      for (AppId a : v) std::printf(" %u", a);
      std::printf("\n");
    };
    print_apps("ref", victim_apps(ref, mem_));
    print_apps("daemon", victim_apps(cur_.daemon, mem_));
    MigrationPlan mine = cur_.daemon;
    mine.incoming_app = cur_.app;
    mine.bytes_in = cur_.in;
    mine.bytes_out = cur_.out;
    const ExecResult r = execute(mine, mem_, hw_, pc, 0);
    std::map<int, std::vector<const TransferRecord*>> by_lane;
    for (const TransferRecord& t : r.events) by_lane[lane_of(t.src, t.dst)].push_back(&t);
    for (auto& [lane, recs] : by_lane)
      for (const TransferRecord* t : recs)
        std::printf("L %" PRIu64 " %d %" PRIu64 " %s %s\n", cur_.k, lane, t->block, tier_name(t->src), tier_name(t->dst));
    mem_.audit();
  }

  const std::string& mode() const { return mode_; }

 private:
  MemState mem_;
  HardwareConfig hw_;
  PlannerConfig pc_;
  std::string mode_ = "reference";
  PendingPlan cur_;
};

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_replay <trace-file>\n");
    return 2;
  }
  try {
    std::ifstream f(argv[1]);
    if (!f) throw std::runtime_error(std::string("cannot open ") + argv[1]);
    Replay r;
    for (std::string l; std::getline(f, l);) r.line(l);
    r.flush();
    std::printf("M %s\n", r.mode().c_str());
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_replay: %s\n", e.what());
    return 1;
  }
}
