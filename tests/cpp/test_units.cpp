// Host-only unit tests of the interposer's placement logic (no GPU):
//   SlabPlacer (csrc/daemon/slab_placer.hpp): slot arithmetic, sharing of a
//     slab by the blocks of one vslab, release, affinity, exhaustion,
//     mapping bookkeeping;
//   RangeAlloc (csrc/shim/range_alloc.hpp): first fit, slab alignment,
//     coalescing on free;
//   UnitRing (csrc/engine/phys.hpp): FIFO order, contiguity-preferring
//     acquire_after, stale entries, never handing out a unit twice.
// Built by paper_2601_11743_b200/Makefile (lib/nx_unit_tests); run by
// tests/test_interposer_host.py.
#include <cstdio>
#include <cstdlib>
#include <set>
#include <string>
#include <algorithm>

#include "nixie/planner.hpp"
#include "phys.hpp"
#include "range_alloc.hpp"
#include "slab_placer.hpp"

using namespace nixie;
using namespace nixie::b200;

static int failures = 0, checks = 0;
#define CHECK(c)                                                       \
  do {                                                                 \
    ++checks;                                                          \
    if (!(c)) {                                                        \
      ++failures;                                                      \
      std::fprintf(stderr, "%s:%d CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
    }                                                                  \
  } while (0)

static void slab_placer() {
  const std::uint32_t sb = 4;      // blocks per slab
  SlabPlacer p(3, sb);             // 3 physical slabs
  // app 7: blocks 0..5 at range blocks 2..7 (vslab 0: slots 2,3; vslab 1: slots 0..3)
  p.expect(0, 6, 7, 2);
  const std::uint32_t f0 = p.acquire(0), f1 = p.acquire(1), f2 = p.acquire(2);
  CHECK(f0 / sb == f1 / sb);            // same vslab -> same physical slab
  CHECK(f0 % sb == 2 && f1 % sb == 3);  // at the blocks' slots
  CHECK(f2 / sb != f0 / sb && f2 % sb == 0);
  CHECK(p.free_slabs() == 1);
  auto as = p.take_assigned();
  CHECK(as.size() == 2);                // two vslabs got slabs
  CHECK(p.take_assigned().empty());
  p.release(0, f0);
  CHECK(p.take_released().empty());     // vslab 0 still holds block 1
  p.release(1, f1);
  auto rel = p.take_released();
  CHECK(rel.size() == 1 && rel[0].first == 7 && rel[0].second == 0);
  CHECK(p.free_slabs() == 2);
  // affinity: vslab 0 gets its old slab back while it is free
  const std::uint32_t g0 = p.acquire(0);
  CHECK(g0 / sb == f0 / sb);
  // ... but not once another vslab took it
  p.release(0, g0);
  p.expect(6, 4, 9, 0);                 // app 9, vslab 0
  const std::uint32_t h = p.acquire(6);
  const std::uint32_t h2 = p.acquire(7);  // app 9 takes another free slab for the same vslab? no: same vslab
  CHECK(h / sb == h2 / sb);
  const std::uint32_t again = p.acquire(0);
  CHECK(again / sb != h / sb);
  // exhaustion
  p.expect(10, 4, 11, 0);
  bool threw = false;
  try {
    p.acquire(10);
  } catch (const InvariantViolation&) {
    threw = true;
  }
  CHECK(threw);
  // mapping bookkeeping
  const SlabPlacer::Key k{7, 1};
  CHECK(p.mapped(k) == ipc::kNoFrame);
  p.set_mapped(k, 2);
  CHECK(p.mapped(k) == 2);
  p.granted(7);
  CHECK(p.mapped(k) == p.map_of(7, 1).phys);
  CHECK(p.backed(7).size() == 2);
  CHECK(p.backed(9).size() == 1);
}

static void slab_growth() {
  SlabPlacer p(1, 2);
  std::uint32_t next = 1;
  p.set_grow([&] { return next++; });
  p.expect(0, 6, 3, 0);  // 3 vslabs of 2 blocks
  const std::uint32_t a = p.acquire(0), b = p.acquire(2), c = p.acquire(4);
  CHECK(a / 2 == 0 && b / 2 == 1 && c / 2 == 2);  // slabs 1 and 2 were created on demand
  CHECK(p.grown() == 2 && p.slabs() == 3 && p.free_slabs() == 0);
  p.release(2, b);
  CHECK(p.free_slabs() == 1);
  p.release(4, c);
  // shrink: grown free slabs beyond the kept slack leave the pool
  auto drop = p.take_droppable(0);
  CHECK(drop.size() == 2 && p.free_slabs() == 0);
  CHECK(p.dropped(1) && p.dropped(2) && !p.dropped(0));
  // the next growth refills a dropped slot with a new generation
  next = 2;
  const std::uint32_t gen_before = p.gen(2);
  const std::uint32_t d = p.acquire(2);
  CHECK(d / 2 == 2 && p.gen(2) == gen_before + 1 && !p.dropped(2));
}

// Slab-aligned victims: same bytes as the reference planner, whole vslabs
// first (fewest resident blocks first), one split group at most.
static void slab_victims() {
  MemState st;
  st.set_capacity(TierId::Gpu, 16 * kBlockBytes);
  st.set_capacity(TierId::PinnedHost, 64 * kBlockBytes);
  SlabPlacer p(4, 4);
  // app 1: chunks of 3, 2, 3, 2 blocks -> blocks 0..9 at range blocks 0..9
  // (vslabs {0..3} {4..7} {8,9}); app 2: 8 blocks in pinned memory
  for (Bytes sz : {3, 2, 3, 2}) st.allocate(1, sz * kBlockBytes, TierId::Gpu);
  p.expect(0, 10, 1, 0);
  for (BlockId b = 0; b < 10; ++b) p.acquire(b);
  st.allocate(2, 8 * kBlockBytes, TierId::PinnedHost);
  PlannerConfig cfg;
  auto evicted = [](const MigrationPlan& plan) {
    std::vector<BlockId> v;
    for (const Move& m : plan.moves)
      if (m.kind == MoveKind::EvictFromGpu) v.push_back(m.block);
    std::sort(v.begin(), v.end());
    return v;
  };
  const MigrationPlan ref = plan_switch(2, st, cfg);
  CHECK(ref.bytes_out == 2 * kBlockBytes);  // 8 in, 6 free
  CHECK((evicted(ref) == std::vector<BlockId>{0, 1}));  // largest chunk first
  st.allocate(1, 2 * kBlockBytes, TierId::Gpu);  // blocks 18, 19 at range blocks 10, 11: vslab 2 full; 4 free
  p.expect(18, 2, 1, 10);
  const MigrationPlan ref2 = plan_switch(2, st, cfg);
  CHECK((evicted(ref2) == std::vector<BlockId>{0, 1, 2, 5}));  // both 3-block chunks: vslabs 0 and 1 split
  cfg.gpu_victims = [&](const MemState& s, const std::vector<AppId>& order, Bytes want) {
    return p.slab_victims(s, order, want);
  };
  const MigrationPlan ours = plan_switch(2, st, cfg);
  CHECK(ours.bytes_out == ref2.bytes_out && ours.bytes_in == ref2.bytes_in);
  CHECK(evicted(ours).size() == 4);
  std::set<std::uint32_t> touched;
  for (BlockId b : evicted(ours)) touched.insert(static_cast<std::uint32_t>((b < 10 ? b : b - 8) / 4));
  CHECK(touched.size() == 1);  // one whole vslab
}

static void range_alloc() {
  {  // bump (default): allocation order = range order, no reuse
    nixie::shim::RangeAlloc b;
    b.reset(1024);
    std::uint64_t x = 0, y = 0, z = 0;
    CHECK(b.take(3, 64, x) && x == 0);
    CHECK(b.take(10, 64, y) && y == 3);
    b.give(x, 3);
    CHECK(b.take(2, 64, z) && z == 13);  // not the freed hole
    CHECK(b.take(40, 64, z) && z == 64);  // slab aligned
  }
  nixie::shim::RangeAlloc r;
  r.reset(1024, true);
  std::uint64_t a = 0, b = 0, c = 0, d = 0;
  CHECK(r.take(3, 64, a) && a == 0);     // small: first fit
  CHECK(r.take(40, 64, b) && b == 64);   // >= half a slab: slab aligned
  CHECK(r.take(10, 64, c) && c == 3);    // fills the hole
  CHECK(!r.take(2000, 64, d));
  r.give(b, 40);
  r.give(a, 3);
  r.give(c, 10);
  CHECK(r.runs().size() == 1 && r.runs().begin()->first == 0 && r.runs().begin()->second == 1024);  // coalesced
  CHECK(r.take(1024, 64, d) && d == 0);
  CHECK(!r.take(1, 64, d));
}

static void unit_ring() {
  UnitRing r;
  r.reset(8);
  CHECK(r.acquire("t") == 0 && r.acquire("t") == 1 && r.free_units() == 6);  // FIFO
  r.release(0);                                                          // free order: 2..7, 0
  CHECK(r.acquire_after(1, "t") == 2);                                   // contiguous after 1
  CHECK(r.acquire_after(2, "t") == 3);
  r.release(1);                                                          // 4..7, 0, 1
  CHECK(r.acquire_after(7, "t") == 4);                                   // 8 is out of range: FIFO head
  CHECK(r.acquire_after(UnitRing::kNone, "t") == 5);
  CHECK(r.acquire_after(5, "t") == 6);
  CHECK(r.acquire("t") == 7);                                           // 2, 3 and 6 were stale entries
  CHECK(r.acquire("t") == 0 && r.acquire("t") == 1 && r.free_units() == 0);
  bool threw = false;
  try {
    r.acquire("t");
  } catch (const InvariantViolation&) {
    threw = true;
  }
  CHECK(threw);
  // Random churn: every acquired unit is free before and never handed out twice.
  r.reset(64);
  std::set<std::uint32_t> held;
  std::uint32_t prev = UnitRing::kNone;
  unsigned x = 12345;
  for (int i = 0; i < 20000; ++i) {
    x = x * 1103515245u + 12345u;
    if ((x >> 16) % 3 != 0 && held.size() < 64) {
      const std::uint32_t u = ((x >> 8) & 1) ? r.acquire_after(prev, "t") : r.acquire("t");
      CHECK(held.insert(u).second);
      prev = u;
    } else if (!held.empty()) {
      auto it = held.begin();
      std::advance(it, (x >> 4) % held.size());
      r.release(*it);
      held.erase(it);
    }
    CHECK(r.free_units() == 64 - held.size());
  }
}

int main() {
  unit_ring();
  slab_placer();
  slab_growth();
  range_alloc();
  slab_victims();
  std::printf("nx_unit_tests: %d checks, %d failures\n", checks, failures);
  return failures ? 1 : 0;
}
