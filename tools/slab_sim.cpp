// Host-only replay of the interposer's slab placement over modeled switches
// (no GPU): two PyTorch-like apps (the config-2 LLM pair's allocation sizes)
// alternate; each switch is plan_switch + the reference lane model
// (execute), and its transfer log is replayed onto SlabPlacer in time order
// (acquire when a leg toward the GPU starts, release when a leg away from it
// ends). Prints, per switch, the slabs the incoming app must remap, the
// partly resident slabs and growth. Used to study victim/affinity policies
// (DESIGN.md §10). `slab_sim ref` uses the planner's own victims; SIM_DESC=1
// evicts each run in descending virtual-slab order. The model ignores the victims'
// post-switch unmaps (every returning vslab then needs a map on hardware).
//   g++ -std=c++20 -O2 -Iinclude -Ipaper_2601_11743_b200/csrc/daemon -Ipaper_2601_11743_b200/csrc/ipc
//       tools/slab_sim.cpp paper_2601_11743_b200/lib/libnixie_host.a -o /tmp/slab_sim
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <vector>

#include "nixie/planner.hpp"
#include "nixie/transfer.hpp"
#include "slab_placer.hpp"

using namespace nixie;
using namespace nixie::b200;

int main(int argc, char** argv) {
  const bool ref = argc > 1 && std::strcmp(argv[1], "ref") == 0;
  const std::uint32_t slack = argc > 2 ? std::atoi(argv[2]) : 4;
  const std::uint32_t sb = 256;
  MemState mem;
  HardwareConfig hw;
  hw.tier_capacity[0] = 32 * kGiB;
  hw.tier_capacity[1] = 16 * kGiB;
  hw.tier_capacity[2] = 96 * kGiB;
  hw.apply_to(mem);
  SlabPlacer p(64 + slack, sb);
  std::uint32_t next = 64 + slack;
  p.set_grow([&] { return next++; });
  PlannerConfig cfg;
  if (!ref) cfg.gpu_victims = [&](const MemState& s, const std::vector<AppId>& o, Bytes w) { return p.slab_victims(s, o, w); };

  // allocation sizes in 2 MiB blocks, bump placement (range_alloc.hpp)
  std::map<AppId, std::uint64_t> va;
  std::map<BlockId, std::uint32_t> frame;
  auto alloc = [&](AppId app, std::uint64_t n, TierId tier) {
    std::uint64_t& cur = va[app];
    if (n >= sb / 2) cur = (cur + sb - 1) / sb * sb;
    const auto chunks = mem.allocate(app, n * kBlockBytes, tier);
    const BlockId first = mem.chunk(chunks.front()).blocks.front();
    p.expect(first, n, app, cur);
    if (tier == TierId::Gpu)
      for (std::uint64_t k = 0; k < n; ++k) frame[first + k] = p.acquire(first + k);
    cur += n;
  };
  auto model = [&](AppId app, int layers, std::uint64_t qo, std::uint64_t kv, std::uint64_t mlp, std::uint64_t emb,
                   TierId tier) {
    alloc(app, emb, tier);
    for (int l = 0; l < layers; ++l) {
      alloc(app, qo, tier); alloc(app, kv, tier); alloc(app, kv, tier); alloc(app, qo, tier);
      alloc(app, mlp, tier); alloc(app, mlp, tier); alloc(app, mlp, tier); alloc(app, 1, tier);
    }
    alloc(app, emb, tier);
  };
  model(0, 36, 16, 4, 48, 594, TierId::Gpu);        // ~15.3 GiB
  model(1, 53, 18, 18, 54, 300, TierId::PagedHost);  // ~23 GiB
  p.take_assigned();
  std::map<SlabPlacer::Key, std::uint32_t> mapped;
  for (auto& k : p.backed(0)) mapped[{0, k.vslab}] = k.phys;

  AppId cur = 0;
  for (int sw = 0; sw < 12; ++sw) {
    const AppId to = 1 - cur;
    cfg.eviction_policy.victim_order = {cur};
    MigrationPlan plan = plan_switch(to, mem, cfg);
    if (std::getenv("SIM_DESC")) {
      auto& mv = plan.moves;
      for (std::size_t i = 0; i < mv.size();) {
        std::size_t j = i + 1;
        if (mv[i].kind == MoveKind::EvictFromGpu)
          while (j < mv.size() && mv[j].kind == MoveKind::EvictFromGpu && mv[j].dst == mv[i].dst) ++j;
        std::stable_sort(mv.begin() + i, mv.begin() + j,
                         [&](const Move& a, const Move& b) { return p.vslab_of(a.block) > p.vslab_of(b.block); });
        i = j;
      }
    }
    const ExecResult r = execute(plan, mem, hw, cfg);
    // replay onto the placer: (time, release-before-acquire, block)
    std::vector<std::tuple<double, int, BlockId, bool>> ev;
    for (const auto& t : r.events) {
      if (t.dst == TierId::Gpu) ev.emplace_back(t.start, 1, t.block, true);
      if (t.src == TierId::Gpu) ev.emplace_back(t.end, 0, t.block, false);
    }
    std::sort(ev.begin(), ev.end());
    for (auto& [t, kind, b, acq] : ev) {
      if (acq) frame[b] = p.acquire(b);
      else p.release(b, frame[b]);
    }
    int remaps = 0;
    for (auto& k : p.backed(to)) {
      auto it = mapped.find({to, k.vslab});
      if (it == mapped.end() || it->second != k.phys) ++remaps;
      mapped[{to, k.vslab}] = k.phys;
    }
    p.take_assigned();
    p.take_released();
    std::printf("switch %d -> app %u: in %llu out %llu blocks, remaps %d, partial %llu, free %zu, grown %u\n", sw, to,
                (unsigned long long)(plan.bytes_in / kBlockBytes), (unsigned long long)(plan.bytes_out / kBlockBytes), remaps,
                (unsigned long long)p.partial(), p.free_slabs(), p.grown());
    cur = to;
  }
}
