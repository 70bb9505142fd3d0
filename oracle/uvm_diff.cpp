// TEST INFRASTRUCTURE ONLY (oracle/). Seeded random UvmSim workloads printed
// as a decision trace; built twice by oracle/Makefile: against the unmodified
// reference (proj/src/uvm.cpp) and against this repo's include/nixie/uvm.hpp
// + libnixie_host.a. tests/test_dropin.py diffs the two outputs.
// Usage: uvm_diff <seed> <ops>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "nixie/uvm.hpp"

using namespace nixie;

static std::uint64_t rng_state;
static std::uint64_t rnd() {
  std::uint64_t z = (rng_state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int main(int argc, char** argv) {
  rng_state = argc > 1 ? std::strtoull(argv[1], nullptr, 0) : 1;
  const int ops = argc > 2 ? std::atoi(argv[2]) : 200;
  const Bytes cap = (8 + rnd() % 40) * kBlockBytes;
  UvmConfig cfg;
  cfg.prefetch_pages = static_cast<int>(rnd() % 20);
  std::vector<TransferRecord> tlog;
  std::vector<FaultLogRow> flog;
  UvmSim u(cap, LinkConfig{64.0 * kGiB, 32.0 * kGiB, Duplex::HalfDuplex}, cfg, &tlog, &flog);
  std::vector<std::pair<AppId, ChunkId>> live;
  std::uint64_t npages = 0;
  double now = 0;
  for (int i = 0; i < ops; ++i) {
    const int op = static_cast<int>(rnd() % 10);
    const AppId app = static_cast<AppId>(rnd() % 3);
    try {
      if (op < 3 || live.empty()) {
        const Bytes sz = (1 + rnd() % 70) * kMiB;
        for (ChunkId c : u.register_alloc(app, sz)) live.push_back({app, c});
        npages += block_count_for(sz);
        std::printf("A %u %" PRIu64 "\n", app, sz);
      } else if (op < 7) {
        std::vector<ChunkId> mine;
        for (auto& [a, c] : live)
          if (a == app && rnd() % 2) mine.push_back(c);
        const double d = u.touch_kernel(app, mine, 0.001, now);
        now += d;
        std::printf("K %u %zu %.17g\n", app, mine.size(), d);
      } else if (op < 9) {
        const AppId a = live[rnd() % live.size()].first;
        const PageId p = rnd() % npages;  // may belong to another app or a freed chunk
        if (!u.page_resident(p)) {
          FaultResolution r = u.on_fault(a, p, now, {});
          std::printf("F %" PRIu64 " e%zu f%zu %.17g\n", p, r.evicted.size(), r.fetched.size(), r.service_time);
          for (PageId e : r.evicted) std::printf(" %" PRIu64, e);
          std::printf("\n");
        }
      } else {
        const std::size_t k = rnd() % live.size();
        std::printf("D %u %" PRIu64 " %" PRIu64 "\n", live[k].first, live[k].second, u.free_chunk(live[k].first, live[k].second));
        live.erase(live.begin() + static_cast<long>(k));
      }
    } catch (const SimError& e) {
      std::printf("X %s\n", e.what());
    }
    std::printf("S %" PRIu64 " %" PRIu64 " %" PRIu64 " %" PRIu64 " %" PRIu64 "\n", u.gpu_used(), u.pinned_mirror_usage(),
                u.pinned_mirror_peak(), u.faulted_bytes_total(), u.fault_count());
  }
  std::printf("T %zu %zu\n", tlog.size(), flog.size());
  for (const auto& t : tlog) std::printf("t %.17g %.17g %" PRIu64 " %" PRIu64 "\n", t.start, t.end, t.block, t.bytes);
  return 0;
}
