"""Config 4 (2 x 16 GiB round robin on a 16 GiB cap): steady switch latency
per pinned budget under different lane concurrency limits (host legs in
flight per host lane, PCIe legs in flight per direction). Explains and tunes
the budget curve of tools/budget_sweep.py. One JSON line per point."""
import itertools
import json
import statistics
import sys
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_11743_b200 import GIB, PlannerConfig, SwapEngine  # noqa: E402
from paper_2601_11743_b200._lib import TIER_PAGED  # noqa: E402

budgets = [float(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,4,8").split(",")]
hosts = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "16,64").split(",")]
pcies = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "256,1024").split(",")]
for b, h, p in itertools.product(budgets, hosts, pcies):
    e = SwapEngine(gpu_capacity=16 * GIB, pinned_capacity=int(b * GIB), paged_capacity=64 * GIB, host_legs_in_flight=h,
                   pcie_legs_in_flight=p)
    e.allocate(0, 16 * GIB, TIER_PAGED)
    e.allocate(1, 16 * GIB, TIER_PAGED)
    e.fill_pattern(0, 9)
    e.fill_pattern(1, 9)
    pc = PlannerConfig(pinned_budget=int(b * GIB))
    nxt, lat = 0, []
    for _ in range(5):
        pc.victim_order = [1 - nxt]
        st = e.switch_to(nxt, pc)
        assert st["mismatches"] == 0
        nxt = 1 - nxt
        lat.append(round(st["wall_s"] + st["plan_s"], 4))
    ok = e.verify_pattern(0, 9) + e.verify_pattern(1, 9) == 0
    th = e.host_threads()
    e.close()
    print(json.dumps({"budget_gib": b, "host_legs_in_flight": h, "pcie_legs_in_flight": p, "host_threads": th,
                      "latency_s": lat, "steady_s": statistics.median(lat[2:]), "byte_exact": ok}), flush=True)
