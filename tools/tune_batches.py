"""Config-2 steady switch device span vs batching knobs (first_batch_legs,
legs_per_launch, pcie_legs_in_flight), alternating configs to average out
host noise. Prints one line per config."""
import itertools, json, statistics, sys
sys.path.insert(0, ".")
from paper_2601_11743_b200 import GIB, MIB, PlannerConfig, SwapEngine
from paper_2601_11743_b200._lib import TIER_GPU, TIER_PINNED

configs = [dict(first_batch_legs=8, legs_per_launch=128, pcie_legs_in_flight=512),
           dict(first_batch_legs=16, legs_per_launch=128, pcie_legs_in_flight=1024),
           dict(first_batch_legs=8, legs_per_launch=128, pcie_legs_in_flight=1024),
           dict(first_batch_legs=16, legs_per_launch=64, pcie_legs_in_flight=1024),
           dict(first_batch_legs=32, legs_per_launch=128, pcie_legs_in_flight=1024),
           dict(first_batch_legs=16, legs_per_launch=128, pcie_legs_in_flight=2048)]
if len(sys.argv) > 1:  # a JSON list of configs replaces the default set
    configs = json.loads(sys.argv[1])
res = {i: [] for i in range(len(configs))}
engines = []
for rnd in range(4):
    for i, c in enumerate(configs):
        e = SwapEngine(gpu_capacity=32 * GIB, pinned_capacity=16 * GIB, paged_capacity=2 * GIB, **c)
        e.allocate(0, 16 * GIB, TIER_GPU); e.allocate(1, 16 * GIB, TIER_GPU); e.allocate(1, 8 * GIB, TIER_PINNED)
        e.fill_pattern(0, 1); e.fill_pattern(1, 1)
        pc = PlannerConfig(streaming_window=512 * MIB, pinned_budget=16 * GIB)
        nxt = 0
        for k in range(6):
            pc.victim_order = [1 - nxt]
            st = e.switch_to(nxt, pc)
            nxt = 1 - nxt
            if k >= 2:
                res[i].append((st["device_span_s"] * 1e3, (st["wall_s"] + st["plan_s"]) * 1e3))
        e.close()
for i, c in enumerate(configs):
    spans = [x[0] for x in res[i]]; walls = [x[1] for x in res[i]]
    print(json.dumps({**c, "span_ms_median": round(statistics.median(spans), 2), "wall_ms_median": round(statistics.median(walls), 2),
                      "n": len(spans)}), flush=True)
