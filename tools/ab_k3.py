import json, sys, time
sys.path.insert(0, ".")
from paper_2601_11743_b200 import GIB, MIB, PlannerConfig, SwapEngine
from paper_2601_11743_b200._lib import TIER_GPU, TIER_PINNED
for opts in (dict(k3_tma=False), dict(k3_tma=True), dict(k3_tma=False, legs_per_launch=64, pcie_legs_in_flight=256), dict(k3_tma=True, verify=False)):
    e = SwapEngine(gpu_capacity=32 * GIB, pinned_capacity=16 * GIB, paged_capacity=2 * GIB, **opts)
    e.allocate(0, 16 * GIB, TIER_GPU); e.allocate(1, 16 * GIB, TIER_GPU); e.allocate(1, 8 * GIB, TIER_PINNED)
    e.fill_pattern(0, 5); e.fill_pattern(1, 5)
    pc = PlannerConfig(pinned_budget=16 * GIB); nxt = 0; res = []
    for i in range(7):
        pc.victim_order = [1 - nxt]
        st = e.switch_to(nxt, pc); nxt = 1 - nxt
        if i >= 2:
            b = st["bytes_in"] + st["bytes_out"]
            res.append((round(b / st["device_span_s"] / 1e9, 1), round(st["wall_s"] * 1e3, 1), st["k3_launches"], round(st["k3_busy_s"] * 1e3, 2)))
    print(json.dumps({"opts": opts, "res": res}), flush=True)
    e.close()
