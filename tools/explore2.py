"""Batch-size sweep on the bench workload (config 2 steady state)."""
import json, sys
sys.path.insert(0, ".")
from paper_2601_11743_b200 import GIB, MIB, PlannerConfig, SwapEngine
from paper_2601_11743_b200._lib import TIER_PAGED
for legs, first in ((64, 8), (32, 8), (16, 4), (128, 8)):
    e = SwapEngine(gpu_capacity=32 * GIB, pinned_capacity=16 * GIB, paged_capacity=96 * GIB, legs_per_launch=legs, first_batch_legs=first)
    e.allocate(0, 16 * GIB, TIER_PAGED); e.allocate(1, 24 * GIB, TIER_PAGED)
    e.fill_pattern(0, 5); e.fill_pattern(1, 5)
    pc = PlannerConfig(pinned_budget=16 * GIB); nxt = 0; res = []
    for i in range(8):
        pc.victim_order = [1 - nxt]
        st = e.switch_to(nxt, pc); nxt = 1 - nxt
        if i >= 3:
            b = st["bytes_in"] + st["bytes_out"]
            res.append((round(b / st["device_span_s"] / 1e9, 2), round(st["wall_s"] * 1e3, 1), round(st["k3_bytes"] / st["k3_busy_s"] / 1e9)))
    print(json.dumps({"legs": legs, "first": first, "res": res, "bad": e.verify_pattern(0, 5) + e.verify_pattern(1, 5)}), flush=True)
    e.close()
