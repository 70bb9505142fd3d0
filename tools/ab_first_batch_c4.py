"""Config 4 steady switch latency, batch ramp start 8 vs 2 legs, interleaved."""
import json, sys
sys.path.insert(0, '.')
from paper_2601_11743_b200 import GIB, PlannerConfig, SwapEngine
from paper_2601_11743_b200._lib import TIER_PAGED
for p in (8, 16, 32):
    for fb in (8, 2, 8, 2):
        e = SwapEngine(gpu_capacity=16 * GIB, pinned_capacity=p * GIB, paged_capacity=64 * GIB, host_threads=16,
                       host_legs_in_flight=64, first_batch_legs=fb)
        e.allocate(0, 16 * GIB, TIER_PAGED); e.allocate(1, 16 * GIB, TIER_PAGED)
        e.fill_pattern(0, 9); e.fill_pattern(1, 9)
        pc = PlannerConfig(pinned_budget=p * GIB); nxt = 0; lat = []
        for i in range(5):
            pc.victim_order = [1 - nxt]
            st = e.switch_to(nxt, pc); nxt = 1 - nxt
            lat.append(round(st["wall_s"] + st["plan_s"], 4))
        e.close()
        print(json.dumps({"pinned": p, "first_batch_legs": fb, "steady": round(sum(lat[2:]) / 3, 4), "lat": lat}), flush=True)
