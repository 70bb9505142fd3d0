"""BASELINE config 4: pinned budget vs switch latency for a 16 GiB <-> 16 GiB
round robin at a 16 GiB GPU cap (two-hop through pageable memory when the
budget is small). Prints one JSON line per budget; model predictions from the
reference's link model are printed beside the measurement."""
import json, sys, time
sys.path.insert(0, '.')
from paper_2601_11743_b200 import GIB, MIB, PlannerConfig, SwapEngine, run_scenario_model
from paper_2601_11743_b200._lib import TIER_PAGED
threads = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for p in (2, 4, 8, 16, 32):
    e = SwapEngine(gpu_capacity=16 * GIB, pinned_capacity=p * GIB, paged_capacity=64 * GIB, host_threads=threads,
                   host_legs_in_flight=4 * threads)
    e.allocate(0, 16 * GIB, TIER_PAGED); e.allocate(1, 16 * GIB, TIER_PAGED)
    e.fill_pattern(0, 9); e.fill_pattern(1, 9)
    pc = PlannerConfig(pinned_budget=p * GIB); nxt = 0; lat = []
    for i in range(5):
        pc.victim_order = [1 - nxt]
        st = e.switch_to(nxt, pc); nxt = 1 - nxt
        lat.append(round(st["wall_s"] + st["plan_s"], 4))
    peak = e.pinned_physical()[1]
    bad = e.verify_pattern(0, 9) + e.verify_pattern(1, 9)
    e.close()
    spec = open('paper_2601_11743_b200/scenarios/c4_budget_%dg.scn' % p).read() if p in (2, 4, 8, 16) else None
    model = None
    if spec:
        t = run_scenario_model(spec)
        ts = [ln.split() for ln in t.splitlines() if ln.startswith('T ')]
        model = [round(float(x[3]) - float(x[2]), 4) for x in ts]
    print(json.dumps({"pinned_budget_gib": p, "host_threads": threads, "switch_latency_s": lat,
                      "steady_latency_s": round(sum(lat[2:]) / len(lat[2:]), 4), "pinned_peak_gib": round(peak / GIB, 3),
                      "byte_exact": bad == 0, "reference_model_latency_s": model}), flush=True)
