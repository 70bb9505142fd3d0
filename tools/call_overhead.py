import sys, time, statistics
sys.path.insert(0, '.')
from paper_2601_11743_b200 import GIB, MIB, PlannerConfig, SwapEngine
from paper_2601_11743_b200._lib import TIER_GPU, TIER_PINNED
e = SwapEngine(gpu_capacity=32 * GIB, pinned_capacity=16 * GIB, paged_capacity=2 * GIB)
e.allocate(0, 16 * GIB, TIER_GPU); e.allocate(1, 16 * GIB, TIER_GPU); e.allocate(1, 8 * GIB, TIER_PINNED)
e.fill_pattern(0, 7); e.fill_pattern(1, 7)
pc = PlannerConfig(streaming_window=512 * MIB, pinned_budget=16 * GIB)
nxt = 0
rows = []
for i in range(14):
    pc.victim_order = [1 - nxt]
    t0 = time.perf_counter()
    st = e.switch_to(nxt, pc)
    t1 = time.perf_counter()
    nxt = 1 - nxt
    if i >= 4:
        rows.append(((t1 - t0) * 1e3, (st["wall_s"] + st["plan_s"]) * 1e3, st["device_span_s"] * 1e3, st["plan_s"] * 1e3))
for r in rows: print([round(x, 3) for x in r], round(r[0] - r[1], 3))
print("median call-internal", statistics.median(r[0] - r[1] for r in rows), "internal-device", statistics.median(r[1] - r[2] for r in rows))
e.close()
