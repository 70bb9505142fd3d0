import json, sys, statistics
sys.path.insert(0, ".")
from paper_2601_11743_b200 import GIB, PlannerConfig, SwapEngine
from paper_2601_11743_b200._lib import TIER_GPU, TIER_PINNED
one = (sys.argv[1] != "0") if len(sys.argv) > 1 else True
grp = (sys.argv[2] != "0") if len(sys.argv) > 2 else True
print("k3_one_stream", one, "k3_grouped", grp)
e = SwapEngine(gpu_capacity=32 * GIB, pinned_capacity=16 * GIB, paged_capacity=2 * GIB, k3_one_stream=one, k3_grouped=grp)
e.allocate(0, 16 * GIB, TIER_GPU); e.allocate(1, 16 * GIB, TIER_GPU); e.allocate(1, 8 * GIB, TIER_PINNED)
e.fill_pattern(0, 5); e.fill_pattern(1, 5)
pc = PlannerConfig(pinned_budget=16 * GIB); nxt = 0
for i in range(5):
    pc.victim_order = [1 - nxt]; st = e.switch_to(nxt, pc); nxt = 1 - nxt
t = e.k3_trace()
by = {}
for a, z, legs, lane in t:
    by.setdefault((legs, lane), []).append((z - a) * 1e6)
for k, v in sorted(by.items()):
    print(k, len(v), "min", round(min(v), 1), "med", round(statistics.median(v), 1), "max", round(max(v), 1), "us")
# overlap with the other lane: fraction of time both lanes' K3 run
print("span ms", round((max(z for _, z, _, _ in t) - min(a for a, _, _, _ in t)) * 1e3, 2), "sum ms", round(sum(z - a for a, z, _, _ in t) * 1e3, 2),
      "GBps", round((st['bytes_in'] + st['bytes_out']) / st['device_span_s'] / 1e9, 1))
print([(round(a * 1e3, 3), round((z - a) * 1e6, 1), legs, lane) for a, z, legs, lane in t[:30]])
print("k3 events busy ms", round(st["k3_busy_s"] * 1e3, 3), "k3 kernel-clock ms", round(st["k3_kernel_s"] * 1e3, 3), "bytes GB", st["pcie_h2d_bytes"] * 2 / 1e9)
print("TB/s events", round(2 * st["pcie_h2d_bytes"] / st["k3_busy_s"] / 1e12, 2), "TB/s kernel", round(2 * st["pcie_h2d_bytes"] / st["k3_kernel_s"] / 1e12, 2))
print("ce_calls", st["ce_calls"], "ce_batches", st["ce_batches_h2d"] + st["ce_batches_d2h"], "legs", st["pcie_h2d_bytes"] * 2 // (2 << 20))
