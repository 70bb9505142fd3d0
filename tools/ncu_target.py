"""Short swap workload for ncu captures (one GPU): a few steady switches of a
scaled-down config-2 shape (8 GiB cap, 4+6 GiB apps, 4 GiB pinned budget)."""
import sys
sys.path.insert(0, '.')
from paper_2601_11743_b200 import GIB, MIB, PlannerConfig, SwapEngine, parse_path
from paper_2601_11743_b200._lib import TIER_PAGED
path = parse_path(sys.argv[1] if len(sys.argv) > 1 else 'ce')
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
e = SwapEngine(gpu_capacity=8 * GIB, pinned_capacity=4 * GIB, paged_capacity=16 * GIB, path=path)
e.allocate(0, 4 * GIB, TIER_PAGED)
e.allocate(1, 6 * GIB, TIER_PAGED)
e.fill_pattern(0, 3)
e.fill_pattern(1, 3)
pc = PlannerConfig(streaming_window=512 * MIB, pinned_budget=4 * GIB)
nxt = 0
for i in range(n):
    pc.victim_order = [1 - nxt]
    st = e.switch_to(nxt, pc)
    print(i, round((st['bytes_in'] + st['bytes_out']) / st['device_span_s'] / 1e9, 1), 'GB/s', st['k1_launches'], st['k3_launches'], flush=True)
    nxt = 1 - nxt
assert e.verify_pattern(0, 3) == 0 and e.verify_pattern(1, 3) == 0
e.close()
