"""Short swap workload for ncu captures (one GPU): a few steady switches of a
scaled-down config-2 shape (8 GiB cap, 4+6 GiB apps, 4 GiB pinned budget), or
of bench.py's full config 2 (32 GiB cap, 16+24 GiB apps, 16 GiB pinned) with
a third argument "c2"."""
import sys
sys.path.insert(0, '.')
from paper_2601_11743_b200 import GIB, MIB, PlannerConfig, SwapEngine, parse_path
from paper_2601_11743_b200._lib import TIER_PAGED
path = parse_path(sys.argv[1] if len(sys.argv) > 1 else 'ce')
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
full = len(sys.argv) > 3 and sys.argv[3] == 'c2'
cap, pin, a0, a1 = (32, 16, 16, 24) if full else (8, 4, 4, 6)
e = SwapEngine(gpu_capacity=cap * GIB, pinned_capacity=pin * GIB, paged_capacity=(48 if full else 16) * GIB, path=path)
e.allocate(0, a0 * GIB, TIER_PAGED)
e.allocate(1, a1 * GIB, TIER_PAGED)
e.fill_pattern(0, 3)
e.fill_pattern(1, 3)
pc = PlannerConfig(streaming_window=512 * MIB, pinned_budget=pin * GIB)
nxt = 0
for i in range(n):
    pc.victim_order = [1 - nxt]
    st = e.switch_to(nxt, pc)
    print(i, round((st['bytes_in'] + st['bytes_out']) / st['device_span_s'] / 1e9, 1), 'GB/s', st['k1_launches'], st['k3_launches'], flush=True)
    nxt = 1 - nxt
assert e.verify_pattern(0, 3) == 0 and e.verify_pattern(1, 3) == 0
e.close()
