"""Design-space sweep of the swap engine on one GPU (development tool).

Runs the 16 GiB <-> 16 GiB exchange (GPU capped at 16 GiB, incoming app in
the pinned ring) under several engine settings and prints device-timed and
wall-clock bidirectional GB/s per switch.
"""
import itertools
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2601_11743_b200 import GIB, MIB, EngineConfig, PlannerConfig, SwapEngine  # noqa: E402

SIZE = int(sys.argv[1]) if len(sys.argv) > 1 else 16
variants = [
    dict(path=1, fused_launch=False, legs_per_launch=64, pcie_legs_in_flight=256),
    dict(path=1, fused_launch=True, legs_per_launch=128, pcie_legs_in_flight=256),
    dict(path=2, fused_launch=False, legs_per_launch=64, pcie_legs_in_flight=256),
    dict(path=2, fused_launch=False, legs_per_launch=16, pcie_legs_in_flight=128),
    dict(path=1, fused_launch=False, legs_per_launch=128, pcie_legs_in_flight=512),
    dict(path=1, fused_launch=False, legs_per_launch=32, pcie_legs_in_flight=256),
]
eng = SwapEngine(gpu_capacity=SIZE * GIB, pinned_capacity=(2 * SIZE + 2) * GIB, paged_capacity=4 * GIB)
eng.allocate(0, SIZE * GIB, 0)
eng.allocate(1, SIZE * GIB, 1)
seed = 7
eng.fill_pattern(0, seed)
eng.fill_pattern(1, seed)
pc = PlannerConfig()
print(json.dumps(eng.probe_pcie(1 * GIB, 64 * MIB)))
cur = 0
for v in variants:
    # engine options are fixed at creation; emulate by a fresh engine per variant would re-pin memory,
    # so only the first variant uses `eng`; the rest create their own engines.
    pass
eng.close()

for v in variants:
    e = SwapEngine(gpu_capacity=SIZE * GIB, pinned_capacity=(2 * SIZE + 2) * GIB, paged_capacity=4 * GIB, **v)
    e.allocate(0, SIZE * GIB, 0)
    e.allocate(1, SIZE * GIB, 1)
    e.fill_pattern(0, seed)
    e.fill_pattern(1, seed)
    res = []
    nxt = 1
    for i in range(5):
        pc.victim_order = [1 - nxt]
        st = e.switch_to(nxt, pc)
        nxt = 1 - nxt
        b = st["bytes_in"] + st["bytes_out"]
        res.append((b / st["device_span_s"] / 1e9, b / st["wall_s"] / 1e9, st["wall_s"], st["launches_h2d"] + st["launches_d2h"],
                    st["ce_batches_h2d"] + st["ce_batches_d2h"], st["mismatches"], st["tp_bidir"] / 1e9))
    bad = e.verify_pattern(0, seed) + e.verify_pattern(1, seed)
    print(json.dumps({"variant": v, "dev_GBps": [round(r[0], 1) for r in res], "wall_GBps": [round(r[1], 1) for r in res],
                      "wall_s": [round(r[2], 4) for r in res], "launches": res[-1][3], "ce": res[-1][4],
                      "tp_bidir": [round(r[6], 1) for r in res], "bad": bad}), flush=True)
    e.close()
