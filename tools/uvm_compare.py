"""UVM vs the swap engine on one B200 (PAPER.md:313 claims
Nixie switches ~2x faster than UVM). Same exchange both ways: two 16 GiB
working sets on 17 GiB of usable device memory (UVM: a cudaMalloc balloon
caps it; engine: 16 GiB budget). UVM: tests/apps/uvm_rr.cu, fault-driven and
with cudaMemPrefetchAsync. Engine: 16 GiB <-> 16 GiB switches through the C
ABI (both directions at once, verified restores). Prints JSON lines."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
UVM = os.path.join(ROOT, "paper_2601_11743_b200", "lib", "nx_uvm_rr")
ws, cap = 16, 17
for pf in (0, 1):
    p = subprocess.run([UVM, "--cap-gib", str(cap), "--ws-gib", str(ws), "--rounds", "3", "--prefetch", str(pf)],
                       capture_output=True, text=True, timeout=900)
    print(p.stdout.strip() or json.dumps({"mode": "uvm", "error": p.stderr[-300:]}), flush=True)

from paper_2601_11743_b200 import GIB, PlannerConfig, SwapEngine  # noqa: E402
from paper_2601_11743_b200._lib import TIER_GPU, TIER_PINNED  # noqa: E402

e = SwapEngine(gpu_capacity=ws * GIB, pinned_capacity=2 * ws * GIB + 2 * GIB, paged_capacity=2 * GIB)
e.allocate(0, ws * GIB, TIER_GPU)
e.allocate(1, ws * GIB, TIER_PINNED)
e.fill_pattern(0, 1)
e.fill_pattern(1, 1)
lat = []
nxt = 1
for _ in range(6):
    st = e.switch_to(nxt, PlannerConfig(victim_order=[1 - nxt]))
    assert st["mismatches"] == 0
    lat.append(round((st["wall_s"] + st["plan_s"]) * 1e3, 2))
    nxt = 1 - nxt
ok = e.verify_pattern(0, 1) == 0 and e.verify_pattern(1, 1) == 0
e.close()
lat_s = sorted(lat)
print(json.dumps({"mode": "nixie-b200 swap engine", "ws_gib": ws, "switch_cost_ms": lat, "median_ms": lat_s[len(lat_s) // 2],
                  "bidir_equiv_gbps": round(2 * ws * GIB / (lat_s[len(lat_s) // 2] * 1e-3) / 1e9, 2), "byte_exact": ok}))
