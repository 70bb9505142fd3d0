"""The UVM comparator as a gated result.

The reference models UVM as fault-driven, half-duplex evict-then-fetch
migration (proj/src/uvm.cpp:114-193) and claims Nixie switches about 2x
faster (the paper's hardware claim). Here both
sides run on the B200: tests/apps/uvm_rr.cu (cudaMallocManaged round-robin,
a device balloon caps the usable memory, every switch evicts the other app
and faults this one in) and the swap engine moving the same exchange
(2 GiB <-> 2 GiB, both PCIe directions at once, every restore verified)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
UVM = os.path.join(ROOT, "paper_2601_11743_b200", "lib", "nx_uvm_rr")

pytestmark = pytest.mark.gpu
WS_GIB = 2


def _uvm(prefetch, ws=WS_GIB):
    p = subprocess.run([UVM, "--cap-gib", str(ws + 1), "--ws-gib", str(ws), "--rounds", "3",
                        "--prefetch", str(prefetch)], capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-500:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def _engine(ws=WS_GIB):
    from paper_2601_11743_b200 import GIB, PlannerConfig, SwapEngine
    from paper_2601_11743_b200._lib import TIER_GPU, TIER_PINNED
    lat = []
    with SwapEngine(gpu_capacity=ws * GIB, pinned_capacity=2 * ws * GIB + 2 * GIB, paged_capacity=2 * GIB) as e:
        e.allocate(0, ws * GIB, TIER_GPU)
        e.allocate(1, ws * GIB, TIER_PINNED)
        e.fill_pattern(0, 5)
        e.fill_pattern(1, 5)
        nxt = 1
        for _ in range(6):
            st = e.switch_to(nxt, PlannerConfig(victim_order=[1 - nxt]))
            assert st["mismatches"] == 0 and st["bytes_in"] == ws * GIB and st["bytes_out"] == ws * GIB, st
            lat.append((st["wall_s"] + st["plan_s"]) * 1e3)
            nxt = 1 - nxt
        exact = e.verify_pattern(0, 5) == 0 and e.verify_pattern(1, 5) == 0
    return sorted(lat[2:])[len(lat[2:]) // 2], exact


def test_engine_beats_uvm_on_the_same_exchange():
    uvm = _uvm(0)
    assert uvm["mismatches"] == 0, uvm  # UVM's data survived its migrations
    eng_ms, exact = _engine()
    assert exact
    speedup = uvm["median_ms"] / eng_ms
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "uvm_gate.json"), "w") as f:
            json.dump({"ws_gib": WS_GIB, "uvm": uvm, "engine_switch_ms_p50": eng_ms, "speedup": speedup}, f)
    # The reference claims ~2x; the gate is 1.5x.
    assert speedup >= 1.5, (uvm["median_ms"], eng_ms)


def test_engine_not_slower_than_uvm_with_prefetch_hints():
    """UVM's best case: cudaMemPrefetchAsync bulk migration instead of demand
    faults. It narrows with size: measured 1.06x at 2 GiB, 1.07x at 4 GiB,
    1.44x at 16 GiB (profiles/r02_budget_sweep.jsonl). Gate: on an 8 GiB
    exchange the engine is not slower."""
    uvm = _uvm(1, ws=8)
    assert uvm["mismatches"] == 0, uvm
    eng_ms, exact = _engine(ws=8)
    assert exact
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "uvm_gate_prefetch.json"), "w") as f:
            json.dump({"ws_gib": 8, "uvm": uvm, "engine_switch_ms_p50": eng_ms, "speedup": uvm["median_ms"] / eng_ms}, f)
    assert uvm["median_ms"] / eng_ms >= 1.0, (uvm["median_ms"], eng_ms)
