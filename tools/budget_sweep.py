"""BASELINE config 4: pinned-memory budget sweep, pinned bytes vs switch
latency, against UVM's pinned mirror (Nixie matches UVM's
latency with 33.2-40.2% of UVM's pinned memory).

Workload: two 16 GiB apps round-robin on a 16 GiB GPU cap (the paper's
"each model's working set nearly fills the GPU"); every switch moves 16 GiB
out and 16 GiB in. Below a 32 GiB budget the engine's plans go two-hop through
pageable memory (pinned <-> paged on the host copy pool).

Per budget (one JSON line):
  * steady switch latency (p50 of the switches after the first two), byte-exact;
  * the budget held (pinned physical peak);
  * the two-hop path's host roofline: host-memcpy bytes per switch / latency
    against the same run's host copy peak (SwapEngine.calibrate_host, which
    also sized the pool: EngineConfig.host_threads = 0);
  * the reference's link model's latency for the same scenario (where a
    scenario file exists).
UVM side (one line each):
  * measured on the B200: tests/apps/uvm_rr.cu, 16 GiB <-> 16 GiB on a 17 GiB
    cap, fault-driven and with cudaMemPrefetchAsync, plus the host memory its
    managed backing took;
  * UVM's pinned mirror for the same round robin from the reference's UvmSim
    model (proj/include/nixie/uvm.hpp:58-63, through nx_uvm_*): every page
    ever resident on the GPU keeps a pinned host page.
Summary line: for each UVM latency, the smallest budget whose steady latency
is at most UVM's (linear interpolation between measured budgets), as bytes and
as a fraction of UVM's pinned mirror.

Usage: python tools/budget_sweep.py [--budgets 2,4,8,12,16,24,32] [--switches 6] [--no-uvm] [--ws-gib 16]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_11743_b200 import GIB, MIB, PlannerConfig, SwapEngine, run_scenario_model  # noqa: E402
from paper_2601_11743_b200._lib import TIER_PAGED, check, lib  # noqa: E402

UVM = os.path.join(ROOT, "paper_2601_11743_b200", "lib", "nx_uvm_rr")


def engine_point(budget_gib: float, ws_gib: int, switches: int) -> dict:
    e = SwapEngine(gpu_capacity=ws_gib * GIB, pinned_capacity=int(budget_gib * GIB), paged_capacity=4 * ws_gib * GIB)
    hc = e.calibrate_host(1024 * MIB)
    e.allocate(0, ws_gib * GIB, TIER_PAGED)
    e.allocate(1, ws_gib * GIB, TIER_PAGED)
    e.fill_pattern(0, 9)
    e.fill_pattern(1, 9)
    pc = PlannerConfig(pinned_budget=int(budget_gib * GIB))
    nxt, lat, host_b, pcie_b = 0, [], [], []
    for _ in range(switches):
        pc.victim_order = [1 - nxt]
        st = e.switch_to(nxt, pc)
        assert st["mismatches"] == 0, st
        nxt = 1 - nxt
        lat.append(st["wall_s"] + st["plan_s"])
        host_b.append(st["host_bytes"])
        pcie_b.append(st["pcie_h2d_bytes"] + st["pcie_d2h_bytes"])
    peak = e.pinned_physical()[1]
    bad = e.verify_pattern(0, 9) + e.verify_pattern(1, 9)
    threads = e.host_threads()
    e.close()
    steady = lat[2:] if len(lat) > 2 else lat
    p50 = statistics.median(steady)
    hb = statistics.median(host_b[2:] if len(host_b) > 2 else host_b)
    model = None
    scn = os.path.join(ROOT, "paper_2601_11743_b200", "scenarios", f"c4_budget_{int(budget_gib)}g.scn")
    if ws_gib == 16 and float(budget_gib).is_integer() and os.path.exists(scn):
        t = run_scenario_model(open(scn).read())
        ts = [ln.split() for ln in t.splitlines() if ln.startswith("T ")]
        model = [round(float(x[3]) - float(x[2]), 4) for x in ts]
    host_gbs = hb / p50 / 1e9
    pb = statistics.median(pcie_b[2:] if len(pcie_b) > 2 else pcie_b)
    # Host DRAM traffic of a switch: every PCIe byte is a DMA read or write of
    # host memory, every host-copy byte is read once and written once. The
    # ceiling is the host copy pool's own DRAM traffic at its calibrated peak
    # (2 x its payload GB/s): what the memory system sustained for copies.
    dram_gbs = (pb + 2 * hb) / p50 / 1e9
    return {"series": "engine", "pinned_budget_gib": budget_gib, "ws_gib": ws_gib, "switch_latency_s": [round(x, 4) for x in lat],
            "steady_latency_s": round(p50, 4), "pinned_peak_bytes": peak, "budget_held": peak <= budget_gib * GIB,
            "byte_exact": bad == 0, "host_threads": threads, "host_calibration": hc,
            "host_bytes_per_switch": hb, "pcie_bytes_per_switch": statistics.median(pcie_b),
            "host_copy": {"achieved_gbs": round(host_gbs, 2), "peak_gbs": round(hc["peak_gbs"], 2),
                          "frac": round(host_gbs / hc["peak_gbs"], 3) if hc["peak_gbs"] else None,
                          "what": "host-copy payload of a steady switch / its latency vs the copy pool's standalone peak"},
            "host_roofline": {"bound": "host DRAM", "achieved_gbs": round(dram_gbs, 2), "peak_gbs": round(2 * hc["peak_gbs"], 2),
                              "frac": round(dram_gbs / (2 * hc["peak_gbs"]), 3) if hc["peak_gbs"] else None,
                              "what": "(PCIe DMA bytes + 2 x host-copy bytes) of a steady switch / its latency vs 2 x the "
                                      "copy pool's standalone payload peak (a copy reads and writes each byte)"},
            "reference_model_latency_s": model}


def uvm_measured(ws_gib: int, prefetch: int) -> dict:
    p = subprocess.run([UVM, "--cap-gib", str(ws_gib + 1), "--ws-gib", str(ws_gib), "--rounds", "2", "--prefetch", str(prefetch)],
                       capture_output=True, text=True, timeout=1800)
    if p.returncode != 0:
        return {"series": "uvm", "prefetch": prefetch, "error": p.stderr[-300:]}
    r = json.loads(p.stdout.strip().splitlines()[-1])
    return {"series": "uvm_measured", "prefetch": prefetch, "ws_gib": ws_gib, "switch_ms_median": r["median_ms"],
            "switch_ms": r["switch_cost_ms"], "byte_exact": r["mismatches"] == 0,
            "host_mem_used_peak_bytes": r.get("host_mem_used_peak_bytes"), "host_peak_rss_bytes": r.get("host_peak_rss_bytes")}


def uvm_model_mirror(ws_gib: int) -> dict:
    """UvmSim (the reference's UVM model, our drop-in) on the same round robin:
    its pinned-mirror peak (uvm.hpp:58-63)."""
    h = ctypes.c_void_p()
    bw = 52.4 * GIB
    check(lib.nx_uvm_create(ctypes.c_uint64((ws_gib + 1) * GIB), ctypes.c_double(bw), ctypes.c_double(bw), 1,
                            ctypes.c_double(30e-6), 15, ctypes.byref(h)))
    try:
        for a in (0, 1):
            check(lib.nx_uvm_register(h, a, ctypes.c_uint64(ws_gib * GIB)))
        t = 0.0
        dur = ctypes.c_double()
        for k in range(6):
            check(lib.nx_uvm_touch(h, k % 2, ctypes.c_double(0.01), ctypes.c_double(t), ctypes.byref(dur)))
            t += dur.value
        f, fb, mp = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        check(lib.nx_uvm_stats(h, ctypes.byref(f), ctypes.byref(fb), ctypes.byref(mp)))
    finally:
        lib.nx_uvm_destroy(h)
    return {"series": "uvm_model", "ws_gib": ws_gib, "pinned_mirror_peak_bytes": mp.value, "faults": f.value,
            "model": "UvmSim (proj/src/uvm.cpp:114-193) via nx_uvm_*: every GPU-resident page keeps a pinned host page"}


def budget_at_latency(points: list, target_s: float):
    """Smallest budget whose steady latency is <= target (interpolated)."""
    pts = sorted((p["pinned_budget_gib"], p["steady_latency_s"]) for p in points)
    if pts[0][1] <= target_s:
        return pts[0][0]
    for (b0, l0), (b1, l1) in zip(pts, pts[1:]):
        if l1 <= target_s < l0:
            return b0 + (b1 - b0) * (l0 - target_s) / (l0 - l1)
    return None


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--budgets", default="2,4,8,12,16,24,32")
    ap.add_argument("--switches", type=int, default=6)
    ap.add_argument("--ws-gib", type=int, default=16)
    ap.add_argument("--no-uvm", action="store_true")
    a = ap.parse_args()
    pts = []
    for b in [float(x) for x in a.budgets.split(",")]:
        pts.append(engine_point(b, a.ws_gib, a.switches))
        print(json.dumps(pts[-1]), flush=True)
    if a.no_uvm:
        return 0
    mirror = uvm_model_mirror(a.ws_gib)
    print(json.dumps(mirror), flush=True)
    uvms = [uvm_measured(a.ws_gib, pf) for pf in (0, 1)]
    for u in uvms:
        print(json.dumps(u), flush=True)
    summ = {"series": "summary", "uvm_pinned_mirror_bytes": mirror["pinned_mirror_peak_bytes"], "equal_latency": []}
    for u in uvms:
        if "switch_ms_median" not in u:
            continue
        b = budget_at_latency(pts, u["switch_ms_median"] / 1e3)
        summ["equal_latency"].append({
            "uvm": "prefetch" if u["prefetch"] else "fault-driven", "uvm_latency_s": u["switch_ms_median"] / 1e3,
            "engine_budget_gib_at_equal_latency": round(b, 3) if b is not None else None,
            "fraction_of_uvm_pinned_mirror": round(b * GIB / mirror["pinned_mirror_peak_bytes"], 4) if b is not None else None,
            "paper": "33.2-40.2% (PAPER.md:342, RTX 5090)"})
    print(json.dumps(summ), flush=True)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
