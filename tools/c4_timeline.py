"""Config-4 switch timeline per lane (2 x 16 GiB round robin on a 16 GiB cap,
pinned budget B): from the engine's per-leg log (nx_leg_records) of a steady
switch, for each lane (gpu->pinned, pinned->gpu, pinned->paged,
paged->pinned) its legs, first start, last end and the bytes it moved in
each 25 ms bin. Shows which lane idles while another is the bottleneck.

Usage: python tools/c4_timeline.py [--budgets 8,12] [--switches 5] [k=v engine options ...]"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_11743_b200 import GIB, PlannerConfig, SwapEngine  # noqa: E402
from paper_2601_11743_b200._lib import TIER_PAGED  # noqa: E402

NAMES = {0: "gpu", 1: "pinned", 2: "paged", 3: "disk"}
BIN = 0.025


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budgets", default="8,12")
    ap.add_argument("--switches", type=int, default=5)
    ap.add_argument("--out")
    ap.add_argument("overrides", nargs="*")
    a = ap.parse_args()
    ov = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.overrides}
    rows = []
    for b in (float(x) for x in a.budgets.split(",")):
        e = SwapEngine(gpu_capacity=16 * GIB, pinned_capacity=int(b * GIB), paged_capacity=64 * GIB, **ov)
        e.allocate(0, 16 * GIB, TIER_PAGED)
        e.allocate(1, 16 * GIB, TIER_PAGED)
        e.fill_pattern(0, 9)
        e.fill_pattern(1, 9)
        pc = PlannerConfig(pinned_budget=int(b * GIB))
        nxt = 0
        for i in range(a.switches):
            pc.victim_order = [1 - nxt]
            st = e.switch_to(nxt, pc)
            nxt = 1 - nxt
            if i < 2:
                continue
            recs = e.leg_records()
            lanes = {}
            for r in recs:
                k = f"{NAMES[r['src']]}->{NAMES[r['dst']]}"
                lanes.setdefault(k, []).append(r)
            end = max(r["end_s"] for r in recs)
            nb = int(end / BIN) + 1
            out = {}
            for k, v in sorted(lanes.items()):
                bins = [0] * nb
                for r in v:
                    bins[min(nb - 1, int(r["end_s"] / BIN))] += 2
                out[k] = {"legs": len(v), "first_start_ms": round(min(r["start_s"] for r in v) * 1e3, 1),
                          "last_end_ms": round(max(r["end_s"] for r in v) * 1e3, 1),
                          "mib_landed_per_25ms": bins}
            row = {"budget_gib": b, "switch": i, "wall_ms": round((st["wall_s"] + st["plan_s"]) * 1e3, 1),
                   "host_bytes_gib": st["host_bytes"] / GIB, "pcie_gib": (st["pcie_h2d_bytes"] + st["pcie_d2h_bytes"]) / GIB,
                   "host_threads": e.host_threads(), "lanes": out}
            rows.append(row)
            print(json.dumps({k: v for k, v in row.items() if k != "lanes"}), flush=True)
            for k, v in out.items():
                print("   ", k, {kk: vv for kk, vv in v.items() if kk != "mib_landed_per_25ms"}, v["mib_landed_per_25ms"], flush=True)
        assert e.verify_pattern(0, 9) == 0 and e.verify_pattern(1, 9) == 0
        e.close()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rows, f)


if __name__ == "__main__":
    main()
