"""Paired A/B of engine tunables on config 4 (16 GiB <-> 16 GiB at a 16 GiB
GPU cap, pinned budget B, both apps starting in pageable memory): one engine
per budget, variants take turns (two switches each per round, one per
direction), so a noisy shared host affects every variant alike.

Usage: python tools/ab_c4.py [--budgets 2,8] [--rounds 4] VARIANT [VARIANT ...]
  VARIANT = comma-separated k=v (SwapEngine.set_option), "base" = defaults.
Prints one JSON line per (budget, variant): median switch wall, paired delta
vs the first variant, byte exactness."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_11743_b200 import GIB, PlannerConfig, SwapEngine  # noqa: E402
from paper_2601_11743_b200._lib import TIER_PAGED  # noqa: E402

DEFAULTS = {"legs_per_launch": 128, "first_batch_legs": 8, "d2h_commit_legs": 32, "early_frame_release": 1,
            "k3_verify_group": 4096, "pace_lag_legs": 64, "fetch_first_pump": 1, "host_streaming_copy": 1}


def parse(v: str) -> dict:
    if v == "base":
        return {}
    return {kv.split("=")[0]: int(kv.split("=")[1]) for kv in v.split(",")}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--budgets", default="2,8")
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("variants", nargs="+")
    a = ap.parse_args()
    variants = [(v, {**DEFAULTS, **parse(v)}) for v in a.variants]
    for budget in (int(x) for x in a.budgets.split(",")):
        e = SwapEngine(gpu_capacity=16 * GIB, pinned_capacity=budget * GIB, paged_capacity=64 * GIB)
        e.allocate(0, 16 * GIB, TIER_PAGED)
        e.allocate(1, 16 * GIB, TIER_PAGED)
        e.fill_pattern(0, 9)
        e.fill_pattern(1, 9)
        pc = PlannerConfig(pinned_budget=budget * GIB)
        nxt = 0

        def switch():
            nonlocal nxt
            pc.victim_order = [1 - nxt]
            st = e.switch_to(nxt, pc)
            assert st["mismatches"] == 0 and st["unverified"] == 0, st
            nxt = 1 - nxt
            return st

        for _ in range(3):
            switch()
        samples = {v: [] for v, _ in variants}
        for r in range(a.rounds):
            order = variants if r % 2 == 0 else variants[::-1]
            for name, opts in order:
                for k, val in opts.items():
                    e.set_option(k, val)
                for _ in range(2):
                    st = switch()
                    samples[name].append({"round": r, "wall_ms": (st["wall_s"] + st["plan_s"]) * 1e3,
                                          "pace_waits": st["pace_waits"]})
        exact = e.verify_pattern(0, 9) == 0 and e.verify_pattern(1, 9) == 0
        e.close()
        base = variants[0][0]

        def per_round(name):
            d = {}
            for s in samples[name]:
                d.setdefault(s["round"], []).append(s["wall_ms"])
            return {k: sum(v) / len(v) for k, v in d.items()}

        b = per_round(base)
        for name, opts in variants:
            w = [s["wall_ms"] for s in samples[name]]
            mine = per_round(name)
            deltas = [mine[k] - b[k] for k in mine if k in b]
            print(json.dumps({"pinned_gib": budget, "variant": name, "n": len(w), "wall_ms_p50": round(statistics.median(w), 2),
                              "wall_ms_min": round(min(w), 2),
                              "paired_delta_ms_p50_vs_" + base: round(statistics.median(deltas), 2),
                              "pace_waits_p50": statistics.median(s["pace_waits"] for s in samples[name]),
                              "byte_exact": exact}), flush=True)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
