"""Paired A/B of engine tunables on config 2 (bench.py's workload) inside one
engine: variants take turns, two switches each (one per direction) per round,
so a noisy shared host affects every variant alike. SwapEngine.set_option
changes the per-switch tunables between switches.

Usage: python tools/ab_switch.py [--rounds 12] VARIANT [VARIANT ...]
  VARIANT = comma-separated k=v (engine options), "base" = no change from the
  engine defaults. Example:
    python tools/ab_switch.py base early_frame_release=0,d2h_commit_legs=0 d2h_commit_legs=128
Prints one JSON line per variant (median device span and wall per switch,
paired delta vs the first variant) and writes the raw samples with --out."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_11743_b200 import GIB, MIB, PlannerConfig, SwapEngine, parse_path  # noqa: E402
from paper_2601_11743_b200._lib import TIER_GPU, TIER_PINNED  # noqa: E402

DEFAULTS = {"legs_per_launch": 128, "first_batch_legs": 8, "d2h_commit_legs": 32, "early_frame_release": 1,
            "k3_verify_group": 4096, "pace_lag_legs": 64, "fetch_first_pump": 1,
            "sm_tma_ctas": -1}


def parse(v: str) -> dict:
    if v == "base":
        return {}
    return {kv.split("=")[0]: int(kv.split("=")[1]) for kv in v.split(",")}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=12)
    ap.add_argument("--out")
    ap.add_argument("--path", default="auto", help="copy path: auto, sm or ce (sm: K1 / K1T variants via sm_tma_ctas)")
    ap.add_argument("variants", nargs="+")
    a = ap.parse_args()
    variants = [(v, {**DEFAULTS, **parse(v)}) for v in a.variants]
    e = SwapEngine(gpu_capacity=32 * GIB, pinned_capacity=16 * GIB, paged_capacity=2 * GIB, path=parse_path(a.path))
    probe = e.probe_pcie(1 * GIB, 64 * MIB)
    e.allocate(0, 16 * GIB, TIER_GPU)
    e.allocate(1, 16 * GIB, TIER_GPU)
    e.allocate(1, 8 * GIB, TIER_PINNED)
    e.fill_pattern(0, 7)
    e.fill_pattern(1, 7)
    pc = PlannerConfig(streaming_window=512 * MIB, pinned_budget=16 * GIB)
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
                samples[name].append({"round": r, "span_ms": st["device_span_s"] * 1e3,
                                      "wall_ms": (st["wall_s"] + st["plan_s"]) * 1e3, "ce_calls": st["ce_calls"], "pace_waits": st["pace_waits"],
                                      "ce_batches": [st["ce_batches_h2d"], st["ce_batches_d2h"]],
                                      "k3_s": st["k3_s"], "k3_kernel_s": st["k3_kernel_s"], "k3_bytes": st["k3_bytes"],
                                      "k3_launches": st["k3_launches"]})
    exact = e.verify_pattern(0, 7) == 0 and e.verify_pattern(1, 7) == 0
    e.close()
    base = variants[0][0]

    def per_round(name, key):
        d = {}
        for s in samples[name]:
            d.setdefault(s["round"], []).append(s[key])
        return {k: sum(v) / len(v) for k, v in d.items()}

    b_span = per_round(base, "span_ms")
    for name, opts in variants:
        sp = [s["span_ms"] for s in samples[name]]
        wl = [s["wall_ms"] for s in samples[name]]
        mine = per_round(name, "span_ms")
        deltas = [mine[k] - b_span[k] for k in mine if k in b_span]
        print(json.dumps({"variant": name, "options": opts, "n": len(sp), "span_ms_p50": round(statistics.median(sp), 2),
                          "span_ms_min": round(min(sp), 2), "wall_ms_p50": round(statistics.median(wl), 2),
                          "paired_delta_ms_p50_vs_" + base: round(statistics.median(deltas), 2) if deltas else None,
                          "gbs_p50": round(16 * GIB / (statistics.median(sp) * 1e-3) / 1e9, 2),
                          "ce_calls_p50": statistics.median(s["ce_calls"] for s in samples[name]),
                          "pace_waits_p50": statistics.median(s["pace_waits"] for s in samples[name]),
                          "k3_launches_p50": statistics.median(s["k3_launches"] for s in samples[name]),
                          "k3_event_gbs": round(sum(s["k3_bytes"] for s in samples[name]) / max(1e-12, sum(s["k3_s"] for s in samples[name])) / 1e9, 1),
                          "k3_kernel_gbs": round(sum(s["k3_bytes"] for s in samples[name]) / max(1e-12, sum(s["k3_kernel_s"] for s in samples[name])) / 1e9, 1),
                          "probe_ce_bidir_total": round(probe["ce_bidir_total"], 2), "byte_exact": exact}), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"probe": probe, "samples": samples}, f)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
