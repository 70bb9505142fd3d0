"""Per-switch timeline of config 2 (bench.py's workload): where the link idles.

For each steady switch it reads the engine's batch trace (nx_batch_trace:
device start / copy end / end of every PCIe batch, and the host times of its
submission and commit) and attributes the device span to
  head    first batch start .. first H2D batch start (fetches wait for the
          first evictions to land: the GPU is full)
  both    both directions copying
  d2h_only / h2d_only   one direction copying alone
  idle    neither direction copying (host or dependency stalls)
  tail    last copy end .. span end (arrival checks after the last copy)
and reports per-stream gaps between consecutive batches.

Usage: python tools/timeline.py [--switches 6] [--out gpurun_out/timeline.json] [engine overrides k=v ...]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GIB, MIB = 1 << 30, 1 << 20


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def measure(iv_a, iv_b, t0, t1):
    """Seconds in [t0,t1] covered by both / only a / only b / neither."""
    pts = sorted({t0, t1, *[x for ab in iv_a + iv_b for x in ab]})
    both = oa = ob = none = 0.0

    def cov(iv, t):
        return any(a <= t < b for a, b in iv)
    for x, y in zip(pts, pts[1:]):
        if y <= t0 or x >= t1:
            continue
        m = (x + y) / 2
        ca, cb = cov(iv_a, m), cov(iv_b, m)
        d = y - x
        if ca and cb:
            both += d
        elif ca:
            oa += d
        elif cb:
            ob += d
        else:
            none += d
    return both, oa, ob, none


def analyse(tr, st):
    h = [b for b in tr if b["stream"] == 0]
    d = [b for b in tr if b["stream"] == 1]
    start = min(b["start_s"] for b in tr)
    end = max(b["end_s"] for b in tr)
    copy_end = max(b["copied_s"] for b in tr)
    iv_h = union([[b["start_s"], b["copied_s"]] for b in h])
    iv_d = union([[b["start_s"], b["copied_s"]] for b in d])
    both, d_only, h_only, idle = measure(iv_d, iv_h, start, copy_end)

    def gaps(bs):
        bs = sorted(bs, key=lambda b: b["start_s"])
        return [round((y["start_s"] - x["copied_s"]) * 1e3, 3) for x, y in zip(bs, bs[1:]) if y["start_s"] - x["copied_s"] > 20e-6]
    return {
        "span_ms": (end - start) * 1e3, "device_span_ms": st["device_span_s"] * 1e3,
        "wall_ms": st["wall_s"] * 1e3, "plan_ms": st["plan_s"] * 1e3,
        "head_ms": ((min(b["start_s"] for b in h) - start) * 1e3) if h else None,
        "first_d2h_legs": sorted(d, key=lambda b: b["start_s"])[0]["legs"] if d else None,
        "d2h_end_ms": (max(b["copied_s"] for b in d) - start) * 1e3 if d else None,
        "h2d_end_ms": (max(b["copied_s"] for b in h) - start) * 1e3 if h else None,
        "tail_ms": (end - copy_end) * 1e3,
        "both_ms": both * 1e3, "d2h_only_ms": d_only * 1e3, "h2d_only_ms": h_only * 1e3, "idle_ms": idle * 1e3,
        "batches": [len(h), len(d)], "h2d_gaps_ms": gaps(h), "d2h_gaps_ms": gaps(d),
        "h2d_rate_gbs": sum(b["legs"] for b in h) * 2 * MIB / max(1e-9, sum(y - x for x, y in iv_h)) / 1e9,
        "d2h_rate_gbs": sum(b["legs"] for b in d) * 2 * MIB / max(1e-9, sum(y - x for x, y in iv_d)) / 1e9,
        "host_first_submit_ms": min(b["host_submit_s"] for b in tr) * 1e3,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--switches", type=int, default=6)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "timeline.json"))
    ap.add_argument("overrides", nargs="*", help="EngineConfig field=value")
    a = ap.parse_args()
    from paper_2601_11743_b200 import PlannerConfig, SwapEngine
    from paper_2601_11743_b200._lib import TIER_GPU, TIER_PINNED
    ov = {}
    for kv in a.overrides:
        k, v = kv.split("=")
        ov[k] = int(v) if v.lstrip("-").isdigit() else v
    eng = SwapEngine(gpu_capacity=32 * GIB, pinned_capacity=16 * GIB, paged_capacity=2 * GIB, **ov)
    probe = eng.probe_pcie(1 * GIB, 64 * MIB)
    eng.allocate(0, 16 * GIB, TIER_GPU)
    eng.allocate(1, 16 * GIB, TIER_GPU)
    eng.allocate(1, 8 * GIB, TIER_PINNED)
    eng.fill_pattern(0, 7)
    eng.fill_pattern(1, 7)
    pc = PlannerConfig(streaming_window=512 * MIB, pinned_budget=16 * GIB)
    nxt = 0
    rows, raw = [], []
    for i in range(a.switches + 2):
        pc.victim_order = [1 - nxt]
        st = eng.switch_to(nxt, pc)
        nxt = 1 - nxt
        if i < 2:
            continue
        tr = eng.batch_trace()
        raw.append({"stats": {k: st[k] for k in ("bytes_in", "bytes_out", "device_span_s", "wall_s", "plan_s")}, "batches": tr,
                    "k3": eng.k3_trace()})
        row = analyse(tr, st)
        row["ce_calls"] = st["ce_calls"]
        row["mib_per_ce_call"] = (st["pcie_h2d_bytes"] + st["pcie_d2h_bytes"]) / MIB / max(1, st["ce_calls"])
        for k in ("ce_calls_dir", "run_breaks_src", "run_breaks_dst"):
            row[k] = st[k]
        rows.append(row)
    bad = eng.verify_pattern(0, 7) + eng.verify_pattern(1, 7)
    eng.close()
    summary = {"probe": {k: probe[k] for k in ("ce_bidir_h2d", "ce_bidir_d2h", "ce_bidir_total", "ce_h2d", "ce_d2h")},
               "overrides": ov, "byte_exact": bad == 0, "switches": rows}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump({"summary": summary, "raw": raw}, f)
    for r in rows:
        print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items() if not k.endswith("gaps_ms")}))
        print("  gaps h2d", r["h2d_gaps_ms"][:12], "d2h", r["d2h_gaps_ms"][:12])
    print(json.dumps(summary["probe"]), "byte_exact", bad == 0)


if __name__ == "__main__":
    main()
