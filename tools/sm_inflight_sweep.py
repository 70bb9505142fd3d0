"""Is the SM copy path's bidirectional ceiling an in-flight (Little's law)
limit of the kernel, or the host link's? Sweeps the raw SM copy variants
(copy_variants.cu: 0 = LDG/STG 16 B x 8 per thread, 32 KiB in flight per
256-thread CTA; 2 = TMA bulk ring, 4 x 32 KiB = 128 KiB in flight per CTA)
over grid sizes, H2D alone, D2H alone and both at once, beside the mixed
shapes (10 = CE H2D + SM D2H, 11 = SM H2D + CE D2H) and the copy engines.

If the SM rate were bound by requests in flight, it would keep rising with
the grid (bytes in flight = CTAs x per-CTA depth) until the link saturates.
A plateau below the copy engines' rate that no grid size or depth moves
means the limit sits past the SMs: the 128-byte PCIe requests SM traffic is
cut into.

Usage: python tools/sm_inflight_sweep.py [--mib 2048] [--passes 3] [--out profiles/r02_sm_inflight_sweep.json]"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_11743_b200 import GIB, MIB, SwapEngine  # noqa: E402
from paper_2601_11743_b200._lib import check, lib  # noqa: E402

INFLIGHT_PER_CTA = {0: 256 * 8 * 16, 2: 4 * 32 * 1024}


def probe(e: SwapEngine, variant: int, nbytes: int, ctas: int) -> dict:
    out = (ctypes.c_double * 3)()
    check(lib.nx_probe_copy_variant(e._h, variant, nbytes, ctas, out))
    return {"h2d": round(out[0], 2), "d2h": round(out[1], 2), "bidir_total": round(out[2], 2)}


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=2048)
    ap.add_argument("--passes", type=int, default=3)
    ap.add_argument("--out")
    a = ap.parse_args()
    nbytes = a.mib * MIB
    e = SwapEngine(gpu_capacity=1 * GIB, pinned_capacity=1 * GIB, paged_capacity=1 * GIB)
    shapes = [(v, c) for v in (0, 2) for c in (4, 8, 16, 37, 74, 148, 296, 592, 1184) if not (v == 2 and c > 296)]
    shapes += [(10, 296), (11, 296)]
    samples = {s: [] for s in shapes}
    ce_samples = []
    try:
        for _ in range(3):  # settle the link (shared hosts) before the first reading
            e.probe_pcie(1 * GIB, 64 * MIB)
        # passes over every shape, each pass with its own copy-engine reading,
        # so a host that drifts affects every shape alike
        for _ in range(a.passes):
            ce = e.probe_pcie(nbytes, 64 * MIB)
            ce_samples.append({"h2d": ce["ce_h2d"], "d2h": ce["ce_d2h"], "bidir_total": ce["ce_bidir_total"]})
            for sh in shapes:
                samples[sh].append(probe(e, sh[0], nbytes, sh[1]))
    finally:
        e.close()

    def med(rs, k):
        return round(statistics.median(r[k] for r in rs), 2)

    rows = [{"what": "copy engines, 64 MiB calls", **{k: med(ce_samples, k) for k in ("h2d", "d2h", "bidir_total")},
             "bidir_samples": [round(r["bidir_total"], 2) for r in ce_samples]}]
    for (variant, ctas), rs in samples.items():
        r = {"variant": variant, "ctas": ctas, **{k: med(rs, k) for k in ("h2d", "d2h", "bidir_total")},
             "bidir_samples": [r["bidir_total"] for r in rs]}
        if variant in INFLIGHT_PER_CTA:
            resident = min(ctas, 148 * (8 if variant == 0 else 1))
            r["inflight_kib_per_direction"] = resident * INFLIGHT_PER_CTA[variant] // 1024
        else:
            r["what"] = {10: "CE H2D + SM D2H", 11: "SM H2D + CE D2H"}[variant]
        rows.append(r)
        print(json.dumps(r), flush=True)
    res = {"bytes_per_direction": nbytes, "passes": a.passes, "statistic": "median over passes of the best of 3 timed reps",
           "rows": rows}
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)
    print(json.dumps(rows[0]))
    return 0


if __name__ == "__main__":
    sys.exit(main())
