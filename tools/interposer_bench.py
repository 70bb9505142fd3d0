"""Config 2 through the interposer: two UNMODIFIED CUDA applications
(tests/apps/vecapp.cu) of 16 GiB (interactive) and 24 GiB (background) on one
B200 capped at 32 GiB (16 GiB pinned budget), run under nixied +
LD_PRELOAD=libnixie_shim.so. Each app computes on its whole working set every
iteration (device-side check of every word) and thinks between iterations,
so the MLFQ switches at every think gap (the holder goes idle) and every
steady-state switch exchanges 8 GiB each way.

Prints one JSON line per switch kind plus a summary; writes the daemon log to
--out (JSON lines)."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_11743_b200.interpose import VECAPP, Daemon, run_apps  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpu", default="32G")
    ap.add_argument("--pinned", default="16G")
    ap.add_argument("--a-mib", type=int, default=16384)
    ap.add_argument("--b-mib", type=int, default=24576)
    ap.add_argument("--iters", type=int, default=12)
    ap.add_argument("--think-ms", type=float, default=300)
    ap.add_argument("--host-check", type=int, default=0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--daemon-arg", action="append", default=[], help="extra nixied flag (repeatable)")
    a = ap.parse_args()
    with Daemon(gpu=a.gpu, pinned=a.pinned, paged="96G", log=a.out, extra=a.daemon_arg) as d:
        cmds = [[VECAPP, "--mib", str(a.a_mib), "--buffers", "8", "--iters", str(a.iters), "--think-ms", str(a.think_ms),
                 "--seed", "7", "--name", "interactive", "--host-check", str(a.host_check)],
                [VECAPP, "--mib", str(a.b_mib), "--buffers", "12", "--iters", str(a.iters), "--think-ms", str(a.think_ms),
                 "--seed", "9", "--name", "background", "--host-check", str(a.host_check)]]
        res = run_apps(d, cmds, timeout=1800, stagger_s=0.5)
        sw = d.switches()
        err = d.stderr()
    ok = all(r["rc"] == 0 for r in res)
    steady = [s for s in sw if s["pcie_h2d"] > 0 and s["pcie_d2h"] > 0 and s["host_bytes"] == 0]
    summ = {"apps_ok": ok, "apps": [r["out"] for r in res], "switches": len(sw), "steady_switches": len(steady)}
    if steady:
        # The first two steady switches map slabs for the first time (and, in
        # the default mapping mode, settle the slab pairs): reported apart, as
        # warm-up, like bench.py's untimed steps.
        first, warm = (steady[:2], steady[2:]) if len(steady) > 4 else ([], steady)
        gbps = [(s["pcie_h2d"] + s["pcie_d2h"]) / (s["copy_ms"] * 1e-3) / 1e9 for s in warm]
        tot = [s["total_ms"] for s in warm]
        summ["warmup_switch_ms"] = [round(s["total_ms"], 1) for s in first]
        summ.update({
            "bytes_each_way_gib": statistics.median([s["pcie_h2d"] for s in steady]) / (1 << 30),
            "copy_bidir_gbps_median": statistics.median(gbps),
            "switch_total_ms": {"p50": statistics.median(tot), "max": max(tot), "min": min(tot)},
            "copy_ms_median": statistics.median([s["copy_ms"] for s in warm]),
            "grant_ms_median": statistics.median([s["grant_ms"] for s in warm]),
            "pause_ms_median": statistics.median([s["pause_ms"] for s in warm]),
            "verified": sum(s["verified"] for s in sw), "mismatches": sum(s["mismatches"] for s in sw),
        })
    if not ok:
        summ["errors"] = [r["stderr"][-400:] for r in res] + [err[-400:]]
    print(json.dumps(summ))


if __name__ == "__main__":
    main()
