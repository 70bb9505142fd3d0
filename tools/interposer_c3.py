"""BASELINE config 3 through the interposer: three UNMODIFIED CUDA programs
(tests/apps/vecapp.cu) under nixied + libnixie_shim.so on one B200 capped at
32 GiB (16 GiB pinned), MLFQ with the paper's constants.
  code completion  16 GiB, a request every --interval s, ~100 ms of compute
  image generation 24 GiB, a request every 5 s, ~1 s of compute
  batch OCR        12 GiB, pages of ~250 ms with 150 ms I/O gaps
Each request is one vecapp iteration (every word of the working set checked
on the device); its latency includes any wait at the launch gate and the swap
that grants it. Prints one JSON line (per-app latency, switches)."""
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
    ap.add_argument("--interval", type=float, default=3.0)
    ap.add_argument("--horizon", type=float, default=60.0)
    ap.add_argument("--prefetch", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("--slab-mib", type=int, default=None)
    a = ap.parse_args()
    h = a.horizon
    apps = [
        ("code-completion", 16384, 8, 18, a.interval, int(h / (a.interval + 0.15))),
        ("image-gen", 24576, 12, 120, 5.0, int(h / 6.0)),
        ("batch-ocr", 12288, 6, 60, 0.15, int(h / 0.5)),
    ]
    cmds = [[VECAPP, "--mib", str(mib), "--buffers", str(bufs), "--passes", str(passes), "--think-ms", str(think * 1e3),
             "--iters", str(iters), "--seed", str(i + 3), "--name", name, "--host-check", "0"]
            for i, (name, mib, bufs, passes, think, iters) in enumerate(apps)]
    with Daemon(gpu="32G", pinned="16G", paged="96G", log=a.out, prefetch=a.prefetch, slab_mib=a.slab_mib) as d:
        res = run_apps(d, cmds, timeout=h * 4 + 300, stagger_s=0.2)
        sw = d.switches()
    grants = sorted(s["grant_ms"] for s in sw)
    out = {"interval_s": a.interval, "horizon_s": h, "prefetch": a.prefetch, "slab_mib": a.slab_mib or 512,  # the daemon default for a 32 GiB budget
           "switches": len(sw),
           "grant_ms": {"p50": grants[len(grants) // 2] if grants else None, "max": grants[-1] if grants else None},
           "apps_ok": all(r["rc"] == 0 for r in res),
           "mismatches": sum(s["mismatches"] for s in sw), "verified": sum(s["verified"] for s in sw),
           "switch_ms": {"p50": statistics.median([s["total_ms"] for s in sw]) if sw else None,
                         "max": max([s["total_ms"] for s in sw]) if sw else None},
           "swapped_gib": round(sum(s["pcie_h2d"] + s["pcie_d2h"] for s in sw) / (1 << 30), 1),
           "per_app": {r["out"]["name"]: {"requests": r["out"]["iters"], "request_ms": r["out"]["iter_ms"],
                                          "device_errors": r["out"]["device_errors"]} if r["out"] else {"error": r["stderr"][-300:]}
                       for r in res}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
