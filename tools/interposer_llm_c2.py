"""BASELINE config 2 with real model stacks under the interposer: an
interactive Qwen3-8B-sized LLM (16 GiB of bf16 weights) and a FLUX-sized
12.8B model (24 GiB) as two unmodified PyTorch programs
(tests/apps/llm_app.py, random weights) on one B200 capped at 32 GiB, 16 GiB
pinned. Both think between requests, so the MLFQ switches whenever the holder
goes idle; every switch moves ~8 GiB each way. Each app checks that every
request's logits equal its first request's bit for bit."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_11743_b200.interpose import Daemon, run_apps  # noqa: E402

LLM = os.path.join(ROOT, "tests", "apps", "llm_app.py")
reqs = int(sys.argv[1]) if len(sys.argv) > 1 else 12
out = (sys.argv[2] or None) if len(sys.argv) > 2 else None
slab = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "0" else None
flags = sys.argv[4].split(",") if len(sys.argv) > 4 else []
ref_victims = "ref" in flags  # the planner's own victim blocks
isolate = "isolate" in flags  # --isolate-victims
nopace = "nopace" in flags  # --pace-lag -1
slack = int(sys.argv[5]) if len(sys.argv) > 5 else None  # physical slack slabs
with Daemon(gpu="32G", pinned="16G", paged="96G", log=out, slab_mib=slab,
            extra=(["--reference-victims"] if ref_victims else []) + (["--isolate-victims"] if isolate else []) + (["--phys-slack", str(slack)] if slack is not None else []) + (["--pace-lag", "-1"] if nopace else [])) as d:
    res = run_apps(d, [[sys.executable, LLM, str(reqs), "1.0", "1", "qwen3-8b", "1", "512"],
                       [sys.executable, LLM, str(reqs), "1.5", "2", "flux-12b", "1", "1024"]], timeout=1800, stagger_s=1.0)
    sw = d.switches()
    grows = sum(1 for r in d.records() if r.get("event") == "slab_grow")
    drops = sum(1 for r in d.records() if r.get("event") == "slab_drop")
    err = d.stderr()
    daemon_rc = d.proc.poll()
steady = [s for s in sw if s["pcie_h2d"] > (1 << 30) and s["pcie_d2h"] > (1 << 30)]
summary = {"apps_ok": all(r["rc"] == 0 for r in res), "apps": [r["out"] for r in res], "switches": len(sw),
           "steady_switches": len(steady),
           "steady_gib_each_way": round(statistics.median([s["pcie_h2d"] for s in steady]) / 2**30, 2) if steady else None,
           "copy_bidir_gbps_median": round(statistics.median([(s["pcie_h2d"] + s["pcie_d2h"]) / (s["copy_ms"] * 1e-3) / 1e9 for s in steady]), 1) if steady else None,
           "switch_ms": {"p50": statistics.median([s["total_ms"] for s in steady]), "max": max(s["total_ms"] for s in steady)} if steady else None,
           "verified": sum(s["verified"] for s in sw), "mismatches": sum(s["mismatches"] for s in sw),
           "slab_mib": slab or 512, "victims": "reference" if ref_victims else "slab", "phys_slack": slack, "isolate_victims": isolate, "slabs_grown": grows, "slabs_dropped": drops,
           "live_slabs_after_switches": [s["live_slabs"] for s in sw][-6:],
           "grant_ms_p50": statistics.median([s["grant_ms"] for s in steady]) if steady else None}
if not summary["apps_ok"]:
    summary["errors"] = [r["stderr"][-500:] for r in res] + [d.stderr()[-2000:]]  # after the daemon exited
    summary["daemon_rc"] = daemon_rc
print(json.dumps(summary))
