"""BASELINE config 3 on one B200: 3-app mix under MLFQ, interactive latency
at 1 s / 3 s / 6 s request intervals."""
import json, sys
sys.path.insert(0, ".")
from paper_2601_11743_b200.workload import config3_mix, run_workload
horizon = float(sys.argv[1]) if len(sys.argv) > 1 else 30.0
for interval in (1.0, 3.0, 6.0):
    r = run_workload(config3_mix(interval), horizon_s=horizon)
    r["interval_s"] = interval
    print(json.dumps(r), flush=True)
