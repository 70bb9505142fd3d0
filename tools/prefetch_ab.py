"""Config 3 on one B200 with and without MLFQ prefetch: the
3-app mix (16 + 24 + 12 GiB on a 32 GiB budget) with a small pinned budget,
so part of the working sets lives in pageable memory and every switch that
brings it back pays the two-hop path unless the scheduler's next candidate
was prefetched into pinned while the incumbent computed.
Usage: python tools/prefetch_ab.py [horizon_s] [pinned_gib] [interval_s]"""
import json
import sys

sys.path.insert(0, ".")
from paper_2601_11743_b200.workload import config3_mix, run_workload  # noqa: E402

horizon = float(sys.argv[1]) if len(sys.argv) > 1 else 30.0
pinned = int(sys.argv[2]) if len(sys.argv) > 2 else 8
interval = float(sys.argv[3]) if len(sys.argv) > 3 else 3.0
for pf in (False, True):
    r = run_workload(config3_mix(interval), horizon_s=horizon, pinned_gib=pinned, prefetch=pf)
    r["interval_s"] = interval
    print(json.dumps(r), flush=True)
