"""Golden random instances (tests/golden/random_tiny.json, the robust ones)
through the CUDA engine under several engine shapes; reports every case
whose decisions differ from the reference's or that fails (deadlock).

Usage: python tools/fuzz_real.py [shape indices, e.g. 0,1,2]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_11743_b200 import NixieError, run_scenario_real, trace_lines  # noqa: E402
from paper_2601_11743_b200._lib import PATH_CE, PATH_SM  # noqa: E402

SHAPES = [dict(path=PATH_CE), dict(path=PATH_CE, pace_lag_legs=0, d2h_commit_legs=1, first_batch_legs=1),
          dict(path=PATH_CE, pace_lag_legs=2, legs_per_launch=3, pcie_legs_in_flight=5),
          dict(path=PATH_CE, pace_lag_legs=-1, early_frame_release=False),
          dict(path=PATH_SM, legs_per_launch=2), dict(path=PATH_CE, pace_lag_legs=1, pcie_legs_in_flight=1),
          dict(path=PATH_CE, pace_lag_legs=-1), dict(path=PATH_CE, pace_lag_legs=-1, pcie_legs_in_flight=1)]
which = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else range(len(SHAPES))
cases = [c for c in json.load(open(os.path.join(ROOT, "tests", "golden", "random_tiny.json"))) if c["robust"]]
for si in which:
    bad = []
    for c in cases:
        try:
            real = run_scenario_real(c["spec"], seed=7, host_threads=2, **SHAPES[si])
        except NixieError as e:
            bad.append((c["seed"], str(e)[:160]))
            continue
        if trace_lines(real) != trace_lines(c["trace"]):
            bad.append((c["seed"], "decisions differ"))
        elif any(ln.split()[3] != "0" for ln in real.splitlines() if ln.startswith("V ")):
            bad.append((c["seed"], "bytes differ"))
    print(json.dumps({"shape": si, "opts": SHAPES[si], "cases": len(cases), "bad": bad}), flush=True)
