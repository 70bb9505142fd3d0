"""Differential fuzz: product lanes (1..64 legs per lane) vs the unmodified
reference on seeded random tiny scenarios."""
import subprocess, sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
from scenario_gen import random_scenario
from paper_2601_11743_b200 import run_scenario_model, NixieError, trace_lines
lo, hi = int(sys.argv[1]), int(sys.argv[2])
stats = {"ok": 0, "ref_err": 0, "bad": []}
for seed in range(lo, hi):
    spec = random_scenario(seed)
    p = subprocess.run(['oracle/_ref/ref_trace', '-'], input=spec, capture_output=True, text=True)
    if p.returncode != 0:
        stats["ref_err"] += 1
        try:
            run_scenario_model(spec); stats["bad"].append((seed, 1, "product ok, ref failed"))
        except NixieError:
            pass
        continue
    stats["ok"] += 1
    if run_scenario_model(spec) != p.stdout:
        stats["bad"].append((seed, 1, "exact"))
    for k in (2, 4, 8, 64):
        try:
            if trace_lines(run_scenario_model(spec, k)) != trace_lines(p.stdout):
                stats["bad"].append((seed, k, "det"))
        except NixieError as e:
            stats["bad"].append((seed, k, str(e)[:60]))
print(stats["ok"], stats["ref_err"], len(stats["bad"]), stats["bad"][:20])
