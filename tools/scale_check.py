"""Full-size real-engine parity runs (development tool; tests/test_gpu_scale.py is the gate)."""
import hashlib, json, sys, time
sys.path.insert(0, '.')
from paper_2601_11743_b200 import load_scenario, run_scenario_real, trace_lines
g = json.load(open('tests/golden/scenarios.json'))
names = sys.argv[1:] or ['c2_interactive_background', 'c4_budget_2g', 'c4_budget_8g', 'x16_exchange']
for name in names:
    t0 = time.time()
    real = run_scenario_real(load_scenario(name), seed=11)
    dt = time.time() - t0
    det = hashlib.sha256("\n".join(trace_lines(real)).encode()).hexdigest()
    v = [ln for ln in real.splitlines() if ln[0] in 'VF']
    print(json.dumps({"name": name, "secs": round(dt, 1), "parity": det == g[name]['det_sha256'], "VF": v}), flush=True)
