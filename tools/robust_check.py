"""(a) shipped scenarios never deadlock for any link timing x lane concurrency;
(b) random instances the reference completes under every timing also complete
with concurrent lanes, with identical decisions."""
import glob, subprocess, sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
from scenario_gen import random_scenario
from paper_2601_11743_b200 import run_scenario_model, NixieError, trace_lines
SPEEDS = [(64, 32), (64, 1), (1, 64), (64, 64), (4, 200), (200, 4), (16, 32), (32, 16)]
def retime(base, pc, host):
    return '\n'.join(l for l in base.splitlines() if not l.startswith('link')) + \
        f"\nlink 0 {pc}GiB/s {pc}GiB/s full\nlink 1 {host}GiB/s {host}GiB/s full\n"
mode = sys.argv[1]
if mode == 'shipped':
    for f in sorted(glob.glob('paper_2601_11743_b200/scenarios/*.scn')):
        base = open(f).read(); bad = []
        ref_det = trace_lines(run_scenario_model(base))
        for (pc, host) in SPEEDS:
            for k in (1, 2, 8, 64, 256):
                try:
                    t = run_scenario_model(retime(base, pc, host), k)
                    if trace_lines(t) != ref_det: bad.append((pc, host, k, 'det'))
                except NixieError as e: bad.append((pc, host, k, 'DL'))
        print(f.split('/')[-1], 'OK' if not bad else bad[:6], flush=True)
else:
    lo, hi = int(sys.argv[2]), int(sys.argv[3]); robust = 0; bad = []
    for seed in range(lo, hi):
        base = random_scenario(seed)
        outs = []
        for pc, host in SPEEDS:
            p = subprocess.run(['oracle/_ref/ref_trace', '-'], input=retime(base, pc, host), capture_output=True, text=True)
            outs.append(p.returncode == 0)
        if not all(outs): continue
        robust += 1
        for k in (2, 8, 64):
            for pc, host in SPEEDS[:4]:
                try: run_scenario_model(retime(base, pc, host), k)
                except NixieError: bad.append((seed, k, pc, host))
    print('robust', robust, 'bad', len(bad), bad[:10])
