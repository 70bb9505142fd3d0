"""Golden random instances (tests/golden/random_tiny.json, the robust ones)
through the CUDA engine under several engine shapes; reports every case
whose decisions differ from the reference's or that fails (deadlock).

Usage: python tools/fuzz_real.py [shape indices, e.g. 0,1,2]
       python tools/fuzz_real.py - medium 0:100   (larger random instances vs the model)"""
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
which = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 and sys.argv[1] != "-" else range(len(SHAPES))
medium = len(sys.argv) > 2 and sys.argv[2] == "medium"
cases = [] if medium else [c for c in json.load(open(os.path.join(ROOT, "tests", "golden", "random_tiny.json"))) if c["robust"]]
for si in ([] if medium else which):
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


def medium_scenario(seed: int) -> str:
    """Larger random instances than the golden ones (64-600 blocks per tier),
    so batching, commit groups, pacing and slot contiguity all engage."""
    import random
    r = random.Random(seed)
    blk = 2 << 20
    caps = {"gpu": r.randint(64, 400) * blk, "pinned": r.randint(16, 300) * blk, "paged": r.randint(400, 1200) * blk}
    lines = [f"capacity gpu {caps['gpu']}", f"capacity pinned {caps['pinned']}", f"capacity paged {caps['paged']}",
             "capacity disk 0", f"window {r.choice([4, 16, 64]) * blk}"]
    if r.random() < 0.3:
        lines.append(f"budget {r.randint(16, 300) * blk}")
    used = {"gpu": 0, "pinned": 0, "paged": 0}
    apps = []
    for a in range(r.randint(2, 4)):
        size = r.randint(8, caps["gpu"] // blk) * blk - r.choice([0, 0, 1 << 20])
        fp = -(-size // blk) * blk
        order = ["gpu", "pinned", "paged"]
        r.shuffle(order)
        for t in order:
            if used[t] + fp <= caps[t]:
                used[t] += fp
                lines.append(f"app {a} {size} {t}")
                apps.append(a)
                break
    t, prev = 0.0, None
    for _ in range(r.randint(3, 8)):
        choices = [a for a in apps if a != prev]
        if not choices:
            break
        nxt = r.choice(choices)
        t += r.choice([0.001, 0.5, 3.0])
        lines.append(f"switch {t} {nxt} {r.choice([0.0, 0.01, 1.0])}")
        prev = nxt
    return "\n".join(lines) + "\n"


def reference_deadlocks(spec: str) -> bool:
    import itertools
    from paper_2601_11743_b200 import run_scenario_model
    base = "\n".join(ln for ln in spec.splitlines() if not ln.startswith("link"))
    for up, down, hup, hdown in itertools.product((1, 16, 64), repeat=4):
        try:
            run_scenario_model(f"{base}\nlink 0 {up}GiB/s {down}GiB/s full\nlink 1 {hup}GiB/s {hdown}GiB/s full\n")
        except NixieError as e:
            if "transfer deadlock" in str(e):
                return True
    return False


if __name__ == "__main__" and len(sys.argv) > 2 and sys.argv[2] == "medium":
    from paper_2601_11743_b200 import run_scenario_model
    lo, hi = (int(x) for x in sys.argv[3].split(":"))
    stats = {"ok": 0, "model_error": 0, "ref_deadlock": 0, "bad": []}
    for seed in range(lo, hi):
        spec = medium_scenario(seed)
        try:
            want = run_scenario_model(spec)
        except NixieError:
            stats["model_error"] += 1
            continue
        shape = SHAPES[seed % len(SHAPES)]
        try:
            real = run_scenario_real(spec, seed=7, host_threads=4, **shape)
        except NixieError as e:
            if "transfer deadlock" in str(e) and reference_deadlocks(spec):
                stats["ref_deadlock"] += 1
            else:
                stats["bad"].append((seed, shape, str(e)[:200]))
            continue
        if trace_lines(real) != trace_lines(want):
            stats["bad"].append((seed, shape, "decisions differ"))
        elif any(ln.split()[3] != "0" for ln in real.splitlines() if ln.startswith("V ")):
            stats["bad"].append((seed, shape, "bytes differ"))
        else:
            stats["ok"] += 1
    print(json.dumps(stats), flush=True)
