"""MLFQ-driven workloads (config 3 and seeded random ones) on the virtual
clock: the product's trace equals the reference's, byte for byte.

The workload engine (include/nixie_workload/workload_sim.hpp) is written
against the `nixie` namespace API alone; the product instantiates it over
this library (nx_workload_model) and the oracle over the UNMODIFIED reference
library and headers (oracle/_ref/ref_workload). A difference in any
scheduler decision (enqueue/grant/yield/demote/promote and its timing), plan,
per-lane leg order, placement or request latency shows up in the trace."""
import hashlib
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from paper_2601_11743_b200 import NixieError, run_workload_model  # noqa: E402
from workload_gen import random_workload  # noqa: E402

REF = os.path.join(ROOT, "oracle", "_ref", "ref_workload")
WL_DIR = os.path.join(ROOT, "paper_2601_11743_b200", "workloads")
GOLDEN = os.path.join(ROOT, "tests", "golden", "workloads.json")
C3 = sorted(f for f in os.listdir(WL_DIR) if f.endswith(".wl"))


def ref(spec):
    p = subprocess.run([REF, "-"], input=spec, capture_output=True, text=True, timeout=300)
    if p.returncode:
        return None, p.stderr.strip().removeprefix("ref_workload: ").split(":", 1)[0]
    return p.stdout, None


def ours(spec):
    try:
        return run_workload_model(spec), None
    except NixieError as e:
        return None, e.kind


def sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


@pytest.mark.parametrize("name", C3)
def test_config3_matches_golden_reference_trace(name):
    """Against the committed reference trace hash (no reference needed)."""
    gold = json.load(open(GOLDEN))["c3"][name]
    trace, err = ours(open(os.path.join(WL_DIR, name)).read())
    assert err is None
    assert sha(trace) == gold["sha256"]
    assert [ln for ln in trace.splitlines() if ln[0] in "XSQ"][:400] == gold["summary"][:400]


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref/ref_workload not built")
@pytest.mark.parametrize("name", C3)
def test_config3_matches_live_reference(name):
    spec = open(os.path.join(WL_DIR, name)).read()
    r, rerr = ref(spec)
    o, oerr = ours(spec)
    assert rerr is None and oerr is None
    assert o == r


def test_random_workloads_match_golden():
    gold = json.load(open(GOLDEN))["random"]
    assert len(gold) >= 60
    for seed, g in gold.items():
        spec = random_workload(int(seed))
        assert sha(spec) == g["spec_sha256"], "generator changed; regenerate tests/golden"
        o, err = ours(spec)
        if g["error"]:
            assert err == g["error"], (seed, err)
        else:
            assert err is None, (seed, err)
            assert sha(o) == g["sha256"], seed


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref/ref_workload not built")
def test_random_workloads_match_live_reference():
    for seed in range(1000, 1040):
        spec = random_workload(seed)
        r, rerr = ref(spec)
        o, oerr = ours(spec)
        assert (rerr, r) == (oerr, o), seed


def test_workload_properties():
    """determinism, grant exclusivity, every app served."""
    spec = open(os.path.join(WL_DIR, "c3_mlfq_mix_3s.wl")).read()
    a, b = run_workload_model(spec), run_workload_model(spec)
    assert a == b
    xs = [ln.split() for ln in a.splitlines() if ln.startswith("X ")]
    assert len(xs) >= 5
    # switches are sequential: each starts after the previous completion
    for prev, cur in zip(xs, xs[1:]):
        assert float(cur[2]) >= float(prev[4])
        assert float(cur[3]) >= float(cur[2]) and float(cur[4]) >= float(cur[3])
    served = {ln.split()[1] for ln in a.splitlines() if ln.startswith("Q ")}
    assert {"0", "1"} <= served
    grants = [ln.split() for ln in a.splitlines() if ln.startswith("E ") and ln.split()[2] == "grant"]
    assert {g[1] for g in grants} == {"0", "1", "2"}


def test_prefetch_shortens_switches():
    """with prefetch the same config-3 workload spends less
    time in context switches (fetches of the next app come from pinned)."""
    base = run_workload_model(open(os.path.join(WL_DIR, "c3_mlfq_mix_3s.wl")).read())
    pf = run_workload_model(open(os.path.join(WL_DIR, "c3_mlfq_mix_3s_prefetch.wl")).read())

    def switch_time(tr):
        return sum(float(x.split()[4]) - float(x.split()[2]) for x in tr.splitlines() if x.startswith("X "))

    assert any(ln.startswith("H ") for ln in pf.splitlines())
    assert not any(ln.startswith("H ") for ln in base.splitlines())
    assert switch_time(pf) < switch_time(base)


def test_workload_parse_errors():
    with pytest.raises(NixieError) as e:
        run_workload_model("capacity gpu 1GiB\nbogus\n")
    assert e.value.kind == "ParseError"
    with pytest.raises(NixieError) as e:
        run_workload_model("capacity gpu 64MiB\ninteractive 0 128MiB paged 0 1 1 0.01 0\n")
    assert e.value.kind == "ValidationError"
