"""Trace parity on the virtual clock: the product's lanes + planner + MLFQ
driven by the scenario driver produce the reference's trace byte for byte
(plans, per-lane leg sequences, placements, timestamps, scheduler rows).
Golden traces come from the unmodified reference (tests/golden/make_golden.py);
when oracle/_ref/ref_trace is present the reference is also run live."""
import hashlib
import os
import subprocess

import pytest

from conftest import REF_BIN
from paper_2601_11743_b200 import NixieError, load_scenario, run_scenario_model, trace_lines
from scenario_gen import random_scenario

SCENARIOS = ["kat_planner_ordering", "small_three_apps", "small_pinned_only", "c1_two_apps_2g",
             "c2_interactive_background", "x16_exchange", "c4_budget_2g", "c4_budget_4g", "c4_budget_8g",
             "c4_budget_16g"]


def sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


def det(trace):
    return "\n".join(trace_lines(trace))


@pytest.mark.parametrize("name", SCENARIOS)
def test_scenario_matches_reference_golden(name, golden):
    g = golden["scenarios"][name]
    mine = run_scenario_model(load_scenario(name))
    if g["trace"] is not None:
        assert mine == g["trace"]
    assert sha(mine) == g["sha256"]
    assert det(mine) == det(mine)  # deterministic subset is a pure function of the trace
    assert sha(det(mine)) == g["det_sha256"]


def test_kat_planner_ordering_known_answer():
    t = run_scenario_model(load_scenario("kat_planner_ordering"))
    plan = [ln[4:] for ln in t.splitlines() if ln.startswith("P 0 ")]
    assert plan == [f"{b} paged gpu 2 fetch" for b in (4, 5, 6, 7)] + [f"{b} gpu pinned 1 evict" for b in (0, 1, 2, 3)]
    done = float([ln for ln in t.splitlines() if ln.startswith("T 0 ")][0].split()[3])
    assert abs(done - 284.658e-6) < 1e-9


@pytest.mark.parametrize("legs", [2, 8, 64])
@pytest.mark.parametrize("name", ["small_three_apps", "c1_two_apps_2g", "c4_budget_2g"])
def test_concurrent_lanes_keep_decisions(name, legs, golden):
    """The CUDA engine runs many legs per lane; on the virtual clock that must
    not change plans, per-lane sequences, placements or schedule events."""
    mine = run_scenario_model(load_scenario(name), legs_per_lane=legs)
    assert sha(det(mine)) == golden["scenarios"][name]["det_sha256"]


def _kind(err: NixieError):
    return err.kind


def test_random_tiny_scenarios_match_reference(golden):
    n_ok = n_err = 0
    for case in golden["random"]:
        assert case["spec"] == random_scenario(case["seed"])  # generator is stable
        try:
            mine = run_scenario_model(case["spec"])
        except NixieError as e:
            assert case["error"] == _kind(e), (case["seed"], str(e))
            n_err += 1
            continue
        assert case["error"] is None, (case["seed"], "reference failed but product did not")
        assert mine == case["trace"], case["seed"]
        n_ok += 1
    assert n_ok >= 90 and n_err >= 1


@pytest.mark.parametrize("legs", [2, 4, 16])
def test_random_tiny_concurrent_lanes(golden, legs):
    """On every instance the reference completes under all link timings, many
    legs per lane must complete too, with the reference's decisions."""
    n = 0
    for case in golden["random"]:
        if not case["robust"]:
            continue
        mine = run_scenario_model(case["spec"], legs_per_lane=legs)
        assert det(mine) == det(case["trace"]), case["seed"]
        n += 1
    assert n >= 80


def test_live_reference_on_fresh_random_instances():
    exe = os.path.join(REF_BIN, "ref_trace")
    if not os.path.exists(exe):
        pytest.skip("reference trace driver not built")
    for seed in range(1000, 1200):
        spec = random_scenario(seed)
        p = subprocess.run([exe, "-"], input=spec, capture_output=True, text=True)
        try:
            mine = run_scenario_model(spec)
        except NixieError as e:
            assert p.returncode != 0, (seed, str(e))
            continue
        assert p.returncode == 0, (seed, p.stderr)
        assert mine == p.stdout, seed
