"""Full-size parity on a B200 (BASELINE.json configs 2 and 4 and the 16 GiB
exchange): the real engine's plans, per-lane leg sequences, placements and
schedule events equal the unmodified reference's golden trace, and every
restore is byte-exact (pattern compare of each incoming app after each switch
and of every app at the end)."""
import hashlib

import pytest

from paper_2601_11743_b200 import load_scenario, run_scenario_real, trace_lines

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c2_interactive_background", "c4_budget_2g", "c4_budget_8g", "x16_exchange"])
def test_full_size_real_trace_equals_reference(gpu, golden, name):
    real = run_scenario_real(load_scenario(name), seed=11)
    det = hashlib.sha256("\n".join(trace_lines(real)).encode()).hexdigest()
    assert det == golden["scenarios"][name]["det_sha256"]
    v = [ln.split() for ln in real.splitlines() if ln.startswith("V ")]
    assert v and all(x[3] == "0" and x[7] == "0" for x in v), v  # byte-exact, no unverified restores
    assert all(ln.split()[2] == "0" for ln in real.splitlines() if ln.startswith("F "))
