"""Header-level drop-in proof: the reference's own unit tests
(proj/tests/test_{mem_model,planner,transfer,mlfq,uvm}.cpp: every test file)
compiled against include/nixie/*.hpp and linked with this repo's host
library, not the reference's, pass unmodified; and seeded random UvmSim
workloads produce the reference's decision trace line for line."""
import os
import subprocess

import pytest

from conftest import REF_BIN


def test_reference_suite_passes_against_our_library():
    exe = os.path.join(REF_BIN, "dropin_unit_tests")
    if not os.path.exists(exe):
        pytest.skip("drop-in binary not built (needs /root/reference at build time)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-3000:]
    assert "test cases: 35 | 0 failed" in p.stdout and "failures: 0" in p.stdout, p.stdout


def test_uvm_model_matches_reference_on_random_workloads():
    ref = os.path.join(REF_BIN, "uvm_diff_ref")
    ours = os.path.join(REF_BIN, "uvm_diff_ours")
    if not (os.path.exists(ref) and os.path.exists(ours)):
        pytest.skip("uvm_diff binaries not built (make -C oracle all dropin)")
    faults = 0
    for seed in range(1, 41):
        a = subprocess.run([ref, str(seed), "300"], capture_output=True, text=True, timeout=120)
        b = subprocess.run([ours, str(seed), "300"], capture_output=True, text=True, timeout=120)
        assert a.returncode == 0 and b.returncode == 0
        assert a.stdout == b.stdout, seed
        faults += sum(1 for ln in a.stdout.splitlines() if ln.startswith("F "))
    assert faults > 500
