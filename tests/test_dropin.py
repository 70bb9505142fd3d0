"""Header-level drop-in proof: the reference's own unit tests
(proj/tests/test_{mem_model,planner,transfer,mlfq}.cpp; UvmSim is out of
scope) compiled against include/nixie/*.hpp and linked with this repo's host
library, not the reference's, pass unmodified."""
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
    assert "test cases: 30 | 0 failed" in p.stdout and "failures: 0" in p.stdout, p.stdout
