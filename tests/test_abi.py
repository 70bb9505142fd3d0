"""The C-ABI library loads without a GPU and exports every symbol that
include/nixie_b200.h declares; errors map to the reference's Err taxonomy."""
import os
import re

import pytest

import paper_2601_11743_b200 as nx
from paper_2601_11743_b200 import _lib
from paper_2601_11743_b200._lib import NixieError, lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "nixie_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nx_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported_and_bound():
    syms = declared_symbols()
    assert len(syms) >= 40
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in nixie_b200.h but not exported"
        assert s in _lib.EXPORTED, f"{s} has no ctypes signature"
    assert set(_lib.EXPORTED) == set(syms)


def test_library_is_the_in_tree_build():
    assert nx.LIB_PATH.endswith(os.path.join("paper_2601_11743_b200", "lib", "libnixie_b200.so"))
    assert os.path.exists(nx.LIB_PATH)
    assert b"sm_100a" in lib.nx_version()


def test_parse_error_maps_to_reference_err():
    with pytest.raises(NixieError) as e:
        nx.run_scenario_model("capacity gpu 1GiB\nbogus 1\n")
    assert e.value.kind == "ParseError"
    with pytest.raises(NixieError) as e:
        nx.run_scenario_model("capacity gpu 2MiB\napp 0 4MiB paged\nswitch 0 0 0\n")
    assert e.value.kind == "AppTooLarge"


def test_engine_without_gpu_fails_loudly():
    if nx.cuda_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(NixieError) as e:
        nx.SwapEngine(gpu_capacity=64 << 20, pinned_capacity=64 << 20, paged_capacity=64 << 20)
    assert e.value.kind == "CudaError"


def test_sm100a_kernels_in_library():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", nx.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
