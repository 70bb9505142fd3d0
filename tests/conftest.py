import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


# Parity gates first, deployment-path tests last: under `pytest -x` a flaky
# interposer test (real processes, wall-clock think times) must never stop
# the run before the engine and full-size parity tests have run.
_FILE_ORDER = ["test_oracle_pinned", "test_dropin", "test_parity_model", "test_parity_workload", "test_abi",
               "test_gpu_engine", "test_gpu_scale", "test_gpu_budget", "test_gpu_workload", "test_gpu_uvm", "test_cli",
               "test_multirank", "test_interposer_host", "test_gpu_daemon_parity", "test_gpu_interposer"]


def pytest_collection_modifyitems(session, config, items):
    def rank(item):
        mod = os.path.splitext(os.path.basename(str(item.fspath)))[0]
        return _FILE_ORDER.index(mod) if mod in _FILE_ORDER else len(_FILE_ORDER)
    items.sort(key=rank)  # stable: file-internal order is kept


@pytest.fixture(scope="session")
def oracle_lib():
    """C restatement of the byte-level functions (oracle/swap_oracle.c)."""
    import ctypes
    path = os.path.join(REF_BIN, "libswap_oracle.so")
    if not os.path.exists(path):
        pytest.skip("oracle/_ref/libswap_oracle.so not built (python -c 'import __graft_entry__ as g; g.build()')")
    lib = ctypes.CDLL(path)
    u64, u32 = ctypes.c_uint64, ctypes.c_uint32
    for name, res, args in [
        ("so_mix64", u64, [u64]), ("so_splitmix64", u64, [u64]), ("so_pattern_word", u64, [u64, u32, u64, u64]),
        ("so_fill_block", None, [ctypes.c_void_p, u64, u32, u64]), ("so_checksum", u64, [ctypes.c_void_p, ctypes.c_size_t]),
        ("so_pattern_block_checksum", u64, [u64, u32, u64]), ("so_compare_block", u64, [ctypes.c_void_p, u64, u32, u64]),
        ("so_copy_blocks", ctypes.c_double, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_int]),
    ]:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


@pytest.fixture(scope="session")
def golden():
    import json
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    with open(os.path.join(here, "scenarios.json")) as f:
        scen = json.load(f)
    with open(os.path.join(here, "random_tiny.json")) as f:
        rnd = json.load(f)
    return {"scenarios": scen, "random": rnd}


@pytest.fixture(scope="session")
def gpu():
    from paper_2601_11743_b200 import cuda_device_count
    if cuda_device_count() < 1:
        pytest.fail("gpu test collected but no CUDA device is visible")
    return True
