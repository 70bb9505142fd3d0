"""nixie-b200: B200-native context-switch swap path of Nixie (arxiv 2601.11743).

The product is the in-tree shared library lib/libnixie_b200.so (C++ host
library with the reference's API + sm_100a CUDA kernels + C ABI in
include/nixie_b200.h). This package is a thin ctypes mirror of that ABI.
"""
from ._lib import NixieError, cuda_device_count, LIB_PATH  # noqa: F401
from .engine import (EngineConfig, LaunchGate, PlannerConfig, SwapEngine, load_scenario, parse_path,  # noqa: F401
                     run_scenario_model, run_scenario_real, run_workload_model, run_workload_real, trace_lines, GIB, MIB,
                     BLOCK_BYTES)

__version__ = "0.1.0"
