"""ctypes binding of the C ABI in include/nixie_b200.h.

The shared library is built in-tree (``make -C paper_2601_11743_b200`` or
``__graft_entry__.build()``) at ``paper_2601_11743_b200/lib/libnixie_b200.so``.
There is no fallback: if the library is missing, importing this module
raises, and every engine call goes through the CUDA code in that library.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, byref, c_char, c_char_p, c_double, c_int, c_size_t, c_uint8, c_uint32,
                    c_uint64, c_void_p)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libnixie_b200.so")

NX_OK = 0
NX_E_INVARIANT = 100
NX_E_CUDA = 200
NX_E_ARG = 300

ERR_NAMES = [
    "CapacityExceeded", "UnknownChunk", "UnknownApp", "ChunkBusy", "NotInFlight", "AppTooLarge",
    "InsufficientEvictable", "InvalidScenario", "ParseError", "ValidationError", "IoError", "InvalidState",
]

TIER_GPU, TIER_PINNED, TIER_PAGED, TIER_DISK = 0, 1, 2, 3
TIER_NAMES = ["gpu", "pinned", "paged", "disk"]
PATH_AUTO, PATH_SM, PATH_CE = 0, 1, 2
UNBOUNDED = (1 << 64) - 1


class NixieError(RuntimeError):
    """A non-zero status from the C ABI. `kind` is the reference Err name,
    'InvariantViolation', 'CudaError' or 'BadArgument'."""

    def __init__(self, code: int, message: str):
        if 1 <= code <= len(ERR_NAMES):
            kind = ERR_NAMES[code - 1]
        elif code == NX_E_INVARIANT:
            kind = "InvariantViolation"
        elif code == NX_E_CUDA:
            kind = "CudaError"
        else:
            kind = "BadArgument"
        super().__init__(f"[{kind}] {message}")
        self.code = code
        self.kind = kind


class EngineConfigC(Structure):
    _fields_ = [
        ("device", c_int), ("gpu_capacity", c_uint64), ("pinned_capacity", c_uint64), ("paged_capacity", c_uint64),
        ("path", c_int), ("pcie_legs_in_flight", c_int), ("legs_per_launch", c_int), ("host_threads", c_int),
        ("host_legs_in_flight", c_int), ("max_ctas", c_int), ("fused_launch", c_int), ("verify", c_int),
        ("numa_bind", c_int), ("first_batch_legs", c_int), ("k3_tma", c_int), ("k3_one_stream", c_int),
        ("k3_grouped", c_int), ("k3_verify_group", c_int), ("d2h_commit_legs", c_int), ("early_frame_release", c_int),
        ("pace_lag_legs", c_int), ("fetch_first_pump", c_int), ("host_streaming_copy", c_int),
    ]


class PlannerConfigC(Structure):
    _fields_ = [("streaming_window", c_uint64), ("pinned_budget", c_uint64), ("victim_order", POINTER(c_uint32)),
                ("n_victims", c_size_t)]


class SwitchStatsC(Structure):
    _fields_ = [
        ("bytes_in", c_uint64), ("bytes_out", c_uint64), ("pcie_h2d_bytes", c_uint64), ("pcie_d2h_bytes", c_uint64),
        ("host_bytes", c_uint64), ("wall_s", c_double), ("plan_s", c_double), ("device_span_s", c_double),
        ("kernel_s_h2d", c_double), ("kernel_s_d2h", c_double), ("launches_h2d", c_int), ("launches_d2h", c_int),
        ("ce_batches_h2d", c_int), ("ce_batches_d2h", c_int), ("host_legs", c_int), ("verified", c_uint64),
        ("unverified", c_uint64), ("mismatches", c_uint64), ("tp_to_gpu", c_double), ("tp_from_gpu", c_double),
        ("tp_bidir", c_double), ("k1_s", c_double), ("k3_s", c_double), ("k1_bytes", c_uint64), ("k3_bytes", c_uint64),
        ("k1_launches", c_int), ("k3_launches", c_int), ("k3_busy_s", c_double), ("k3_kernel_s", c_double),
        ("ce_calls", c_int), ("pace_waits", c_int), ("ce_calls_dir", c_int * 2), ("run_breaks_src", c_int * 2),
        ("run_breaks_dst", c_int * 2),
    ]

    def as_dict(self) -> dict:
        return {name: (list(getattr(self, name)) if name in ("ce_calls_dir", "run_breaks_src", "run_breaks_dst")
                       else getattr(self, name)) for name, _ in self._fields_}



class PcieProbeC(Structure):
    _fields_ = [("h2d", c_double * 2), ("d2h", c_double * 2), ("bidir_h2d", c_double * 2), ("bidir_d2h", c_double * 2),
                ("bidir_total", c_double * 2), ("bytes_per_direction", c_uint64), ("chunk_bytes", c_uint64),
                ("numa_node", c_int)]


class BatchRecordC(Structure):
    _fields_ = [("stream", c_int), ("legs", c_int), ("ce", c_int), ("pad", c_int), ("start_s", c_double),
                ("copied_s", c_double), ("end_s", c_double), ("host_submit_s", c_double), ("host_done_s", c_double)]


class LegRecordC(Structure):
    _fields_ = [("block", c_uint64), ("src", c_uint8), ("dst", c_uint8), ("pad", c_uint8 * 6), ("start_s", c_double),
                ("end_s", c_double)]


class DeviceInfoC(Structure):
    _fields_ = [("pci_bus_id", c_char * 32), ("numa_node", c_int), ("node_from_cpus", c_int), ("n_cpus", c_int),
                ("cpulist", c_char * 256)]


class MlfqConfigC(Structure):
    _fields_ = [("levels", c_int), ("base_allotment", c_double), ("base_preemption", c_double),
                ("idle_threshold", c_double), ("tick", c_double)]


# (name, restype, argtypes) for every symbol of include/nixie_b200.h.
_SIGNATURES = [
    ("nx_last_error", c_char_p, []),
    ("nx_version", c_char_p, []),
    ("nx_cuda_device_count", c_int, [POINTER(c_int)]),
    ("nx_device_info_get", c_int, [c_int, POINTER(DeviceInfoC)]),
    ("nx_engine_config_default", None, [POINTER(EngineConfigC)]),
    ("nx_planner_config_default", None, [POINTER(PlannerConfigC)]),
    ("nx_engine_create", c_int, [POINTER(EngineConfigC), POINTER(c_void_p)]),
    ("nx_engine_destroy", None, [c_void_p]),
    ("nx_alloc", c_int, [c_void_p, c_uint32, c_uint64, c_int, POINTER(c_uint64), c_size_t, POINTER(c_size_t)]),
    ("nx_free_chunk", c_int, [c_void_p, c_uint32, c_uint64, POINTER(c_uint64)]),
    ("nx_audit", c_int, [c_void_p]),
    ("nx_app_resident", c_int, [c_void_p, c_uint32, POINTER(c_uint64)]),
    ("nx_pinned_physical", c_int, [c_void_p, POINTER(c_uint64), POINTER(c_uint64)]),
    ("nx_pinned_overhead", c_int, [c_void_p, POINTER(c_uint64)]),
    ("nx_fill_pattern", c_int, [c_void_p, c_uint32, c_uint64]),
    ("nx_verify_pattern", c_int, [c_void_p, c_uint32, c_uint64, POINTER(c_uint64)]),
    ("nx_block_frame", c_int, [c_void_p, c_uint64, POINTER(c_void_p)]),
    ("nx_block_checksum", c_int, [c_void_p, c_uint64, POINTER(c_uint64)]),
    ("nx_app_blocks", c_int, [c_void_p, c_uint32, POINTER(c_uint64), c_size_t, POINTER(c_size_t)]),
    ("nx_block_read", c_int, [c_void_p, c_uint64, c_void_p]),
    ("nx_block_poke", c_int, [c_void_p, c_uint64, c_uint64, c_uint8]),
    ("nx_plan", c_int, [c_void_p, c_uint32, POINTER(PlannerConfigC), POINTER(c_char), c_size_t, POINTER(c_size_t),
                        POINTER(c_uint64), POINTER(c_uint64)]),
    ("nx_switch", c_int, [c_void_p, c_uint32, POINTER(PlannerConfigC), c_void_p, POINTER(SwitchStatsC)]),
    ("nx_prefetch_begin", c_int, [c_void_p, c_uint32, POINTER(PlannerConfigC), POINTER(c_uint64)]),
    ("nx_prefetch_pump", c_int, [c_void_p, POINTER(c_int)]),
    ("nx_prefetch_quiesce", c_int, [c_void_p, POINTER(c_uint64)]),
    ("nx_lane_trace", c_int, [c_void_p, c_int, POINTER(c_uint64), POINTER(c_uint8), POINTER(c_uint8), c_size_t,
                              POINTER(c_size_t)]),
    ("nx_total_launches", c_uint64, [c_void_p]),
    ("nx_k3_trace", c_int, [c_void_p, POINTER(c_double), POINTER(c_double), POINTER(c_int), POINTER(c_int), c_size_t,
                            POINTER(c_size_t)]),
    ("nx_batch_trace", c_int, [c_void_p, POINTER(BatchRecordC), c_size_t, POINTER(c_size_t)]),
    ("nx_leg_records", c_int, [c_void_p, POINTER(LegRecordC), c_size_t, POINTER(c_size_t)]),
    ("nx_lane_stream", c_void_p, [c_void_p, c_int]),
    ("nx_probe_pcie", c_int, [c_void_p, c_uint64, c_uint64, POINTER(PcieProbeC)]),
    ("nx_probe_pcie_paced", c_int, [c_void_p, c_uint64, c_uint64, c_int, POINTER(c_double)]),
    ("nx_probe_copy_variant", c_int, [c_void_p, c_int, c_uint64, c_int, POINTER(c_double)]),
    ("nx_set_auto_table", c_int, [c_void_p, POINTER(c_int), c_size_t]),
    ("nx_calibrate", c_int, [c_void_p, c_uint64, POINTER(c_double), POINTER(c_double), POINTER(c_int)]),
    ("nx_calibrate_host", c_int, [c_void_p, c_uint64, POINTER(c_int), POINTER(c_double), c_size_t, POINTER(c_size_t),
                                  POINTER(c_int)]),
    ("nx_host_threads", c_int, [c_void_p, POINTER(c_int)]),
    ("nx_engine_set_option", c_int, [c_void_p, c_char_p, c_int]),
    ("nx_probe_checksum_launch", c_int, [c_void_p, POINTER(c_double)]),
    ("nx_probe_checksum_launch_ex", c_int, [c_void_p, c_int, POINTER(c_double)]),
    ("nx_mlfq_config_default", None, [POINTER(MlfqConfigC)]),
    ("nx_gate_create", c_int, [c_void_p, POINTER(MlfqConfigC), POINTER(PlannerConfigC), POINTER(c_void_p)]),
    ("nx_gate_destroy", None, [c_void_p]),
    ("nx_gate_attach", c_int, [c_void_p, c_uint32, c_void_p, c_double]),
    ("nx_gate_before_launch", c_int, [c_void_p, c_uint32, c_double, c_double, POINTER(c_int)]),
    ("nx_gate_after_launch", c_int, [c_void_p, c_uint32]),
    ("nx_gate_api_event", c_int, [c_void_p, c_uint32, c_double, c_int]),
    ("nx_gate_tick", c_int, [c_void_p, c_double, POINTER(c_uint32)]),
    ("nx_gate_switches", c_uint64, [c_void_p]),
    ("nx_gate_set_prefetch", c_int, [c_void_p, c_int]),
    ("nx_gate_prefetched_bytes", c_uint64, [c_void_p]),
    ("nx_launch_busy_kernel", c_int, [c_void_p, c_uint64]),
    ("nx_gate_select_next", c_int, [c_void_p, c_double, POINTER(c_uint32)]),
    ("nx_gate_switch", c_int, [c_void_p, c_uint32, c_double, POINTER(SwitchStatsC)]),
    ("nx_gate_granted", c_int, [c_void_p, POINTER(c_uint32)]),
    ("nx_gate_app_checksum_async", c_int, [c_void_p, c_uint32, c_void_p, POINTER(c_uint64)]),
    ("nx_stream_sync", c_int, [c_void_p]),
    ("nx_stream_create", c_int, [POINTER(c_void_p)]),
    ("nx_stream_destroy", None, [c_void_p]),
    ("nx_stream_query", c_int, [c_void_p, POINTER(c_int)]),
    ("nx_pinned_alloc", c_int, [c_size_t, POINTER(c_void_p)]),
    ("nx_pinned_free", None, [c_void_p]),
    ("nx_scenario_model", c_int, [c_char_p, POINTER(c_void_p), POINTER(c_size_t)]),
    ("nx_scenario_model_lanes", c_int, [c_char_p, c_int, POINTER(c_void_p), POINTER(c_size_t)]),
    ("nx_scenario_real", c_int, [c_char_p, POINTER(EngineConfigC), c_uint64, POINTER(c_void_p), POINTER(c_size_t)]),
    ("nx_workload_model", c_int, [c_char_p, POINTER(c_void_p), POINTER(c_size_t)]),
    ("nx_workload_real", c_int, [c_char_p, POINTER(EngineConfigC), c_uint64, POINTER(c_void_p), POINTER(c_size_t)]),
    ("nx_uvm_create", c_int, [c_uint64, c_double, c_double, c_int, c_double, c_int, POINTER(c_void_p)]),
    ("nx_uvm_register", c_int, [c_void_p, c_uint32, c_uint64]),
    ("nx_uvm_touch", c_int, [c_void_p, c_uint32, c_double, c_double, POINTER(c_double)]),
    ("nx_uvm_stats", c_int, [c_void_p, POINTER(c_uint64), POINTER(c_uint64), POINTER(c_uint64)]),
    ("nx_uvm_destroy", None, [c_void_p]),
    ("nx_free", None, [c_void_p]),
]

EXPORTED = [name for name, _, _ in _SIGNATURES]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2601_11743_b200` or "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, restype, argtypes in _SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    return lib


lib = _load()


def check(code: int) -> None:
    if code != NX_OK:
        raise NixieError(code, lib.nx_last_error().decode(errors="replace"))


def take_string(ptr: c_void_p, length: c_size_t) -> str:
    try:
        return ctypes.string_at(ptr.value, length.value).decode()
    finally:
        lib.nx_free(ptr)


def cuda_device_count() -> int:
    n = c_int(0)
    check(lib.nx_cuda_device_count(byref(n)))
    return n.value


def device_info(device: int) -> dict:
    """PCI bus id, NUMA node and local CPUs of a CUDA device (nx_device_info_get)."""
    d = DeviceInfoC()
    check(lib.nx_device_info_get(device, byref(d)))
    return {"pci_bus_id": d.pci_bus_id.decode(), "numa_node": d.numa_node, "numa_from_cpulist": bool(d.node_from_cpus),
            "n_cpus": d.n_cpus, "cpulist": d.cpulist.decode()}


__all__ = [
    "lib", "check", "take_string", "NixieError", "EngineConfigC", "PlannerConfigC", "SwitchStatsC", "PcieProbeC",
    "MlfqConfigC", "EXPORTED", "LIB_PATH", "TIER_GPU", "TIER_PINNED", "TIER_PAGED", "TIER_DISK", "TIER_NAMES",
    "PATH_AUTO", "PATH_SM", "PATH_CE", "UNBOUNDED", "cuda_device_count", "c_uint64", "c_uint32", "c_size_t", "c_int",
    "c_void_p", "c_uint8", "byref",
]
