"""Python mirror of the swap-path interface (reference proj/include/nixie/*.hpp)
over the C ABI. Method names follow the reference: allocate / free_chunk
(MemState, mem_model.cpp:48-116), plan_switch (planner.cpp:111-216),
switch_to = plan_switch + execute (transfer.cpp:250-271), audit
(mem_model.cpp:274-325), and the launch gate / MLFQ grant (mlfq.cpp:132-201).
Errors raise NixieError carrying the reference Err name.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field, fields
from typing import Dict, List, Optional, Sequence, Tuple

from . import _lib as L
from ._lib import NixieError, byref, c_int, c_size_t, c_uint32, c_uint64, c_uint8, c_void_p, check, lib

KIB, MIB, GIB = 1 << 10, 1 << 20, 1 << 30
BLOCK_BYTES = 2 * MIB
SCENARIO_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scenarios")


@dataclass
class EngineConfig:
    """include/nixie/swap_engine.hpp EngineConfig."""
    device: int = 0
    gpu_capacity: int = 32 * GIB
    pinned_capacity: int = 16 * GIB
    paged_capacity: int = 96 * GIB
    path: int = L.PATH_AUTO
    pcie_legs_in_flight: int = 1024
    legs_per_launch: int = 128
    host_threads: int = 0  # 0: measured at construction (calibrate_host)
    host_legs_in_flight: int = 64
    max_ctas: int = 0
    fused_launch: bool = False
    verify: bool = True
    numa_bind: bool = True
    first_batch_legs: int = 8
    k3_tma: bool = True
    k3_one_stream: bool = True
    k3_grouped: bool = True
    k3_verify_group: int = 4096
    d2h_commit_legs: int = 32
    early_frame_release: bool = True
    pace_lag_legs: int = 64
    fetch_first_pump: bool = True
    host_streaming_copy: bool = True

    def to_c(self) -> L.EngineConfigC:
        c = L.EngineConfigC()
        for f in fields(self):
            setattr(c, f.name, int(getattr(self, f.name)))
        return c


@dataclass
class PlannerConfig:
    """reference PlannerConfig (planner.hpp:39-43)."""
    streaming_window: int = 512 * MIB
    pinned_budget: int = L.UNBOUNDED
    victim_order: List[int] = field(default_factory=list)

    def to_c(self) -> Tuple[L.PlannerConfigC, object]:
        arr = (c_uint32 * max(1, len(self.victim_order)))(*self.victim_order)
        c = L.PlannerConfigC(self.streaming_window, self.pinned_budget,
                             ctypes.cast(arr, ctypes.POINTER(c_uint32)) if self.victim_order else None,
                             len(self.victim_order))
        return c, arr  # keep `arr` alive for the call


class SwapEngine:
    """One per-GPU Nixie instance (device arena, pinned staging ring, paged
    store, host copy pool, two PCIe lane streams)."""

    def __init__(self, config: Optional[EngineConfig] = None, **overrides):
        cfg = config or EngineConfig()
        for k, v in overrides.items():
            if not hasattr(cfg, k):
                raise TypeError(f"unknown engine option {k}")
            setattr(cfg, k, v)
        self.config = cfg
        h = c_void_p()
        check(lib.nx_engine_create(byref(cfg.to_c()), byref(h)))
        self._h = h

    # -- lifecycle --
    def close(self) -> None:
        if self._h:
            lib.nx_engine_destroy(self._h)
            self._h = c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- registry --
    def allocate(self, app: int, size: int, tier: int = L.TIER_GPU) -> List[int]:
        cap = (size + 128 * MIB - 1) // (128 * MIB) + 1
        out = (c_uint64 * cap)()
        n = c_size_t()
        check(lib.nx_alloc(self._h, app, size, tier, out, cap, byref(n)))
        return list(out[: n.value])

    def free_chunk(self, app: int, chunk: int) -> int:
        r = c_uint64()
        check(lib.nx_free_chunk(self._h, app, chunk, byref(r)))
        return r.value

    def audit(self) -> None:
        check(lib.nx_audit(self._h))

    def app_bytes_resident(self, app: int) -> List[int]:
        out = (c_uint64 * 4)()
        check(lib.nx_app_resident(self._h, app, out))
        return list(out)

    def pinned_physical(self) -> Tuple[int, int]:
        now, peak = c_uint64(), c_uint64()
        check(lib.nx_pinned_physical(self._h, byref(now), byref(peak)))
        return now.value, peak.value

    def pinned_overhead(self) -> int:
        """Pinned bytes outside the budgeted ring (bounce buffer, table stages)."""
        v = c_uint64()
        check(lib.nx_pinned_overhead(self._h, byref(v)))
        return v.value

    def app_blocks(self, app: int) -> List[int]:
        n = c_size_t()
        check(lib.nx_app_blocks(self._h, app, None, 0, byref(n)))
        out = (c_uint64 * max(1, n.value))()
        check(lib.nx_app_blocks(self._h, app, out, n.value, byref(n)))
        return list(out[: n.value])

    # -- K4 synthetic working set --
    def fill_pattern(self, app: int, seed: int) -> None:
        check(lib.nx_fill_pattern(self._h, app, seed))

    def verify_pattern(self, app: int, seed: int) -> int:
        bad = c_uint64()
        check(lib.nx_verify_pattern(self._h, app, seed, byref(bad)))
        return bad.value

    def read_block(self, block: int) -> bytes:
        buf = ctypes.create_string_buffer(BLOCK_BYTES)
        check(lib.nx_block_read(self._h, block, buf))
        return buf.raw

    def poke_block(self, block: int, offset: int, value: int) -> None:
        check(lib.nx_block_poke(self._h, block, offset, value))

    def block_checksum(self, block: int) -> int:
        v = c_uint64()
        check(lib.nx_block_checksum(self._h, block, byref(v)))
        return v.value

    def block_frame(self, block: int) -> int:
        p = c_void_p()
        check(lib.nx_block_frame(self._h, block, byref(p)))
        return p.value or 0

    # -- swap-engine interface --
    def plan_switch(self, incoming: int, planner: Optional[PlannerConfig] = None) -> Tuple[str, int, int]:
        pc, keep = (planner or PlannerConfig()).to_c()
        n = c_size_t()
        bi, bo = c_uint64(), c_uint64()
        check(lib.nx_plan(self._h, incoming, byref(pc), None, 0, byref(n), byref(bi), byref(bo)))
        buf = ctypes.create_string_buffer(n.value + 1)
        check(lib.nx_plan(self._h, incoming, byref(pc), buf, n.value + 1, byref(n), byref(bi), byref(bo)))
        del keep
        return buf.value.decode(), bi.value, bo.value

    def switch_to(self, incoming: int, planner: Optional[PlannerConfig] = None, drain_stream: int = 0) -> Dict:
        pc, keep = (planner or PlannerConfig()).to_c()
        st = L.SwitchStatsC()
        check(lib.nx_switch(self._h, incoming, byref(pc), c_void_p(drain_stream or None), byref(st)))
        del keep
        return st.as_dict()

    def prefetch_begin(self, app: int, planner: Optional[PlannerConfig] = None) -> int:
        """Starts plan_prefetch(app) in the background; returns its move count."""
        pc, keep = (planner or PlannerConfig()).to_c()
        n = c_uint64()
        check(lib.nx_prefetch_begin(self._h, app, byref(pc), byref(n)))
        del keep
        return n.value

    def prefetch_pump(self) -> bool:
        a = c_int()
        check(lib.nx_prefetch_pump(self._h, byref(a)))
        return bool(a.value)

    def prefetch_quiesce(self) -> int:
        """cancel_pending + quiesced; returns bytes committed by prefetch so far."""
        b = c_uint64()
        check(lib.nx_prefetch_quiesce(self._h, byref(b)))
        return b.value

    def lane_trace(self, lane: int) -> List[Tuple[int, str, str]]:
        n = c_size_t()
        check(lib.nx_lane_trace(self._h, lane, None, None, None, 0, byref(n)))
        k = max(1, n.value)
        b, s, d = (c_uint64 * k)(), (c_uint8 * k)(), (c_uint8 * k)()
        check(lib.nx_lane_trace(self._h, lane, b, s, d, n.value, byref(n)))
        return [(b[i], L.TIER_NAMES[s[i]], L.TIER_NAMES[d[i]]) for i in range(n.value)]

    def total_launches(self) -> int:
        return int(lib.nx_total_launches(self._h))

    def k3_trace(self) -> List[Tuple[float, float, int, int]]:
        """(start_s, end_s, legs, lane) of the last switch's checksum launches."""
        n = c_size_t()
        check(lib.nx_k3_trace(self._h, None, None, None, None, 0, byref(n)))
        k = max(1, n.value)
        a, z = (ctypes.c_double * k)(), (ctypes.c_double * k)()
        g, l = (c_int * k)(), (c_int * k)()
        check(lib.nx_k3_trace(self._h, a, z, g, l, n.value, byref(n)))
        return [(a[i], z[i], g[i], l[i]) for i in range(n.value)]

    def batch_trace(self) -> List[Dict]:
        """The last switch's PCIe batches (device and host times, s)."""
        n = c_size_t()
        check(lib.nx_batch_trace(self._h, None, 0, byref(n)))
        arr = (L.BatchRecordC * max(1, n.value))()
        check(lib.nx_batch_trace(self._h, arr, n.value, byref(n)))
        keys = ("stream", "legs", "ce", "start_s", "copied_s", "end_s", "host_submit_s", "host_done_s")
        return [{k: getattr(arr[i], k) for k in keys} for i in range(n.value)]

    def leg_records(self) -> List[Dict]:
        """Every leg of the last switch (TransferRecord log): block, src/dst tier,
        start/end (s from the switch start: host times of the leg's start and
        commit; device batch times for PCIe legs on the SM path)."""
        n = c_size_t()
        check(lib.nx_leg_records(self._h, None, 0, byref(n)))
        arr = (L.LegRecordC * max(1, n.value))()
        check(lib.nx_leg_records(self._h, arr, n.value, byref(n)))
        return [{"block": arr[i].block, "src": arr[i].src, "dst": arr[i].dst, "start_s": arr[i].start_s, "end_s": arr[i].end_s}
                for i in range(n.value)]

    def lane_stream(self, lane: int) -> int:
        return lib.nx_lane_stream(self._h, lane) or 0

    # -- host link --
    def probe_pcie(self, bytes_per_direction: int = 1 * GIB, chunk_bytes: int = 64 * MIB) -> Dict:
        p = L.PcieProbeC()
        check(lib.nx_probe_pcie(self._h, bytes_per_direction, chunk_bytes, byref(p)))
        out = {}
        for key in ("h2d", "d2h", "bidir_h2d", "bidir_d2h", "bidir_total"):
            arr = getattr(p, key)
            out[f"ce_{key}"] = arr[0]
            out[f"sm_{key}"] = arr[1]
        out.update(bytes_per_direction=p.bytes_per_direction, chunk_bytes=p.chunk_bytes, numa_node=p.numa_node)
        return out

    def probe_pcie_paced(self, bytes_per_direction: int = 2 * GIB, chunk_bytes: int = 64 * MIB, lag_chunks: int = 2) -> Dict:
        """Both directions on the copy engines, D2H chunk i held until H2D chunk
        i - lag_chunks landed (the engine's paced shape)."""
        g = (ctypes.c_double * 3)()
        check(lib.nx_probe_pcie_paced(self._h, bytes_per_direction, chunk_bytes, lag_chunks, g))
        return {"ce_bidir_h2d": g[0], "ce_bidir_d2h": g[1], "ce_bidir_total": g[2], "bytes_per_direction": bytes_per_direction,
                "chunk_bytes": chunk_bytes, "lag_chunks": lag_chunks}

    def calibrate(self, bytes_per_direction: int = 256 * MIB) -> Dict:
        """Measure SM kernel vs copy engines per batch size (1..128 legs) with
        both directions running; installs the faster per size (path=AUTO)."""
        sm, ce, pick = (ctypes.c_double * 8)(), (ctypes.c_double * 8)(), (c_int * 8)()
        check(lib.nx_calibrate(self._h, bytes_per_direction, sm, ce, pick))
        return {"legs": [1 << k for k in range(8)], "sm_gbps": list(sm), "ce_gbps": list(ce),
                "sm_faster": [bool(x) for x in pick]}

    def calibrate_host(self, bytes_per_direction: int = 1024 * MIB) -> Dict:
        """Size the host copy pool (two-hop pinned<->paged lanes) from a
        measurement; returns GB/s per worker count and the installed count."""
        th, gb, n, ch = (c_int * 16)(), (ctypes.c_double * 16)(), ctypes.c_size_t(), c_int()
        check(lib.nx_calibrate_host(self._h, bytes_per_direction, th, gb, 16, ctypes.byref(n), ctypes.byref(ch)))
        return {"threads": list(th)[:n.value], "gbps": list(gb)[:n.value], "chosen": ch.value,
                "peak_gbs": max(list(gb)[:n.value], default=0.0)}

    def set_option(self, name: str, value: int) -> None:
        """Per-switch tunable between switches (SwapEngine::set_option)."""
        check(lib.nx_engine_set_option(self._h, name.encode(), int(value)))

    def host_threads(self) -> int:
        v = c_int()
        check(lib.nx_host_threads(self._h, ctypes.byref(v)))
        return v.value

    def set_auto_table(self, sm_faster: Sequence[bool]) -> None:
        arr = (c_int * max(1, len(sm_faster)))(*[int(bool(x)) for x in sm_faster])
        check(lib.nx_set_auto_table(self._h, arr, len(sm_faster)))


class LaunchGate:
    """MLFQ scheduler + kernel-launch gate over one engine."""

    def __init__(self, engine: SwapEngine, planner: Optional[PlannerConfig] = None):
        self.engine = engine
        m = L.MlfqConfigC()
        lib.nx_mlfq_config_default(byref(m))
        pc, keep = (planner or PlannerConfig()).to_c()
        h = c_void_p()
        check(lib.nx_gate_create(engine._h, byref(m), byref(pc), byref(h)))
        del keep
        self._h = h

    def close(self):
        if self._h:
            lib.nx_gate_destroy(self._h)
            self._h = c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def attach(self, app: int, stream: int, now: float = 0.0) -> None:
        check(lib.nx_gate_attach(self._h, app, c_void_p(stream or None), now))

    def before_launch(self, app: int, now: float, timeout_s: float = 120.0) -> bool:
        """True: the app may launch now. False: it was held until its swap-in
        was submitted and its stream now waits on the device for it to land.
        Blocks the calling thread (ctypes releases the GIL). Returns holding
        the app's launch lock: call after_launch(app) once the kernel is
        enqueued (or use `with gate.launching(app, now):`)."""
        ok = c_int()
        check(lib.nx_gate_before_launch(self._h, app, now, timeout_s, byref(ok)))
        return bool(ok.value)

    def after_launch(self, app: int) -> None:
        check(lib.nx_gate_after_launch(self._h, app))

    def launching(self, app: int, now: float, timeout_s: float = 120.0):
        gate = self

        class _Launch:
            def __enter__(self_):
                self_.passed = gate.before_launch(app, now, timeout_s)
                return self_

            def __exit__(self_, *exc):
                gate.after_launch(app)

        return _Launch()

    def api_event(self, app: int, now: float, kind: int) -> None:
        """0 NonBlockingReturn, 1 BlockingEnter, 2 BlockingExit (mlfq.cpp:71-85)."""
        check(lib.nx_gate_api_event(self._h, app, now, kind))

    def tick(self, now: float) -> Optional[int]:
        a = c_uint32()
        check(lib.nx_gate_tick(self._h, now, byref(a)))
        return None if a.value == 0xFFFFFFFF else a.value

    def switches(self) -> int:
        return int(lib.nx_gate_switches(self._h))

    def set_prefetch(self, on: bool) -> None:
        """MLFQ prefetch of the next candidate's pageable blocks."""
        check(lib.nx_gate_set_prefetch(self._h, 1 if on else 0))

    def prefetched_bytes(self) -> int:
        return int(lib.nx_gate_prefetched_bytes(self._h))

    def select_next(self, now: float) -> Optional[int]:
        a = c_uint32()
        check(lib.nx_gate_select_next(self._h, now, byref(a)))
        return None if a.value == 0xFFFFFFFF else a.value

    def context_switch(self, to: int, now: float) -> Dict:
        st = L.SwitchStatsC()
        check(lib.nx_gate_switch(self._h, to, now, byref(st)))
        return st.as_dict()

    def granted(self) -> Optional[int]:
        a = c_uint32()
        check(lib.nx_gate_granted(self._h, byref(a)))
        return None if a.value == 0xFFFFFFFF else a.value

    def app_checksum_async(self, app: int, stream: int, out_pinned: int) -> None:
        check(lib.nx_gate_app_checksum_async(self._h, app, c_void_p(stream or None),
                                             ctypes.cast(c_void_p(out_pinned), ctypes.POINTER(c_uint64))))


def run_scenario_model(spec: str, legs_per_lane: int = 1) -> str:
    """Scenario on the virtual clock (no GPU): the trace the reference would print."""
    p, n = c_void_p(), c_size_t()
    if legs_per_lane == 1:
        check(lib.nx_scenario_model(spec.encode(), byref(p), byref(n)))
    else:
        check(lib.nx_scenario_model_lanes(spec.encode(), legs_per_lane, byref(p), byref(n)))
    return L.take_string(p, n)


def run_scenario_real(spec: str, seed: int = 0x4E495849, config: Optional[EngineConfig] = None, **overrides) -> str:
    """Scenario through the CUDA engine: real copies, byte checks (V/F lines)."""
    cfg = config or EngineConfig()
    for k, v in overrides.items():
        setattr(cfg, k, v)
    p, n = c_void_p(), c_size_t()
    check(lib.nx_scenario_real(spec.encode(), byref(cfg.to_c()), seed, byref(p), byref(n)))
    return L.take_string(p, n)


def run_workload_model(spec: str) -> str:
    """MLFQ-driven workload on the virtual clock (no GPU); its reference twin is
    oracle/_ref/ref_workload (same engine over the reference library)."""
    p, n = c_void_p(), c_size_t()
    check(lib.nx_workload_model(spec.encode(), byref(p), byref(n)))
    return L.take_string(p, n)


def run_workload_real(spec: str, seed: int = 0x4E495849, config: Optional[EngineConfig] = None, **overrides) -> str:
    """The same workload with every switch's bytes moved by the CUDA engine
    (M/V/F lines: placement vs the model, byte checks)."""
    cfg = config or EngineConfig()
    for k, v in overrides.items():
        setattr(cfg, k, v)
    p, n = c_void_p(), c_size_t()
    check(lib.nx_workload_real(spec.encode(), byref(cfg.to_c()), seed, byref(p), byref(n)))
    return L.take_string(p, n)


def parse_path(name: str) -> int:
    """'auto' | 'sm' | 'ce' -> PATH_* constant."""
    return {"auto": L.PATH_AUTO, "sm": L.PATH_SM, "ce": L.PATH_CE}[name]


def load_scenario(name: str) -> str:
    path = name if os.path.sep in name else os.path.join(SCENARIO_DIR, name if name.endswith(".scn") else name + ".scn")
    with open(path) as f:
        return f.read()


def pinned_buffer(nbytes: int) -> int:
    p = c_void_p()
    check(lib.nx_pinned_alloc(nbytes, byref(p)))
    return p.value


def free_pinned(ptr: int) -> None:
    lib.nx_pinned_free(c_void_p(ptr))


def stream_sync(stream: int) -> None:
    check(lib.nx_stream_sync(c_void_p(stream or None)))


def stream_create() -> int:
    s = c_void_p()
    check(lib.nx_stream_create(byref(s)))
    return s.value


def stream_destroy(stream: int) -> None:
    lib.nx_stream_destroy(c_void_p(stream))


def launch_busy_kernel(stream: int, ns: int) -> None:
    """Synthetic application kernel: one warp busy for ~ns on `stream`."""
    check(lib.nx_launch_busy_kernel(c_void_p(stream or None), ns))


def stream_done(stream: int) -> bool:
    d = c_int()
    check(lib.nx_stream_query(c_void_p(stream), byref(d)))
    return bool(d.value)


DETERMINISTIC_TAGS = ("S", "P", "L", "R", "B", "E")


def trace_lines(trace: str, tags: Sequence[str] = DETERMINISTIC_TAGS) -> List[str]:
    """Lines of a scenario trace whose first token is in `tags`."""
    return [ln for ln in trace.splitlines() if ln.split(" ", 1)[0] in tags]
