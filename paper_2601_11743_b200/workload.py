"""Real-time workload driver on one B200 (BASELINE.json config 3: a 3-app mix
under MLFQ, p99 interactive latency).

SPEC.md's workload-sim (absent from the reference code)
describes apps as traces of kernel launches, blocking syncs and think gaps.
Here each app is a thread with its own CUDA stream. Every kernel goes
through the launch gate (the interposer hook), the app's synchronisations
are reported as blocking calls (idleness, §6.1), and a scheduler
thread runs the MLFQ tick every 10 ms. Switches are real swaps
through the CUDA engine. Kernels are synthetic (one busy warp for the given
time); the working sets are real (filled, checksummed on every restore,
compared byte for byte at the end).

Per request: latency to the first kernel's completion (the TTFT analogue
SPEC.md uses) and to the request's completion.
"""
from __future__ import annotations

import random
import statistics
import threading
import time
from dataclasses import dataclass
from typing import Dict, List, Optional

from . import engine as E
from ._lib import TIER_GPU, TIER_PAGED, TIER_PINNED

GIB = 1 << 30


@dataclass
class AppSpec:
    app: int
    name: str
    size_gib: float
    burst: int           # kernels per request
    kernel_ms: float     # per kernel
    think_s: float       # gap between requests
    jitter: float = 0.1  # +-fraction applied to think_s


def config3_mix(interval_s: float = 3.0) -> List[AppSpec]:
    """BASELINE configs[2]: code completion (interactive), image generation,
    batch OCR (pages with short I/O gaps)."""
    return [
        AppSpec(0, "code-completion", 16, burst=5, kernel_ms=20, think_s=interval_s),
        AppSpec(1, "image-gen", 24, burst=10, kernel_ms=100, think_s=5.0),
        AppSpec(2, "batch-ocr", 12, burst=5, kernel_ms=50, think_s=0.15),
    ]


def _pct(xs: List[float], q: float) -> Optional[float]:
    if not xs:
        return None
    s = sorted(xs)
    return s[min(len(s) - 1, int(round(q * (len(s) - 1))))]


def run_workload(apps: List[AppSpec], horizon_s: float = 30.0, gpu_gib: int = 32, pinned_gib: int = 16,
                 paged_gib: int = 64, seed: int = 0x4E495849, tick_s: float = 0.01, prefetch: bool = False) -> Dict:
    eng = E.SwapEngine(gpu_capacity=gpu_gib * GIB, pinned_capacity=pinned_gib * GIB, paged_capacity=paged_gib * GIB)
    gate = None
    streams = {}
    try:
        used = {TIER_GPU: 0, TIER_PINNED: 0}
        caps = {TIER_GPU: gpu_gib * GIB, TIER_PINNED: pinned_gib * GIB}
        for a in apps:  # initial placement: GPU while it fits, then pinned, then paged
            size = int(a.size_gib * GIB)
            tier = next((t for t in (TIER_GPU, TIER_PINNED) if used[t] + size <= caps[t]), TIER_PAGED)
            if tier in used:
                used[tier] += size
            eng.allocate(a.app, size, tier)
            eng.fill_pattern(a.app, seed)
        gate = E.LaunchGate(eng, E.PlannerConfig(pinned_budget=pinned_gib * GIB))
        gate.set_prefetch(prefetch)
        for a in apps:
            streams[a.app] = E.stream_create()
            gate.attach(a.app, streams[a.app], 0.0)

        t0 = time.perf_counter()
        now = lambda: time.perf_counter() - t0  # noqa: E731
        stop = threading.Event()
        lat_first: Dict[int, List[float]] = {a.app: [] for a in apps}
        lat_done: Dict[int, List[float]] = {a.app: [] for a in apps}
        errors: List[str] = []

        def app_loop(a: AppSpec):
            rng = random.Random(seed + a.app)
            s = streams[a.app]
            try:
                while not stop.is_set():
                    t_req = now()
                    for k in range(a.burst):
                        with gate.launching(a.app, now(), timeout_s=horizon_s + 60):
                            E.launch_busy_kernel(s, int(a.kernel_ms * 1e6))
                        gate.api_event(a.app, now(), 1)  # BlockingEnter: cudaStreamSynchronize
                        E.stream_sync(s)
                        gate.api_event(a.app, now(), 2)  # BlockingExit
                        if k == 0:
                            lat_first[a.app].append(now() - t_req)
                    lat_done[a.app].append(now() - t_req)
                    think = a.think_s * (1 + a.jitter * (2 * rng.random() - 1))
                    stop.wait(think)
            except Exception as e:  # noqa: BLE001
                if not stop.is_set():
                    errors.append(f"app {a.app}: {e}")

        def sched_loop():
            try:
                while not stop.is_set():
                    gate.tick(now())
                    stop.wait(tick_s)
            except Exception as e:  # noqa: BLE001
                errors.append(f"scheduler: {e}")

        threads = [threading.Thread(target=app_loop, args=(a,), daemon=True) for a in apps]
        threads.append(threading.Thread(target=sched_loop, daemon=True))
        for t in threads:
            t.start()
        time.sleep(horizon_s)
        stop.set()
        threads[-1].join()  # the scheduler thread: from here on this thread ticks
        # A held app thread only wakes when it is scheduled: keep ticking
        # until every app thread has left.
        deadline = time.perf_counter() + 120
        while any(t.is_alive() for t in threads[:-1]) and time.perf_counter() < deadline:
            try:
                gate.tick(now())
            except Exception:  # noqa: BLE001
                pass
            time.sleep(tick_s)
        for t in threads:
            t.join(5)
        for s in streams.values():
            E.stream_sync(s)
        bad = sum(eng.verify_pattern(a.app, seed) for a in apps)
        eng.audit()
        per_app = {}
        for a in apps:
            f, d = lat_first[a.app], lat_done[a.app]
            per_app[a.name] = {
                "requests": len(d),
                "first_kernel_ms": {"p50": _ms(_pct(f, 0.5)), "p99": _ms(_pct(f, 0.99)), "mean": _ms(statistics.mean(f) if f else None)},
                "request_ms": {"p50": _ms(_pct(d, 0.5)), "p99": _ms(_pct(d, 0.99)), "mean": _ms(statistics.mean(d) if d else None)},
            }
        return {"horizon_s": horizon_s, "switches": gate.switches(), "per_app": per_app, "byte_exact": bad == 0,
                "errors": errors, "apps": [a.__dict__ for a in apps], "prefetch": prefetch,
                "prefetched_bytes": gate.prefetched_bytes(), "pinned_gib": pinned_gib}
    finally:
        if gate is not None:
            gate.close()
        for s in streams.values():
            E.stream_destroy(s)
        eng.close()


def _ms(x: Optional[float]) -> Optional[float]:
    return None if x is None else round(x * 1e3, 1)
