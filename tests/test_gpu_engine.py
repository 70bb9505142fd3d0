"""CUDA engine parity on a B200 (run with -m gpu).

Bit-exact bar for this byte path:
  * every restore is byte-identical to the pre-eviction contents (K4 compare
    against the pattern, C-oracle checksums of read-back blocks);
  * the swap/schedule decisions of the real engine (plans, per-lane leg
    sequences, placements, schedule events) equal the unmodified reference's
    golden trace for the same scenario.
"""
import ctypes
import hashlib
import itertools
import threading
import time

import pytest

from paper_2601_11743_b200 import (GIB, MIB, EngineConfig, LaunchGate, NixieError, PlannerConfig, SwapEngine,
                                   load_scenario, run_scenario_model, run_scenario_real, trace_lines)
from paper_2601_11743_b200 import engine as nxe
from paper_2601_11743_b200._lib import PATH_AUTO, PATH_CE, PATH_SM, TIER_GPU, TIER_PAGED, TIER_PINNED

pytestmark = pytest.mark.gpu
SEED = 0x4E495849


def det_sha(trace):
    return hashlib.sha256("\n".join(trace_lines(trace)).encode()).hexdigest()


def oracle_block_ok(eng, oracle_lib, app, block):
    data = eng.read_block(block)
    buf = ctypes.create_string_buffer(data, len(data))
    assert oracle_lib.so_compare_block(buf, SEED, app, block) == 0
    return oracle_lib.so_checksum(buf, len(data) // 8)


def test_fill_verify_every_tier(gpu, oracle_lib):
    with SwapEngine(gpu_capacity=64 * MIB, pinned_capacity=64 * MIB, paged_capacity=256 * MIB) as e:
        e.allocate(0, 16 * MIB, TIER_GPU)
        e.allocate(1, 10 * MIB, TIER_PINNED)
        e.allocate(2, 134 * MIB, TIER_PAGED)  # two chunks, paged bounce path
        for app in (0, 1, 2):
            e.fill_pattern(app, SEED)
            assert e.verify_pattern(app, SEED) == 0
            for b in e.app_blocks(app)[:3]:
                ck = oracle_block_ok(e, oracle_lib, app, b)
                assert ck == oracle_lib.so_pattern_block_checksum(SEED, app, b) == e.block_checksum(b)
        b = e.app_blocks(1)[1]
        e.poke_block(b, 4099, 0xA5)
        assert e.verify_pattern(1, SEED) == 1


# sm_tma_ctas (an engine option, set after construction): the SM path's
# default kernel is K1T (TMA bulk copies, -1 = half the SMs); 0 selects K1 (LDG/STG).
PATHS = [dict(path=PATH_SM), dict(path=PATH_SM, sm_tma_ctas=0), dict(path=PATH_SM, sm_tma_ctas=3),
         dict(path=PATH_SM, fused_launch=True), dict(path=PATH_SM, fused_launch=True, sm_tma_ctas=0), dict(path=PATH_CE),
         dict(path=PATH_AUTO), dict(path=PATH_SM, legs_per_launch=3, pcie_legs_in_flight=5), dict(path=PATH_CE, legs_per_launch=1)]


def engine(opts, **kw):
    opts = dict(opts)
    tma = opts.pop("sm_tma_ctas", None)
    e = SwapEngine(**kw, **opts)
    if tma is not None:
        e.set_option("sm_tma_ctas", tma)
    return e


@pytest.mark.parametrize("opts", PATHS, ids=lambda o: "-".join(f"{k}{v}" for k, v in o.items()))
def test_full_gpu_switch_is_byte_exact(gpu, oracle_lib, opts):
    with engine(opts, gpu_capacity=64 * MIB, pinned_capacity=112 * MIB, paged_capacity=64 * MIB) as e:
        e.allocate(0, 64 * MIB, TIER_GPU)  # the incumbent fills the GPU
        e.allocate(1, 48 * MIB, TIER_PINNED)
        e.fill_pattern(0, SEED)
        e.fill_pattern(1, SEED)
        pc = PlannerConfig(streaming_window=8 * MIB, victim_order=[0])
        plan, bi, bo = e.plan_switch(1, pc)
        st = e.switch_to(1, pc)
        assert (st["bytes_in"], st["bytes_out"]) == (bi, bo) == (48 * MIB, 48 * MIB)
        assert st["verified"] == 24 and st["mismatches"] == 0 and st["unverified"] == 0
        assert st["pcie_h2d_bytes"] == 48 * MIB and st["pcie_d2h_bytes"] == 48 * MIB
        e.audit()
        # Per-lane start order is the plan's order (lane FIFO).
        moves = [ln.split() for ln in plan.splitlines()]
        assert [b for b, *_ in e.lane_trace(0)] == [int(m[0]) for m in moves if m[4] == "fetch"]
        assert [b for b, *_ in e.lane_trace(1)] == [int(m[0]) for m in moves if m[4] == "evict"]
        assert e.verify_pattern(0, SEED) == 0 and e.verify_pattern(1, SEED) == 0
        for b in e.app_blocks(1)[::7]:
            assert oracle_block_ok(e, oracle_lib, 1, b) == oracle_lib.so_pattern_block_checksum(SEED, 1, b)
        assert e.app_bytes_resident(1)[0] == 48 * MIB
        st2 = e.switch_to(0, PlannerConfig(streaming_window=8 * MIB, victim_order=[1]))
        assert st2["mismatches"] == 0 and st2["verified"] == st2["pcie_h2d_bytes"] // (2 * MIB)
        assert e.verify_pattern(0, SEED) == 0 and e.verify_pattern(1, SEED) == 0
        e.audit()


@pytest.mark.parametrize("path", [PATH_SM, PATH_CE])
@pytest.mark.parametrize("name", ["kat_planner_ordering", "small_three_apps", "small_pinned_only", "c1_two_apps_2g"])
def test_real_engine_trace_equals_reference(gpu, golden, name, path):
    real = run_scenario_real(load_scenario(name), seed=SEED, path=path)
    assert det_sha(real) == golden["scenarios"][name]["det_sha256"]
    v = [ln.split() for ln in real.splitlines() if ln.startswith("V ")]
    f = [ln.split() for ln in real.splitlines() if ln.startswith("F ")]
    assert v and all(x[3] == "0" for x in v), v
    assert f and all(x[2] == "0" for x in f), f


@pytest.mark.parametrize("opts", [dict(path=PATH_SM), dict(path=PATH_SM, sm_tma_ctas=0), dict(path=PATH_CE)],
                         ids=["sm-k1t", "sm-k1", "ce"])
def test_corrupted_restore_is_detected(gpu, opts):
    with engine(opts, gpu_capacity=32 * MIB, pinned_capacity=64 * MIB, paged_capacity=64 * MIB) as e:
        e.allocate(0, 32 * MIB, TIER_GPU)
        e.allocate(1, 16 * MIB, TIER_PINNED)
        e.fill_pattern(0, SEED)
        e.fill_pattern(1, SEED)
        victim = e.app_blocks(1)[3]
        e.poke_block(victim, 777, 0x5A)  # bit rot while parked in the pinned ring
        with pytest.raises(NixieError) as err:
            e.switch_to(1, PlannerConfig(streaming_window=4 * MIB, victim_order=[0]))
        assert err.value.kind == "InvariantViolation"
        assert "checksum mismatch" in str(err.value) and str(victim) in str(err.value)


def test_copy_path_option_between_switches(gpu):
    """set_option("path") changes the copy path between executes (bench.py's
    sm_path key): SM-kernel switches launch K1T, copy-engine ones do not."""
    with SwapEngine(gpu_capacity=64 * MIB, pinned_capacity=112 * MIB, paged_capacity=64 * MIB, path=PATH_CE) as e:
        e.allocate(0, 64 * MIB, TIER_GPU)
        e.allocate(1, 48 * MIB, TIER_PINNED)
        e.fill_pattern(0, SEED)
        e.fill_pattern(1, SEED)
        nxt = 1
        for p in (PATH_CE, PATH_SM, PATH_CE, PATH_SM):
            e.set_option("path", p)
            st = e.switch_to(nxt, PlannerConfig(streaming_window=8 * MIB, victim_order=[1 - nxt]))
            assert st["mismatches"] == 0 and st["verified"] == st["pcie_h2d_bytes"] // (2 * MIB)
            assert (st["k1_launches"] > 0) == (p == PATH_SM), (p, st["k1_launches"])
            nxt = 1 - nxt
        assert e.verify_pattern(0, SEED) == 0 and e.verify_pattern(1, SEED) == 0
        e.audit()


def test_launch_gate_holds_kernels_until_swap_in(gpu, oracle_lib):
    e = SwapEngine(gpu_capacity=64 * MIB, pinned_capacity=112 * MIB, paged_capacity=64 * MIB)
    s0, s1 = nxe.stream_create(), nxe.stream_create()
    out = nxe.pinned_buffer(16)
    try:
        e.allocate(0, 64 * MIB, TIER_GPU)
        e.allocate(1, 48 * MIB, TIER_PINNED)
        e.fill_pattern(0, SEED)
        e.fill_pattern(1, SEED)
        gate = LaunchGate(e, PlannerConfig(streaming_window=8 * MIB))
        gate.attach(0, s0, 0.0)
        gate.attach(1, s1, 0.0)
        gate.context_switch(0, 0.0)  # app 0 is resident: empty plan, grant only
        assert gate.granted() == 0 and gate.before_launch(0, 0.1)
        gate.after_launch(0)
        # App 1's "interposed launch" runs on its own thread and is held there.
        passed = {}

        def app1():
            with gate.launching(1, 0.2, timeout_s=60.0) as launch:
                passed["v"] = launch.passed
                gate.app_checksum_async(1, s1, out)  # ordered after the swap-in on the device

        th = threading.Thread(target=app1)
        th.start()
        time.sleep(0.3)
        assert th.is_alive(), "app 1's launch was not held"
        assert gate.select_next(0.3) == 1
        st = gate.context_switch(1, 0.3)  # scheduler thread: swap app 1 in
        th.join(60)
        assert not th.is_alive() and passed["v"] is False
        assert st["bytes_in"] == 48 * MIB and st["mismatches"] == 0
        nxe.stream_sync(s1)
        res = (ctypes.c_uint64 * 2).from_address(out)
        want = sum(oracle_lib.so_pattern_block_checksum(SEED, 1, b) for b in e.app_blocks(1)) % (1 << 64)
        assert res[1] == 0 and res[0] == want
        assert gate.granted() == 1
        with pytest.raises(NixieError):  # app 0 lost the grant: its launch is held (here: times out)
            gate.before_launch(0, 0.5, timeout_s=0.2)
        gate.close()
    finally:
        nxe.free_pinned(out)
        nxe.stream_destroy(s0)
        nxe.stream_destroy(s1)
        e.close()


def test_calibration_and_probe(gpu):
    with SwapEngine(gpu_capacity=64 * MIB, pinned_capacity=64 * MIB, paged_capacity=64 * MIB) as e:
        p = e.probe_pcie(256 * MIB, 32 * MIB)
        for k in ("ce_h2d", "ce_d2h", "ce_bidir_total", "sm_h2d", "sm_d2h", "sm_bidir_total"):
            assert p[k] > 5.0, p
        c = e.calibrate(64 * MIB)
        assert len(c["legs"]) == 8 and all(x > 1.0 for x in c["ce_gbps"] + c["sm_gbps"])
        q = e.probe_pcie_paced(256 * MIB, 32 * MIB, 2)  # the engine's paced shape
        assert q["ce_bidir_h2d"] > 5.0 and q["ce_bidir_d2h"] > 5.0, q
        assert q["ce_bidir_total"] <= q["ce_bidir_h2d"] + q["ce_bidir_d2h"] + 1e-6, q


def test_leg_records_log_every_hop(gpu):
    """nx_leg_records: one record per hop of the last switch (the reference's
    TransferRecord log) with times inside the switch, PCIe and host hops
    (two-hop through a 16 MiB pinned budget) alike."""
    with SwapEngine(gpu_capacity=64 * MIB, pinned_capacity=16 * MIB, paged_capacity=256 * MIB, path=PATH_CE,
                    host_threads=2) as e:
        e.allocate(0, 64 * MIB, TIER_GPU)
        e.allocate(1, 64 * MIB, TIER_PAGED)
        e.fill_pattern(0, SEED)
        e.fill_pattern(1, SEED)
        pc = PlannerConfig(streaming_window=4 * MIB, pinned_budget=16 * MIB, victim_order=[0])
        plan, bi, bo = e.plan_switch(1, pc)
        st = e.switch_to(1, pc)
        recs = e.leg_records()
        hops = sum(int(m[3]) for m in (ln.split() for ln in plan.splitlines()))  # "block src dst distance kind"
        assert len(recs) == hops > (bi + bo) // (2 * MIB), (len(recs), hops)  # some moves are two-hop
        pcie = [r for r in recs if 0 in (r["src"], r["dst"])]
        host = [r for r in recs if 0 not in (r["src"], r["dst"])]
        assert len(pcie) == (st["pcie_h2d_bytes"] + st["pcie_d2h_bytes"]) // (2 * MIB) and host, (len(pcie), len(host))
        span = st["wall_s"] + 1e-3
        assert all(0 <= r["start_s"] <= r["end_s"] <= span for r in recs), recs[:4]
        assert e.verify_pattern(1, SEED) == 0 and e.verify_pattern(0, SEED) == 0


def test_prefetch_then_switch_is_byte_exact(gpu):
    """Prefetch: the next app's pageable blocks move to the
    pinned tier in the background (host copy pool) while the incumbent owns the
    GPU; the later switch fetches them from pinned, byte-exact. A prefetch
    still running when the switch comes is quiesced first (cancel_pending)."""
    with SwapEngine(gpu_capacity=64 * MIB, pinned_capacity=96 * MIB, paged_capacity=256 * MIB) as e:
        e.allocate(0, 64 * MIB, TIER_GPU)
        e.allocate(1, 48 * MIB, TIER_PAGED)
        e.allocate(2, 48 * MIB, TIER_PAGED)
        for a in (0, 1, 2):
            e.fill_pattern(a, SEED)
        pc = PlannerConfig(streaming_window=8 * MIB, victim_order=[0])
        assert e.prefetch_begin(1, pc) == 24
        while e.prefetch_pump():
            pass
        assert e.prefetch_quiesce() == 48 * MIB
        assert e.app_bytes_resident(1)[1] == 48 * MIB  # all of app 1 now in pinned
        e.audit()
        st = e.switch_to(1, pc)
        assert st["bytes_in"] == 48 * MIB
        app1 = set(e.app_blocks(1))
        assert not [b for b, src, dst in e.lane_trace(2) if b in app1]  # nothing of app 1 came up from paged
        assert e.verify_pattern(1, SEED) == 0
        # cancelled mid-way: the switch quiesces the prefetch first
        pc2 = PlannerConfig(streaming_window=8 * MIB, victim_order=[1, 0])
        n = e.prefetch_begin(2, pc2)
        assert n > 0
        st = e.switch_to(2, pc2)
        e.audit()
        for a in (0, 1, 2):
            assert e.verify_pattern(a, SEED) == 0


@pytest.mark.parametrize("lag", [-1, 0, 8, 64])
@pytest.mark.parametrize("name", ["small_three_apps", "c1_two_apps_2g"])
def test_pacing_keeps_reference_trace(gpu, golden, name, lag):
    """D2H pacing (pace_lag_legs) only delays departure groups on the device:
    plans, per-lane orders and placements still equal the reference's, every
    restore is byte-exact, and lag 0 (the direction lockstep) still finishes."""
    real = run_scenario_real(load_scenario(name), seed=SEED, path=PATH_CE, pace_lag_legs=lag)
    assert det_sha(real) == golden["scenarios"][name]["det_sha256"]
    v = [ln.split() for ln in real.splitlines() if ln.startswith("V ")]
    assert v and all(x[3] == "0" for x in v), v


@pytest.mark.parametrize("lag", [0, 16, 64])
def test_paced_full_gpu_exchange(gpu, oracle_lib, lag):
    """A full GPU exchanging 1 GiB each way: with pacing on, departure groups
    wait for landed fetches (pace_waits > 0), the lanes keep the plan's order
    and both apps stay byte-exact over several switches."""
    with SwapEngine(gpu_capacity=1 * GIB, pinned_capacity=2 * GIB, paged_capacity=64 * MIB, path=PATH_CE,
                    pace_lag_legs=lag) as e:
        e.allocate(0, 1 * GIB, TIER_GPU)
        e.allocate(1, 1 * GIB, TIER_PINNED)
        e.fill_pattern(0, SEED)
        e.fill_pattern(1, SEED)
        nxt = 1
        for _ in range(4):
            pc = PlannerConfig(streaming_window=64 * MIB, victim_order=[1 - nxt])
            plan, bi, bo = e.plan_switch(nxt, pc)
            st = e.switch_to(nxt, pc)
            assert (st["bytes_in"], st["bytes_out"]) == (bi, bo) == (1 * GIB, 1 * GIB)
            assert st["mismatches"] == 0 and st["verified"] == 512 and st["unverified"] == 0
            assert st["pace_waits"] > 0, st
            moves = [ln.split() for ln in plan.splitlines()]
            assert [b for b, *_ in e.lane_trace(0)] == [int(m[0]) for m in moves if m[4] == "fetch"]
            assert [b for b, *_ in e.lane_trace(1)] == [int(m[0]) for m in moves if m[4] == "evict"]
            e.audit()
            nxt = 1 - nxt
        assert e.verify_pattern(0, SEED) == 0 and e.verify_pattern(1, SEED) == 0
        for b in e.app_blocks(1)[::61]:
            assert oracle_block_ok(e, oracle_lib, 1, b) == oracle_lib.so_pattern_block_checksum(SEED, 1, b)


# Engine shapes the fuzz rotates through: copy path, batch and group sizes,
# legs in flight, pacing lag (including the lockstep lag 0).
FUZZ_OPTS = [dict(path=PATH_CE), dict(path=PATH_CE, pace_lag_legs=0, d2h_commit_legs=1, first_batch_legs=1),
             dict(path=PATH_CE, pace_lag_legs=2, legs_per_launch=3, pcie_legs_in_flight=5),
             dict(path=PATH_CE, pace_lag_legs=-1, early_frame_release=False),
             dict(path=PATH_SM, legs_per_launch=2), dict(path=PATH_CE, pace_lag_legs=1, pcie_legs_in_flight=1)]


def _reference_deadlocks_under_some_timing(spec):
    """The reference's lane rules (transfer.cpp:131-171, 235-248) can stall
    for good under some link timings: seed 61 deadlocks in 1134 of 2401 timing
    combinations, the unmodified reference binary included.
    The model with one leg per lane is those rules."""
    base = "\n".join(ln for ln in spec.splitlines() if not ln.startswith("link"))
    for up, down, hup, hdown in itertools.product((1, 16, 64), repeat=4):
        try:
            run_scenario_model(f"{base}\nlink 0 {up}GiB/s {down}GiB/s full\nlink 1 {hup}GiB/s {hdown}GiB/s full\n")
        except NixieError as e:
            if "transfer deadlock" in str(e):
                return True
    return False


def test_random_tiny_scenarios_real_engine(gpu, golden):
    """Every golden random instance the reference completes under its eight
    probe timings (robust), through the CUDA engine under a rotating engine
    shape: the reference's decisions (plans, per-lane orders, placements,
    schedule) and every restore byte-exact. Real copy timings are not the
    probe timings: a run may end in the reference's own transfer deadlock,
    and then the reference must reach that deadlock under some timing too."""
    n = ref_deadlocks = 0
    for i, case in enumerate(c for c in golden["random"] if c["robust"]):
        opts = FUZZ_OPTS[i % len(FUZZ_OPTS)]
        try:
            real = run_scenario_real(case["spec"], seed=SEED, host_threads=2, **opts)
        except NixieError as e:
            assert "transfer deadlock" in str(e) and _reference_deadlocks_under_some_timing(case["spec"]), (case["seed"], opts, e)
            ref_deadlocks += 1
            continue
        assert trace_lines(real) == trace_lines(case["trace"]), (case["seed"], opts)
        v = [ln.split() for ln in real.splitlines() if ln.startswith("V ")]
        assert all(x[3] == "0" for x in v), (case["seed"], opts, v)
        n += 1
    assert n >= 80 and ref_deadlocks <= 3, (n, ref_deadlocks)
