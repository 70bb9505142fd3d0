"""Unmodified CUDA applications under the interposer:
lib/nixied + LD_PRELOAD=lib/libnixie_shim.so.

Applications: tests/apps/vecapp.cu (C++/CUDA, cudaMalloc + <<<>>>), and
tests/apps/torch_app.py (PyTorch elementwise). Their combined working sets
exceed the daemon's GPU budget, so they can only finish if the daemon swaps
them in and out: each app checks every word of its data on the device every
iteration and on the host at the end, and the daemon verifies every restore
by checksum (mismatches would fail the switch)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2601_11743_b200.interpose import NIXIED, SHIM, VECAPP, Daemon, run_apps  # noqa: E402

pytestmark = pytest.mark.gpu


def _vec(mib, iters, think_ms, seed, name):
    return [VECAPP, "--mib", str(mib), "--buffers", "6", "--iters", str(iters), "--think-ms", str(think_ms),
            "--seed", str(seed), "--name", name]


def _save(name, d, res):
    """Keeps the daemon log and app outputs (gpurun_out/ is merged back from the GPU box)."""
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, f"interposer_{name}.jsonl"), "w") as f:
            for r in d.records():
                f.write(json.dumps(r) + "\n")
            for r in res:
                f.write(json.dumps({"event": "app", "rc": r["rc"], "out": r["out"], "stderr": r["stderr"][-500:]}) + "\n")


def _check(res, d):
    for r in res:
        assert r["rc"] == 0, (r["stderr"], d.stderr())
        assert r["out"] is not None, r["stdout"]


@pytest.mark.parametrize("mode", ["default", "isolate_victims", "reference_victims"])
def test_two_vecapps_oversubscribed(mode):
    """2 x 3 GiB on a 4 GiB budget: every iteration after a think gap needs a
    switch. Byte-exact (device + host checks), every restore verified. Also
    with victims unmapping lost slabs right after each switch, and with the
    reference planner's victim blocks."""
    extra = {"default": [], "isolate_victims": ["--isolate-victims"], "reference_victims": ["--reference-victims"]}[mode]
    with Daemon(gpu="4G", pinned="4G", paged="16G", extra=extra) as d:
        res = run_apps(d, [_vec(3072, 6, 250, 11, "a"), _vec(3072, 6, 250, 22, "b")], timeout=600)
        _save("two_vecapps" + ("" if mode == "default" else "_" + mode), d, res)
        _check(res, d)
        sw = d.switches()
    d.stop()
    for r in res:
        assert r["out"]["device_errors"] == 0 and r["out"]["host_mismatch"] == 0
    assert len(sw) >= 3, sw
    assert all(s["mismatches"] == 0 for s in sw)
    assert sum(s["verified"] for s in sw) > 0
    assert sum(s["pcie_h2d"] for s in sw) > 0 and sum(s["pcie_d2h"] for s in sw) > 0
    # both directions in the same switch (bidirectional swap)
    assert any(s["pcie_h2d"] > 0 and s["pcie_d2h"] > 0 for s in sw)


def test_driver_api_launches_are_gated():
    """One app launches through the driver API (cuLaunchKernel obtained with
    cudaGetDriverEntryPoint, i.e. cuGetProcAddress); the shim's wrapped entry
    table gates those launches like runtime ones."""
    with Daemon(gpu="4G", pinned="4G", paged="16G") as d:
        res = run_apps(d, [_vec(3072, 5, 250, 31, "drv") + ["--driver", "1"], _vec(3072, 5, 250, 32, "rt")], timeout=600)
        _save("driver_api", d, res)
        _check(res, d)
        recs = d.records()
    byes = {r["app"]: r for r in recs if r.get("event") == "bye"}
    assert len(byes) == 2
    assert max(b["table_launches"] for b in byes.values()) >= 5 * 6
    assert min(b["table_launches"] for b in byes.values()) == 0
    assert len([r for r in recs if r.get("event") == "switch"]) >= 3
    for r in res:
        assert r["out"]["device_errors"] == 0 and r["out"]["host_mismatch"] == 0


def test_prefetch_under_the_daemon():
    """Three apps on a small pinned budget with the daemon's MLFQ prefetch on:
    pageable blocks of the next candidate move to pinned between switches;
    every app still finishes byte-exact."""
    with Daemon(gpu="4G", pinned="2G", paged="16G", prefetch=True) as d:
        res = run_apps(d, [_vec(2048, 5, 300, 41, "a"), _vec(2048, 5, 300, 42, "b"), _vec(2048, 5, 300, 43, "c")],
                       timeout=600)
        _save("prefetch", d, res)
        _check(res, d)
        recs = d.records()
    for r in res:
        assert r["out"]["device_errors"] == 0 and r["out"]["host_mismatch"] == 0
    assert any(r.get("event") == "prefetch" for r in recs)
    assert all(r["mismatches"] == 0 for r in recs if r.get("event") == "switch")


def test_cuda_graph_apps():
    """Apps that capture their iteration into a CUDA graph (thread-local and
    global capture mode) and launch it every iteration: the capture guard
     keeps the shim's own CUDA calls out of the capture, and
    graph launches are gated like kernel launches."""
    with Daemon(gpu="4G", pinned="4G", paged="16G") as d:
        res = run_apps(d, [_vec(3072, 5, 250, 61, "g1") + ["--graph", "1", "--passes", "2"],
                           _vec(3072, 5, 250, 62, "g2") + ["--graph", "2", "--passes", "2"]], timeout=600)
        _save("graphs", d, res)
        _check(res, d)
        sw = d.switches()
    for r in res:
        assert r["out"]["device_errors"] == 0 and r["out"]["host_mismatch"] == 0
    assert len(sw) >= 3 and all(s["mismatches"] == 0 for s in sw)


def test_torch_stream_ordered_allocator():
    """PyTorch with its cudaMallocAsync backend (cudaMallocAsync /
    cudaFreeAsync interposed) beside a CUDA program on a 5 GiB budget."""
    torch_cmd = ["env", "PYTORCH_CUDA_ALLOC_CONF=backend:cudaMallocAsync", sys.executable,
                 os.path.join(ROOT, "tests", "apps", "torch_app.py"), "2048", "12", "0.3"]
    with Daemon(gpu="5G", pinned="4G", paged="16G") as d:
        res = run_apps(d, [torch_cmd, _vec(3072, 16, 300, 71, "a")], timeout=900, stagger_s=2.0)
        _save("torch_async", d, res)
        _check(res, d)
        sw = d.switches()
        byes = {r["app"]: r for r in d.records() if r.get("event") == "bye"}
    assert res[0]["out"]["mismatch"] == 0 and res[0]["out"]["matmul_mismatch"] == 0
    assert len(sw) >= 2 and all(s["mismatches"] == 0 for s in sw)


def test_two_llm_inference_apps():
    """Two unmodified PyTorch LLM-inference programs (Llama architecture,
    0.75B parameters = 1.4 GiB of bf16 weights each) on a 2 GiB budget: the
    pair cannot share the GPU, so every switch between them must evict at
    least 0.8 GiB of the victim and restore as much of the incoming app
    (independent of when the scheduler switches). Every request's logits
    equal the first request's bit for bit."""
    llm = os.path.join(ROOT, "tests", "apps", "llm_app.py")
    with Daemon(gpu="2G", pinned="4G", paged="16G") as d:
        res = run_apps(d, [[sys.executable, llm, "8", "0.3", "1"], [sys.executable, llm, "8", "0.3", "2"]], timeout=900)
        _save("llm", d, res)
        _check(res, d)
        sw = d.switches()
    for r in res:
        assert r["out"]["logit_mismatch"] == 0
        assert r["out"]["weights_gib"] > 1.3  # the pair does not fit 2 GiB
    assert all(s["mismatches"] == 0 for s in sw)
    between = [s for s in sw if s["from"] >= 0 and s["from"] != s["to"]]
    # Switches before both models are loaded may find the incoming app with
    # nothing allocated yet; from the first switch that restores a model on,
    # every switch must move a model's worth each way.
    first = next(i for i, s in enumerate(between) if s["bytes_in"] > 0)
    between = between[first:]
    assert len(between) >= 3, sw
    for s in between:  # per switch, not a timing-dependent sum
        assert s["pcie_h2d"] >= (512 << 20) and s["pcie_d2h"] >= (512 << 20), s
        assert s["pcie_h2d"] == s["bytes_in"] and s["pcie_d2h"] == s["bytes_out"], s  # the plan's bytes crossed the link


def test_memgetinfo_reports_budget():
    with Daemon(gpu="6G", pinned="2G", paged="8G") as d:
        res = run_apps(d, [_vec(1024, 1, 0, 3, "m")], timeout=300)
        _check(res, d)
    free_b, total_b = res[0]["out"]["memgetinfo"]
    assert total_b == 6 << 30
    assert free_b <= total_b - (1 << 30)


def test_three_apps_with_torch():
    """A PyTorch program (elementwise + cuBLAS matmul) and two CUDA programs
    share a 5 GiB budget."""
    with Daemon(gpu="5G", pinned="4G", paged="16G") as d:
        res = run_apps(d, [_vec(2048, 5, 200, 5, "a"), [sys.executable, os.path.join(ROOT, "tests", "apps", "torch_app.py"),
                                                           "2048", "5", "0.2"], _vec(2048, 5, 200, 6, "c")], timeout=900)
        _save("torch_mix", d, res)
        _check(res, d)
        sw = d.switches()
    assert res[1]["out"]["mismatch"] == 0 and res[1]["out"]["matmul_mismatch"] == 0
    assert res[1]["out"]["memgetinfo"][1] == 5 << 30
    byes = {r["app"]: r for r in d.records() if r.get("event") == "bye"}
    py = [r["app"] for r in d.records() if r.get("event") == "hello" and r["name"].startswith("python")][0]
    assert byes[py]["blas_calls"] > 0  # the matmuls were held at the gate
    assert len(sw) >= 3 and all(s["mismatches"] == 0 for s in sw)


def test_app_killed_mid_run_does_not_stall_the_others():
    """An application killed while it holds or waits for the GPU: the daemon
    reaps it (its chunks return to the registry, its slabs to the pool) and
    the other applications finish byte-exact."""
    import signal
    import time
    with Daemon(gpu="4G", pinned="4G", paged="16G") as d:
        victim = d.spawn(_vec(2048, 1000, 100, 51, "victim"))
        others = [d.spawn(_vec(2048, 6, 200, 52 + i, f"o{i}")) for i in range(2)]
        time.sleep(6.0)
        victim.send_signal(signal.SIGKILL)
        victim.wait(30)
        outs = [p.communicate(timeout=600) for p in others]
        recs = d.records()
        alive = d.proc.poll() is None
    assert alive, d.stderr()
    for p, (out, err) in zip(others, outs):
        assert p.returncode == 0, err
        r = json.loads(out.strip().splitlines()[-1])
        assert r["device_errors"] == 0 and r["host_mismatch"] == 0
    byes = [r for r in recs if r.get("event") == "bye"]
    assert len(byes) == 3
    assert all(r["mismatches"] == 0 for r in recs if r.get("event") == "switch")


@pytest.mark.parametrize("combo", ["pitch_launchex", "drvpitch_async"])
def test_interposer_api_breadth(combo):
    """PAPER.md:137's breadth: working sets allocated with cudaMallocPitch /
    cudaMalloc3D / cuMemAllocPitch / cuMemAllocAsync, kernels launched with
    cuLaunchKernelEx (through the cuGetProcAddress table and through the
    PLT), and every iteration opening with synchronous cudaMemcpy2D,
    cudaMemcpy3D, cudaMemset2D and cuMemsetD32 calls right after a think gap
    (when the app has likely been switched out). Two apps oversubscribe a
    4 GiB budget with stale mappings kept (the default for two apps), so an
    ungated synchronous call would read the other app's data (sync_mismatch)
    or fault; all results must be byte-exact."""
    a, b = {"pitch_launchex": (["--alloc", "pitch", "--driver", "2", "--streams", "8"], ["--alloc", "3d", "--driver", "3"]),
            "drvpitch_async": (["--alloc", "drvpitch", "--driver", "2"], ["--alloc", "async", "--driver", "3", "--streams", "4"])}[combo]
    with Daemon(gpu="4G", pinned="4G", paged="16G") as d:
        res = run_apps(d, [_vec(3072, 5, 250, 91, "a") + a + ["--sync-ops", "1"],
                           _vec(3072, 5, 250, 92, "b") + b + ["--sync-ops", "1"]], timeout=600)
        _save("breadth_" + combo, d, res)
        _check(res, d)
        sw = d.switches()
        recs = d.records()
    for r in res:
        o = r["out"]
        assert o["device_errors"] == 0 and o["host_mismatch"] == 0 and o["sync_mismatch"] == 0, o
        assert o["sync_calls"] == 7 * 5
        assert o["bytes"] >= 3000 << 20
    assert len(sw) >= 3 and all(s["mismatches"] == 0 for s in sw)
    # the managed working sets crossed the link in both directions
    assert sum(s["pcie_h2d"] for s in sw) >= 3 << 30 and sum(s["pcie_d2h"] for s in sw) >= 3 << 30
    byes = [r for r in recs if r.get("event") == "bye"]
    assert len(byes) == 2 and max(b_["table_launches"] for b_ in byes) >= 5 * 6


def test_implicit_allocations_count_against_the_budget():
    """cudaDeviceSetLimit(cudaLimitStackSize) grows the device's local-memory
    reservation: the shim charges the drop in free memory to the app, its
    cudaMemGetInfo reports it as used, and the daemon refuses a managed
    allocation that would push managed + implicit bytes past the budget."""
    with Daemon(gpu="4G", pinned="4G", paged="16G") as d:
        res = run_apps(d, [_vec(1024, 1, 0, 7, "base")], timeout=300)
        _check(res, d)
        res2 = run_apps(d, [_vec(1024, 1, 0, 8, "stack") + ["--stack-kib", "4", "--streams", "4"]], timeout=300)
        _check(res2, d)
    used_base = res[0]["out"]["memgetinfo"][1] - res[0]["out"]["memgetinfo"][0]
    used_stack = res2[0]["out"]["memgetinfo"][1] - res2[0]["out"]["memgetinfo"][0]
    assert used_stack >= used_base + (64 << 20), (used_base, used_stack)
    implicit = used_stack - used_base
    # Now a working set that fits the budget alone but not with the stack
    # reservation: the allocation that crosses the budget fails.
    mib = (4096 - (implicit >> 20) // 2)  # > budget - implicit
    with Daemon(gpu="4G", pinned="4G", paged="16G") as d:
        p = d.spawn(_vec(mib, 1, 0, 9, "over") + ["--stack-kib", "4"])
        out, err = p.communicate(timeout=300)
    assert p.returncode != 0 and "out of memory" in err, (p.returncode, err[-400:])


def test_pause_during_a_capture_with_an_allocation_does_not_deadlock():
    """an app holding the GPU begins a stream capture, the daemon
    switches to another app (Pause), and the capturing thread then calls
    cudaMalloc (a managed allocation: an Alloc RPC) before ending the capture.
    The shim's pause waits for the capture to end, so the daemon must serve
    that RPC while it awaits the Drained ack instead of deadlocking until its
    60 s ack timeout (which used to drop the app)."""
    import time
    with Daemon(gpu="4G", pinned="4G", paged="16G", idle_ms=20) as d:
        t0 = time.time()
        a = d.spawn(_vec(3072, 3, 100, 101, "cap") + ["--graph", "3", "--capture-alloc-ms", "8000"])
        # The capture begins about now; app b's first launch then asks for the
        # GPU. The in-capture cudaMalloc comes 8 s into the capture, well after
        # b's request even where b's CUDA start-up takes seconds (one box: 2.5 s
        # with a 4 s delay let the Alloc land before the switch began).
        time.sleep(2.0)
        b = d.spawn(_vec(3072, 3, 100, 102, "other"))
        outs = [p.communicate(timeout=300) for p in (a, b)]
        elapsed = time.time() - t0
    recs = d.records()  # after stop: the summary line is written at exit
    _save("capture_pause", d, [])
    for p, (out, err) in zip((a, b), outs):
        assert p.returncode == 0, err[-2000:]
    assert elapsed < 50, elapsed  # no ack timeout (60 s) on the way
    summ = [r for r in recs if r.get("event") == "summary"]
    sw = [r for r in recs if r.get("event") == "switch"]
    assert sw and all(s["mismatches"] == 0 for s in sw)
    assert summ and summ[-1]["rpcs_in_switch"] >= 1, summ  # the Alloc was served inside a switch
    assert any(r.get("event") == "rpc_in_switch" and r.get("type") == "alloc" for r in recs)
