"""BASELINE config 3 on hardware, short horizon: three apps (interactive,
image generation, batch OCR) share one capped B200 under MLFQ through the
launch gate; every switch is a real swap; working sets stay byte-exact."""
import pytest

from paper_2601_11743_b200.workload import AppSpec, config3_mix, run_workload

pytestmark = pytest.mark.gpu


def test_three_app_mix_under_mlfq(gpu):
    r = run_workload(config3_mix(1.0), horizon_s=8.0)
    assert r["errors"] == [] and r["byte_exact"]
    assert r["switches"] >= 3
    cc = r["per_app"]["code-completion"]
    assert cc["requests"] >= 2 and cc["request_ms"]["p50"] is not None


def test_three_app_mix_with_prefetch(gpu):
    """The gate's ticks prefetch the next candidate's pageable blocks into the
    pinned tier between switches (small pinned budget); still byte-exact."""
    r = run_workload(config3_mix(1.0), horizon_s=8.0, pinned_gib=8, prefetch=True)
    assert r["errors"] == [] and r["byte_exact"]
    assert r["switches"] >= 3
    assert r["prefetched_bytes"] > 0


def test_small_mix_fast_switches(gpu):
    """Small working sets that do not all fit the 1 GiB GPU: frequent real swaps."""
    apps = [AppSpec(0, "a", 0.5, burst=2, kernel_ms=5, think_s=0.2), AppSpec(1, "b", 0.5, burst=2, kernel_ms=5, think_s=0.2),
            AppSpec(2, "c", 0.5, burst=3, kernel_ms=5, think_s=0.2)]  # all idle > 100 ms between requests
    r = run_workload(apps, horizon_s=4.0, gpu_gib=1, pinned_gib=1, paged_gib=2)
    assert r["errors"] == [] and r["byte_exact"] and r["switches"] >= 4


C3_SMALL = """
# config 3 scaled down 8x (capacities and working sets), same MLFQ constants
capacity gpu 4GiB
capacity pinned 2GiB
capacity paged 32GiB
link 0 64GiB/s 64GiB/s full
link 1 32GiB/s 32GiB/s full
dispatch 5e-6
mlfq 4 8 4 0.1 0.01
seed 0x4E495849
horizon 40
interactive 0 2GiB paged 0.0 3 5 0.02 0.1
interactive 1 3GiB paged 0.3 12 40 0.05 0.1
batch 2 1536MiB paged 0.6 0.04 16
"""


def test_mlfq_workload_real_bytes_follow_reference_decisions(gpu):
    """The config-3 workload's decisions on the virtual clock (identical to the
    reference's, tests/test_parity_workload.py) with every switch's bytes moved
    by the CUDA engine: same trace, the engine's placement equals the model's
    after every switch, every restore byte-exact."""
    from paper_2601_11743_b200 import run_workload_model, run_workload_real
    model = run_workload_model(C3_SMALL)
    real = run_workload_real(C3_SMALL)
    core = [ln for ln in real.splitlines() if not (ln[0] in "MVF" or (ln.startswith("H ") and len(ln.split()) == 3))]
    assert core == model.splitlines()
    ms = [ln.split() for ln in real.splitlines() if ln.startswith("M ")]
    vs = [ln.split() for ln in real.splitlines() if ln.startswith("V ")]
    fs = [ln.split() for ln in real.splitlines() if ln.startswith("F ")]
    assert len(ms) >= 5 and all(m[2] == "0" for m in ms)
    assert vs and all(v[3] == "0" for v in vs)
    assert len(fs) == 3 and all(f[2] == "0" for f in fs)


def test_mlfq_workload_with_prefetch_real_bytes(gpu):
    """Prefetch on: the model's committed prefetch moves are mirrored by the
    engine's real prefetch before each switch; placement equals the model's
    and every restore is byte-exact."""
    from paper_2601_11743_b200 import run_workload_model, run_workload_real
    spec = C3_SMALL.replace("horizon 40", "horizon 40\nprefetch on")
    model = run_workload_model(spec)
    real = run_workload_real(spec)
    core = [ln for ln in real.splitlines() if not (ln[0] in "MVF" or (ln.startswith("H ") and len(ln.split()) == 3))]
    assert core == model.splitlines()
    assert any(ln.startswith("H ") and len(ln.split()) == 3 for ln in real.splitlines())  # real prefetch happened
    assert all(ln.split()[2] == "0" for ln in real.splitlines() if ln.startswith("M "))
    assert all(ln.split()[3] == "0" for ln in real.splitlines() if ln.startswith("V "))
    assert all(ln.split()[2] == "0" for ln in real.splitlines() if ln.startswith("F "))
