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


def test_small_mix_fast_switches(gpu):
    """Small working sets that do not all fit the 1 GiB GPU: frequent real swaps."""
    apps = [AppSpec(0, "a", 0.5, burst=2, kernel_ms=5, think_s=0.2), AppSpec(1, "b", 0.5, burst=2, kernel_ms=5, think_s=0.2),
            AppSpec(2, "c", 0.5, burst=3, kernel_ms=5, think_s=0.2)]  # all idle > 100 ms between requests
    r = run_workload(apps, horizon_s=4.0, gpu_gib=1, pinned_gib=1, paged_gib=2)
    assert r["errors"] == [] and r["byte_exact"] and r["switches"] >= 4
