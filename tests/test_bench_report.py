"""bench.py's report helpers on CPU: the link's raw per-direction rate and the
PCIe counter sampler's plausibility filter (readings above the raw rate are
listed but kept out of the statistics)."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_raw_link_rate():
    assert abs(bench.raw_link_gbs({"gen": 5, "width": 16}) - 32.0 * 16 * 128 / 130 / 8) < 1e-9  # 63.0 GB/s
    assert abs(bench.raw_link_gbs({"gen": 4, "width": 16}) - 31.5) < 0.01
    assert bench.raw_link_gbs({}) == 0.0


def _sampler(readings_kbs):
    c = bench.PcieCounters.__new__(bench.PcieCounters)
    c.stop_ev, c.err = threading.Event(), None
    c.thread = threading.Thread(target=lambda: None)
    c.thread.start()
    c.thr = list(readings_kbs)
    return c


def test_counter_readings_above_the_raw_rate_are_dropped():
    raw = bench.raw_link_gbs({"gen": 5, "width": 16})
    # NVML reports KB/s: (TX, RX) pairs; the middle one over-reads (70 / 90 GB/s)
    out = _sampler([(50e9 / 1024, 48e9 / 1024), (70e9 / 1024, 90e9 / 1024), (54e9 / 1024, 52e9 / 1024)]).stop(raw)
    assert out["available"] and out["samples"] == 3 and out["samples_above_raw_link_rate"] == 1
    assert abs(out["tx_gbs_mean"] - 52.0) < 1e-6 and abs(out["rx_gbs_mean"] - 50.0) < 1e-6
    assert out["rx_gbs_samples"] == [48.0, 90.0, 52.0]


def test_counter_filter_off_without_a_link_rate():
    out = _sampler([(70e9 / 1024, 90e9 / 1024)]).stop(0.0)
    assert out["available"] and out["samples_above_raw_link_rate"] == 0 and abs(out["rx_gbs_mean"] - 90.0) < 1e-6


def test_counter_all_readings_implausible():
    out = _sampler([(70e9 / 1024, 90e9 / 1024)]).stop(63.0)
    assert not out["available"] and "raw rate" in out["error"]
