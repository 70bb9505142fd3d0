"""The nixie CLI (paper_2601_11743_b200/cli.py): scenario
loading and validation, reports, compare / sweep semantics, exit codes. CPU
only: runs go through nx_workload_model on the virtual clock. The report of
the product library is checked against the same metrics computed from the
reference twin's trace (oracle/_ref/ref_workload: the unmodified reference
library under the same workload engine)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2601_11743_b200 import cli  # noqa: E402

SCEN = os.path.join(ROOT, "scenarios", "config3.json")
REF = os.path.join(ROOT, "oracle", "_ref", "ref_workload")

SMALL = {
    "hardware": {"gpu": "256M", "pinned": "128M", "paged": "4G", "pcie_gbs": [4, 4], "host_gbs": [2, 2]},
    "window": "16M", "horizon": 6.0, "mlfq": {"T1": 1.0, "S1": 0.5, "idle": 0.05},
    "apps": [{"id": 0, "kind": "interactive", "size": "160M", "interval": 0.5, "burst": 3, "kernel": 0.02},
             {"id": 1, "kind": "interactive", "size": "128M", "start": 0.2, "interval": 1.0, "burst": 2, "kernel": 0.05},
             {"id": 2, "kind": "batch", "size": "96M", "start": 0.1, "kernel": 0.03, "per_sync": 2}],
}


def _write(tmp_path, obj, name="s.json"):
    p = tmp_path / name
    p.write_text(obj if isinstance(obj, str) else json.dumps(obj))
    return str(p)


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2601_11743_b200.cli", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=300)


def test_defaults_filled_and_round_trip(tmp_path):
    sc = cli.load_scenario(_write(tmp_path, SMALL))
    assert sc["mlfq"]["levels"] == 4 and sc["mlfq"]["tick"] == 0.01   # defaults (SPEC: K=4)
    assert sc["window"] == "16M" and sc["prefetch"] is False
    assert sc["apps"][2]["tier"] == "paged" and sc["apps"][0]["jitter"] == 0.0
    assert cli.normalize(json.loads(json.dumps(sc))) == sc               # load(emit(load(x))) == load(x)


def test_minimal_scenario_loads_with_all_defaults(tmp_path):
    sc = cli.load_scenario(_write(tmp_path, {"apps": [{"id": 0, "kind": "batch", "size": "1G"}]}))
    assert sc["hardware"]["gpu"] == "32G" and sc["window"] == "512M" and sc["mlfq"]["T1"] == 8.0


@pytest.mark.parametrize("bad,needle", [
    ('{"apps": [', "s.json:1:"),                                                      # parse error with position
    ({"apps": []}, "apps"),
    ({"apps": [{"id": 0, "kind": "batch", "size": "64G"}]}, "apps[0].size"),           # larger than the GPU
    ({"apps": [{"id": 0, "kind": "batch", "size": "1G", "colour": 1}]}, "apps[0]: unknown field 'colour'"),
    ({"hardware": {"gpu": "unbounded"}, "apps": [{"id": 0, "kind": "batch", "size": "1G"}]}, "hardware.gpu"),
    ({"mlfq": {"levels": 0}, "apps": [{"id": 0, "kind": "batch", "size": "1G"}]}, "mlfq.levels"),
    ({"apps": [{"id": 0, "kind": "batch", "size": "1G"}, {"id": 0, "kind": "batch", "size": "1G"}]}, "duplicate"),
    ({"apps": [{"id": 0, "kind": "sleepy", "size": "1G"}]}, "apps[0].kind"),
])
def test_scenario_errors_exit_1_naming_the_field(tmp_path, bad, needle):
    p = _cli("run", "--scenario", _write(tmp_path, bad))
    assert p.returncode == 1, p.stderr
    assert needle in p.stderr


def test_run_report_is_deterministic_and_matches_the_trace(tmp_path):
    path = _write(tmp_path, SMALL)
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    assert _cli("run", "--scenario", path, "--out", str(a)).returncode == 0
    assert _cli("run", "--scenario", path, "--out", str(b)).returncode == 0
    assert a.read_bytes() == b.read_bytes()
    rep = json.loads(a.read_text())
    from paper_2601_11743_b200 import engine
    trace = engine.run_workload_model(cli.to_spec(cli.load_scenario(path)))
    run = rep["runs"][0]
    assert run["context_switches"]["count"] == sum(1 for l in trace.splitlines() if l.startswith("X "))
    assert sum(e["requests"] for e in run["apps"].values()) == sum(1 for l in trace.splitlines() if l.startswith("Q "))
    assert rep["scenario"]["mlfq"]["levels"] == 4  # defaults echoed
    assert run["context_switches"]["count"] > 0 and run["apps"]["0"]["requests"] > 0
    assert 0 < run["jain_fairness_interactive"] <= 1


def test_compare_equals_independent_runs(tmp_path):
    path = _write(tmp_path, SMALL)
    sc = cli.load_scenario(path)
    p = _cli("compare", "--scenario", path, "--policies", "nixie,nixie_prefetch")
    assert p.returncode == 0, p.stderr
    rep = json.loads(p.stdout)
    assert [r["policy"] for r in rep["runs"]] == ["nixie", "nixie_prefetch"]
    assert rep["runs"][0] == cli.run_policy(sc, "nixie")
    assert rep["runs"][1] == cli.run_policy(sc, "nixie_prefetch")
    assert _cli("compare", "--scenario", path, "--policies", "nixie,magic").returncode == 1


def test_sweep_varies_one_parameter(tmp_path):
    path = _write(tmp_path, SMALL)
    p = _cli("sweep", "--scenario", path, "--sweep", "pinned=64M,128M,256M", "--format", "json")
    assert p.returncode == 0, p.stderr
    rep = json.loads(p.stdout)
    assert [r["label"] for r in rep["runs"]] == ["pinned=64M", "pinned=128M", "pinned=256M"]
    base = cli.load_scenario(path)
    for r, v in zip(rep["runs"], ("64M", "128M", "256M")):
        sc = dict(base, hardware=dict(base["hardware"], pinned=v))
        expect = cli.run_policy(cli.normalize(sc), "nixie")
        expect["label"] = f"pinned={v}"
        assert r == expect
    assert _cli("sweep", "--scenario", path, "--sweep", "nonsense=1").returncode == 1


def test_csv_and_text_formats(tmp_path):
    path = _write(tmp_path, SMALL)
    p = _cli("run", "--scenario", path, "--format", "csv")
    rows = p.stdout.strip().splitlines()
    # header + 8 switch metrics + 3 global + 5 per app
    assert len(rows) == 1 + 8 + 3 + 5 * len(SMALL["apps"])
    assert any(r.split(",")[2] == "pinned_physical_peak_bytes" and int(r.split(",")[3]) > 0 for r in rows[1:])
    t = _cli("run", "--scenario", path, "--format", "text").stdout
    assert "context switches" in t and "p95" in t and "pinned physical peak" in t and "resident peak" in t
    assert _cli("run", "--scenario", path, "--format", "xml").returncode == 1


def test_validate_prints_the_normalized_scenario():
    p = _cli("validate", "--scenario", SCEN)
    assert p.returncode == 0, p.stderr
    sc = json.loads(p.stdout)
    assert len(sc["apps"]) == 3 and sc["hardware"]["pcie_gbs"] == [52.4, 52.4]


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref/ref_workload not built")
@pytest.mark.parametrize("prefetch", [False, True])
def test_report_equals_the_reference_twins(tmp_path, prefetch):
    """The report of the product library equals the metrics of the reference
    library's trace for the same workload (decisions and virtual-clock timing
    are identical, so every metric is)."""
    sc = cli.load_scenario(_write(tmp_path, dict(SMALL, prefetch=prefetch)))
    spec = cli.to_spec(sc)
    ref = subprocess.run([REF, "-"], input=spec, capture_output=True, text=True, timeout=300)
    assert ref.returncode == 0, ref.stderr
    ours = cli.run_policy(sc, "nixie")
    theirs = {"policy": "nixie", "mode": "model", **cli.metrics(ref.stdout, sc)}
    assert ours == theirs


@pytest.mark.gpu
def test_real_run_matches_the_model_and_is_byte_exact(tmp_path):
    """--real moves every switch's bytes with the CUDA engine: same decisions
    and virtual-clock metrics as the model, every restore byte-exact."""
    path = _write(tmp_path, SMALL)
    p = _cli("compare", "--scenario", path, "--policies", "nixie", "--real")
    assert p.returncode == 0, p.stderr
    real = json.loads(p.stdout)["runs"][0]
    model = cli.run_policy(cli.load_scenario(path), "nixie")
    assert real["mode"] == "real" and real["byte_check_failures"] == 0
    assert {k: v for k, v in real.items() if k != "mode"} == {k: v for k, v in model.items() if k != "mode"}


def test_uvm_round_robin_baselines():
    """uvm_rr_<W>: nvshare-style time slices over the UVM demand-paging model
    (PAPER.md:462). Deterministic; every oversubscribed slice faults; on
    BASELINE config 3 the interactive app waits far longer than under Nixie
    (the paper's comparison)."""
    sc = cli.load_scenario(SCEN)
    a, b = cli.run_policy(sc, "uvm_rr_4"), cli.run_policy(sc, "uvm_rr_4")
    assert a == b
    assert a["uvm"]["faults"] > 0 and a["uvm"]["faulted_bytes"] > 0 and a["uvm"]["pinned_mirror_peak_bytes"] > 0
    assert a["context_switches"]["count"] > 0 and a["apps"]["0"]["requests"] > 0
    nixie = cli.run_policy(sc, "nixie")
    assert nixie["apps"]["0"]["request_latency"]["mean_ms"] < a["apps"]["0"]["request_latency"]["mean_ms"]
    w30 = cli.run_policy(sc, "uvm_rr_30")
    assert w30["context_switches"]["count"] < a["context_switches"]["count"]  # longer slices, fewer handoffs
    for bad in ("uvm_rr_x", "uvm_rr_0", "uvm_rr_-1"):
        with pytest.raises(cli.ScenarioError):
            cli.run_policy(sc, bad)


def test_uvm_fits_without_faults_after_first_touch(tmp_path):
    """Two apps that fit the GPU together fault each page once (first touch)
    and never again: faulted bytes equal the footprints."""
    sc = cli.load_scenario(_write(tmp_path, {
        "hardware": {"gpu": "1G"}, "horizon": 5.0,
        "apps": [{"id": 0, "kind": "interactive", "size": "256M", "interval": 0.5, "burst": 2, "kernel": 0.01},
                 {"id": 1, "kind": "interactive", "size": "256M", "start": 0.1, "interval": 0.5, "burst": 2,
                  "kernel": 0.01}]}))
    r = cli.run_policy(sc, "uvm_rr_4")
    assert r["uvm"]["faulted_bytes"] == 512 << 20


def test_log_keeps_the_requested_trace_lines(tmp_path):
    path = _write(tmp_path, SMALL)
    rep = json.loads(_cli("run", "--scenario", path, "--log", "sched").stdout)
    log = rep["runs"][0]["log"]
    assert log and {l.split()[0] for l in log} <= {"X", "E", "G", "Q"}
    assert sum(1 for l in log if l.startswith("X ")) == rep["runs"][0]["context_switches"]["count"]
    rep = json.loads(_cli("compare", "--scenario", path, "--policies", "nixie,uvm_rr_1", "--log", "transfers").stdout)
    assert {l.split()[0] for l in rep["runs"][0]["log"]} >= {"S", "P", "L"} and rep["runs"][1]["log"] == []
    assert _cli("run", "--scenario", path, "--log", "everything").returncode != 0
