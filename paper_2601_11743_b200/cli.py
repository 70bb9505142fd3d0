"""nixie command line: scenarios in, reports out (module cli).

    python -m paper_2601_11743_b200.cli run --scenario s.json --out r.json [--format json|csv|text]
    python -m paper_2601_11743_b200.cli compare --scenario s.json --policies nixie,nixie_prefetch,uvm_rr_4,uvm_rr_30
    python -m paper_2601_11743_b200.cli sweep --scenario s.json --sweep pinned=16G,24G,32G
    python -m paper_2601_11743_b200.cli validate --scenario s.json
    (run / compare / sweep also take --seed, --real and --log transfers|sched|faults)

The reference ships this module as a spec only. A scenario is a JSON file
(schema below). It is translated into the workload engine's text grammar
(include/nixie_workload/workload_sim.hpp) and run on the virtual clock by
nx_workload_model, or with --real through the CUDA engine (real bytes on
the GPU, nx_workload_real). The trace is reduced to a MetricsReport:
per-app request latency, context switches, bytes moved, pinned residency and
Jain fairness.

Scenario schema (every default is echoed into the report):
    {"hardware": {"gpu": "32G", "pinned": "16G", "paged": "96G", "disk": "unbounded",
                  "pcie_gbs": [64, 64], "host_gbs": [32, 32], "disk_gbs": [4, 4], "dispatch_s": 5e-6},
     "window": "512M", "pinned_budget": "unbounded",
     "mlfq": {"levels": 4, "T1": 8.0, "S1": 4.0, "idle": 0.1, "tick": 0.01},
     "seed": 1, "horizon": 60.0, "prefetch": false,
     "apps": [{"id": 0, "kind": "interactive", "size": "16G", "tier": "gpu", "start": 0,
               "interval": 3.0, "burst": 8, "kernel": 0.0125, "jitter": 0.0},
              {"id": 1, "kind": "batch", "size": "12G", "tier": "paged", "start": 0,
               "kernel": 0.25, "per_sync": 1}]}
Sizes take K/M/G/T suffixes (GiB units) or plain bytes; link rates are GiB/s;
keys starting with '_' are comments.

Exit codes: 0 success, 1 scenario error (parse / validation,
named field), 2 internal invariant violation.
"""
from __future__ import annotations

import argparse
import copy
import csv
import io
import json
import math
import sys
from typing import Any, Dict, List, Optional, Tuple

DEFAULTS: Dict[str, Any] = {
    "hardware": {"gpu": "32G", "pinned": "16G", "paged": "96G", "disk": "unbounded",
                 "pcie_gbs": [64.0, 64.0], "host_gbs": [32.0, 32.0], "disk_gbs": [4.0, 4.0], "dispatch_s": 5e-6},
    "window": "512M",
    "pinned_budget": "unbounded",
    "mlfq": {"levels": 4, "T1": 8.0, "S1": 4.0, "idle": 0.1, "tick": 0.01},
    "seed": 1,
    "horizon": 60.0,
    "prefetch": False,
}
APP_DEFAULTS = {
    "interactive": {"tier": "paged", "start": 0.0, "interval": 3.0, "burst": 8, "kernel": 0.0125, "jitter": 0.0},
    "batch": {"tier": "paged", "start": 0.0, "kernel": 0.25, "per_sync": 1},
}
TIERS = ("gpu", "pinned", "paged", "disk")
POLICIES = ("nixie", "nixie_prefetch", "nixie_noprefetch")


class ScenarioError(Exception):
    """Exit code 1: the scenario names the offending field."""


def parse_size(v: Any, field: str) -> Optional[int]:
    """Bytes, or None for 'unbounded'."""
    if isinstance(v, bool):
        raise ScenarioError(f"{field}: expected a size, got {v!r}")
    if isinstance(v, (int, float)):
        if v < 0:
            raise ScenarioError(f"{field}: negative size")
        return int(v)
    if not isinstance(v, str):
        raise ScenarioError(f"{field}: expected a size, got {v!r}")
    s = v.strip()
    if s == "unbounded":
        return None
    mul = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30, "T": 1 << 40}
    unit = s[-1:].upper()
    try:
        if unit in mul:
            return int(float(s[:-1]) * mul[unit])
        return int(s)
    except ValueError:
        raise ScenarioError(f"{field}: cannot parse size {v!r}") from None


def _num(d: Dict[str, Any], key: str, field: str, positive: bool = False, integer: bool = False) -> float:
    v = d[key]
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        raise ScenarioError(f"{field}.{key}: expected a number, got {v!r}")
    if integer and int(v) != v:
        raise ScenarioError(f"{field}.{key}: expected an integer, got {v!r}")
    if positive and v <= 0:
        raise ScenarioError(f"{field}.{key}: must be positive")
    if v < 0:
        raise ScenarioError(f"{field}.{key}: must not be negative")
    return v


def _merge(defaults: Dict[str, Any], given: Dict[str, Any], field: str) -> Dict[str, Any]:
    out = copy.deepcopy(defaults)
    for k, v in given.items():
        if k.startswith("_"):  # comments
            continue
        if k not in defaults:
            raise ScenarioError(f"{field}: unknown field '{k}'")
        out[k] = _merge(defaults[k], v, f"{field}.{k}") if isinstance(defaults[k], dict) else v
    return out


def normalize(raw: Any) -> Dict[str, Any]:
    """A fully validated scenario with every default filled in (SPEC: load_scenario)."""
    if not isinstance(raw, dict):
        raise ScenarioError("scenario: expected a JSON object")
    apps = raw.get("apps")
    sc = _merge(DEFAULTS, {k: v for k, v in raw.items() if k != "apps"}, "scenario")
    if not isinstance(apps, list) or not apps:
        raise ScenarioError("apps: at least one app is required")
    hw = sc["hardware"]
    cap = {t: parse_size(hw[t], f"hardware.{t}") for t in TIERS}
    if cap["gpu"] is None:
        raise ScenarioError("hardware.gpu: the GPU tier must be bounded")
    for k in ("pcie_gbs", "host_gbs", "disk_gbs"):
        v = hw[k]
        if not (isinstance(v, list) and len(v) == 2 and all(isinstance(x, (int, float)) and x > 0 for x in v)):
            raise ScenarioError(f"hardware.{k}: expected [up, down] GiB/s, both positive")
    _num(hw, "dispatch_s", "hardware")
    parse_size(sc["window"], "window")
    parse_size(sc["pinned_budget"], "pinned_budget")
    m = sc["mlfq"]
    _num(m, "levels", "mlfq", positive=True, integer=True)
    for k in ("T1", "S1", "idle", "tick"):
        _num(m, k, "mlfq", positive=True)
    _num(sc, "seed", "scenario", integer=True)
    _num(sc, "horizon", "scenario", positive=True)
    if not isinstance(sc["prefetch"], bool):
        raise ScenarioError("prefetch: expected true or false")
    seen = set()
    norm_apps = []
    for i, a in enumerate(apps):
        f = f"apps[{i}]"
        if not isinstance(a, dict):
            raise ScenarioError(f"{f}: expected an object")
        kind = a.get("kind")
        if kind not in APP_DEFAULTS:
            raise ScenarioError(f"{f}.kind: expected 'interactive' or 'batch', got {kind!r}")
        for req in ("id", "size"):
            if req not in a:
                raise ScenarioError(f"{f}.{req}: required")
        body = {k: v for k, v in a.items() if k not in ("id", "kind", "size")}
        full = _merge(APP_DEFAULTS[kind], body, f)
        full.update(id=a["id"], kind=kind, size=a["size"])
        _num(full, "id", f, integer=True)
        if full["id"] in seen:
            raise ScenarioError(f"{f}.id: duplicate app id {full['id']}")
        seen.add(full["id"])
        size = parse_size(full["size"], f"{f}.size")
        if size is None or size == 0:
            raise ScenarioError(f"{f}.size: must be a positive size")
        if size > cap["gpu"]:
            raise ScenarioError(f"{f}.size: larger than the GPU tier (the planner's precondition, SPEC.md:443)")
        if full["tier"] not in TIERS:
            raise ScenarioError(f"{f}.tier: expected one of {', '.join(TIERS)}")
        _num(full, "start", f)
        _num(full, "kernel", f, positive=True)
        if kind == "interactive":
            _num(full, "interval", f, positive=True)
            _num(full, "burst", f, positive=True, integer=True)
            _num(full, "jitter", f)
        else:
            _num(full, "per_sync", f, positive=True, integer=True)
        norm_apps.append(full)
    sc["apps"] = norm_apps
    return sc


def load_scenario(path: str) -> Dict[str, Any]:
    try:
        with open(path) as f:
            text = f.read()
    except OSError as e:
        raise ScenarioError(f"{path}: {e.strerror}") from None
    try:
        raw = json.loads(text)
    except json.JSONDecodeError as e:
        raise ScenarioError(f"{path}:{e.lineno}:{e.colno}: {e.msg}") from None
    return normalize(raw)


def _bytes_text(v: Any, field: str) -> str:
    b = parse_size(v, field)
    return "unbounded" if b is None else str(b)


def to_spec(sc: Dict[str, Any], prefetch: Optional[bool] = None) -> str:
    """The workload engine's text grammar (workload_sim.hpp:29-42)."""
    hw = sc["hardware"]
    lines = [f"capacity {t} {_bytes_text(hw[t], t)}" for t in TIERS]
    for i, k in enumerate(("pcie_gbs", "host_gbs", "disk_gbs")):
        lines.append(f"link {i} {hw[k][0]}GiB/s {hw[k][1]}GiB/s full")
    m = sc["mlfq"]
    lines += [f"dispatch {hw['dispatch_s']!r}", f"window {_bytes_text(sc['window'], 'window')}",
              f"budget {_bytes_text(sc['pinned_budget'], 'pinned_budget')}",
              f"mlfq {int(m['levels'])} {m['T1']!r} {m['S1']!r} {m['idle']!r} {m['tick']!r}",
              f"seed {int(sc['seed'])}", f"horizon {sc['horizon']!r}",
              f"prefetch {'on' if (sc['prefetch'] if prefetch is None else prefetch) else 'off'}"]
    for a in sc["apps"]:
        size = parse_size(a["size"], "size")
        if a["kind"] == "interactive":
            lines.append(f"interactive {int(a['id'])} {size} {a['tier']} {a['start']!r} {a['interval']!r} "
                         f"{int(a['burst'])} {a['kernel']!r} {a['jitter']!r}")
        else:
            lines.append(f"batch {int(a['id'])} {size} {a['tier']} {a['start']!r} {a['kernel']!r} {int(a['per_sync'])}")
    return "\n".join(lines) + "\n"


def _pct(xs: List[float], q: float) -> Optional[float]:
    if not xs:
        return None
    s = sorted(xs)
    return s[min(len(s) - 1, max(0, math.ceil(q * len(s)) - 1))]


def _stats_ms(xs: List[float]) -> Dict[str, Optional[float]]:
    return {"count": len(xs), "mean_ms": round(1e3 * sum(xs) / len(xs), 3) if xs else None,
            "p50_ms": None if not xs else round(1e3 * _pct(xs, 0.50), 3),
            "p95_ms": None if not xs else round(1e3 * _pct(xs, 0.95), 3),
            "p99_ms": None if not xs else round(1e3 * _pct(xs, 0.99), 3),
            "max_ms": round(1e3 * max(xs), 3) if xs else None}


def jain(xs: List[float]) -> Optional[float]:
    """Jain's fairness index (sum x)^2 / (n sum x^2); 1 is perfectly fair."""
    xs = [x for x in xs if x is not None]
    if not xs or sum(x * x for x in xs) == 0:
        return None
    return sum(xs) ** 2 / (len(xs) * sum(x * x for x in xs))


def metrics(trace: str, sc: Dict[str, Any]) -> Dict[str, Any]:
    """MetricsReport from a workload trace (Q, X, S, R lines of workload_sim.hpp / scenario.hpp)."""
    req: Dict[int, List[Tuple[float, float, float]]] = {}
    switches, sizes = [], []
    pinned_after: Dict[str, int] = {}  # switch k -> pinned bytes resident over all apps after it
    pinned_physical = None  # Z line: MemState::pinned_physical_peak (transit and reservations included)
    bad = {}
    for line in trace.splitlines():
        t = line.split()
        if not t:
            continue
        if t[0] == "Q":
            req.setdefault(int(t[1]), []).append((float(t[3]), float(t[4]), float(t[5])))
        elif t[0] == "X":
            switches.append(float(t[4]) - float(t[2]))
        elif t[0] == "S":
            sizes.append((int(t[5]), int(t[7])))
        elif t[0] == "R":
            pinned_after[t[1]] = pinned_after.get(t[1], 0) + int(t[4])
        elif t[0] == "Z":
            pinned_physical = int(t[1])
        elif t[0] == "V" and (int(t[3]) != 0 or (len(t) >= 8 and int(t[7]) != 0)):
            bad[line] = True   # restore not byte-exact, or restored without a checksum check
        elif (t[0] == "F" and int(t[2]) != 0) or (t[0] == "M" and int(t[2]) != 0):
            bad[line] = True   # final byte check; placement differing from the model
    apps = {}
    norm = []
    for a in sc["apps"]:
        rs = req.get(int(a["id"]), [])
        lat = [e - b for b, _, e in rs]
        first = [f - b for b, f, _ in rs]
        entry = {"kind": a["kind"], "size_bytes": parse_size(a["size"], "size"), "requests": len(rs),
                 "request_latency": _stats_ms(lat), "first_kernel_latency": _stats_ms(first)}
        if a["kind"] == "interactive" and lat:
            # standalone latency: the burst back to back, no switch
            ideal = a["burst"] * a["kernel"]
            entry["normalized_throughput"] = round(ideal / (sum(lat) / len(lat)), 6)
            norm.append(entry["normalized_throughput"])
        apps[str(a["id"])] = entry
    return {
        "apps": apps,
        "context_switches": {**_stats_ms(switches),
                             "bytes_in": sum(i for i, _ in sizes), "bytes_out": sum(o for _, o in sizes)},
        "pinned_resident_peak_bytes": max(pinned_after.values()) if pinned_after else 0,
        # the figure comparable to UVM's pinned mirror: the registry's physical
        # peak over the run (transient use during switches included)
        "pinned_physical_peak_bytes": pinned_physical,
        "jain_fairness_interactive": None if jain(norm) is None else round(jain(norm), 6),
        "byte_check_failures": len(bad),  # --real only: V / F / M lines that are not clean
    }


def simulate_uvm_rr(sc: Dict[str, Any], window_s: float) -> str:
    """The nvshare-style baseline: apps take the GPU in
    round-robin time slices of `window_s` seconds (a holder keeps it while no
    other app has work) and their memory is demand-paged by the UVM model
    (UvmSim through the C ABI: LRU, sequential evict-then-fetch, 2 MiB pages
    with adjacent-page prefetch). Every kernel touches its app's whole
    footprint, as the Nixie workload model assumes. Same app generators as the
    workload engine (workload_sim.hpp:16-20); jitter draws from Python's
    random seeded by (seed, app). Emits the workload trace's X and Q lines
    plus `U faults faulted_bytes mirror_peak`."""
    from ctypes import byref, c_double, c_uint64, c_void_p
    import random
    from ._lib import check, lib
    hw = sc["hardware"]
    gib = float(1 << 30)
    h = c_void_p()
    check(lib.nx_uvm_create(parse_size(hw["gpu"], "gpu"), hw["pcie_gbs"][0] * gib, hw["pcie_gbs"][1] * gib, 1,
                            30e-6, 15, byref(h)))
    try:
        apps = sorted(sc["apps"], key=lambda a: int(a["id"]))
        st = {}
        for a in apps:
            check(lib.nx_uvm_register(h, int(a["id"]), parse_size(a["size"], "size")))
            st[a["id"]] = {"rng": random.Random(int(sc["seed"]) * 1000003 + int(a["id"])), "next": float(a["start"]),
                           "queue": [], "done": 0, "first": None, "n": 0}
        horizon = float(sc["horizon"])
        out: List[str] = []
        dur = c_double()

        def arrive(a, t):  # interactive arrivals up to t join the queue
            s_ = st[a["id"]]
            while a["kind"] == "interactive" and s_["next"] <= t:
                s_["queue"].append(s_["next"])
                j = float(a["jitter"])
                s_["next"] += float(a["interval"]) * (1 + (s_["rng"].uniform(-j, j) if j else 0.0))

        def has_work(a, t):
            arrive(a, t)
            return bool(st[a["id"]]["queue"]) if a["kind"] == "interactive" else t >= float(a["start"])

        t, holder, slice_start, k = 0.0, None, 0.0, 0
        while t < horizon:
            order = apps if holder is None else apps[apps.index(holder) + 1:] + apps[:apps.index(holder) + 1]
            want = [a for a in order if has_work(a, t)]
            if holder is not None and holder in want and (t - slice_start < window_s or want == [holder]):
                cur = holder
            elif want:
                cur = next(a for a in want if a is not holder) if any(a is not holder for a in want) else want[0]
            else:  # idle until the next arrival or batch start
                nxt = [st[a["id"]]["next"] if a["kind"] == "interactive" else float(a["start"]) for a in apps]
                t = min(x for x in nxt if x > t) if any(x > t for x in nxt) else horizon
                continue
            if cur is not holder:
                out.append(f"X {k} {t!r} {t!r} {t!r} {'-' if holder is None else int(holder['id'])} {int(cur['id'])}")
                k += 1
                holder, slice_start = cur, t
            check(lib.nx_uvm_touch(h, int(cur["id"]), float(cur["kernel"]), t, byref(dur)))
            t += dur.value
            if cur["kind"] == "interactive":
                s_ = st[cur["id"]]
                s_["done"] += 1
                if s_["first"] is None:
                    s_["first"] = t
                if s_["done"] == int(cur["burst"]) and t <= horizon:
                    out.append(f"Q {int(cur['id'])} {s_['n']} {s_['queue'][0]!r} {s_['first']!r} {t!r}")
                if s_["done"] == int(cur["burst"]):
                    s_["queue"].pop(0)
                    s_["n"] += 1
                    s_["done"], s_["first"] = 0, None
        f, fb, mp = c_uint64(), c_uint64(), c_uint64()
        check(lib.nx_uvm_stats(h, byref(f), byref(fb), byref(mp)))
        out.append(f"U {f.value} {fb.value} {mp.value}")
        return "\n".join(out) + "\n"
    finally:
        lib.nx_uvm_destroy(h)


LOG_KINDS = {  # --log: trace lines kept in the report (workload_sim.hpp / scenario.hpp trace formats)
    "transfers": ("S", "P", "L", "R", "H", "h"),  # switch headers, plans, per-lane legs, residency, prefetch
    "sched": ("X", "E", "G", "Q"),                 # switches, scheduler log rows, requests
    "faults": ("U",),                              # UVM policies: fault count, faulted bytes, mirror peak
}


def _with_log(run: Dict[str, Any], trace: str, log: Optional[str]) -> Dict[str, Any]:
    if log:
        keep = LOG_KINDS[log]
        run["log"] = [l for l in trace.splitlines() if l.split(" ", 1)[0] in keep]
    return run


def run_policy(sc: Dict[str, Any], policy: str, real: bool = False, log: Optional[str] = None) -> Dict[str, Any]:
    if log is not None and log not in LOG_KINDS:
        raise ScenarioError(f"--log: expected one of {', '.join(LOG_KINDS)}, got {log!r}")
    if policy.startswith("uvm_rr_"):
        try:
            w = float(policy[len("uvm_rr_"):])
        except ValueError:
            raise ScenarioError(f"policies: bad time slice in '{policy}'") from None
        if w <= 0 or real:
            raise ScenarioError(f"policies: '{policy}' needs a positive slice and runs on the model only")
        trace = simulate_uvm_rr(sc, w)
        u = [l.split() for l in trace.splitlines() if l.startswith("U ")][0]
        m = metrics(trace, sc)
        m["pinned_physical_peak_bytes"] = int(u[3])  # UVM: every GPU-resident page has a pinned mirror page
        return _with_log({"policy": policy, "mode": "model", **m,
                          "uvm": {"faults": int(u[1]), "faulted_bytes": int(u[2]), "pinned_mirror_peak_bytes": int(u[3])}},
                         trace, log)
    if policy not in POLICIES:
        raise ScenarioError(f"policies: unknown policy '{policy}' (known: {', '.join(POLICIES)}, uvm_rr_<seconds>)")
    prefetch = {"nixie": None, "nixie_prefetch": True, "nixie_noprefetch": False}[policy]
    spec = to_spec(sc, prefetch)
    from . import engine  # loads lib/libnixie_b200.so: no fallback
    trace = engine.run_workload_real(spec) if real else engine.run_workload_model(spec)
    return _with_log({"policy": policy, "mode": "real" if real else "model", **metrics(trace, sc)}, trace, log)


def report(sc: Dict[str, Any], runs: List[Dict[str, Any]], **extra) -> Dict[str, Any]:
    return {"scenario": sc, "runs": runs, **extra}


def _rows(rep: Dict[str, Any]) -> List[List[Any]]:
    rows = [["run", "scope", "metric", "value"]]
    for i, r in enumerate(rep["runs"]):
        tag = r.get("label", r["policy"])
        for k in ("count", "mean_ms", "p50_ms", "p95_ms", "p99_ms", "max_ms", "bytes_in", "bytes_out"):
            rows.append([tag, "switch", k, r["context_switches"][k]])
        rows.append([tag, "global", "pinned_physical_peak_bytes", r["pinned_physical_peak_bytes"]])
        rows.append([tag, "global", "pinned_resident_peak_bytes", r["pinned_resident_peak_bytes"]])
        rows.append([tag, "global", "jain_fairness_interactive", r["jain_fairness_interactive"]])
        for app, e in r["apps"].items():
            rows.append([tag, f"app{app}", "requests", e["requests"]])
            for k in ("mean_ms", "p50_ms", "p95_ms", "p99_ms"):
                rows.append([tag, f"app{app}", f"request_{k}", e["request_latency"][k]])
    return rows


def emit_report(rep: Dict[str, Any], fmt: str, path: Optional[str]) -> str:
    if fmt == "json":
        out = json.dumps(rep, sort_keys=True, indent=2) + "\n"
    elif fmt == "csv":
        buf = io.StringIO()
        csv.writer(buf, lineterminator="\n").writerows(_rows(rep))
        out = buf.getvalue()
    elif fmt == "text":
        lines = []
        for r in rep["runs"]:
            cs = r["context_switches"]
            lines.append(f"== {r.get('label', r['policy'])} ({r['mode']})")
            lines.append(f"context switches {cs['count']:>5}  p50 {cs['p50_ms']} ms  p95 {cs['p95_ms']} ms  "
                         f"moved in {cs['bytes_in'] / 2**30:.2f} GiB out {cs['bytes_out'] / 2**30:.2f} GiB")
            pp = r.get("pinned_physical_peak_bytes")
            lines.append(f"pinned physical peak {'-' if pp is None else f'{pp / 2**30:.2f} GiB'}   "
                         f"resident peak after switches {r['pinned_resident_peak_bytes'] / 2**30:.2f} GiB   "
                         f"Jain fairness (interactive) {r['jain_fairness_interactive']}")
            lines.append(f"{'app':>5} {'kind':>12} {'requests':>9} {'mean ms':>10} {'p50 ms':>10} {'p99 ms':>10}")
            for app, e in r["apps"].items():
                rl = e["request_latency"]
                lines.append(f"{app:>5} {e['kind']:>12} {e['requests']:>9} {str(rl['mean_ms']):>10} "
                             f"{str(rl['p50_ms']):>10} {str(rl['p99_ms']):>10}")
        out = "\n".join(lines) + "\n"
    else:
        raise ScenarioError(f"--format: expected json, csv or text, got {fmt!r}")
    if path:
        with open(path, "w") as f:
            f.write(out)
    return out


def _set_path(sc: Dict[str, Any], param: str, value: str) -> Dict[str, Any]:
    """sweep: one named parameter; 'gpu'/'pinned'/... are hardware tiers, 'mlfq.T1' nests."""
    raw = copy.deepcopy(sc)
    keys = param.split(".")
    if len(keys) == 1 and keys[0] in TIERS:
        keys = ["hardware", keys[0]]
    node = raw
    for k in keys[:-1]:
        if not isinstance(node.get(k), dict):
            raise ScenarioError(f"--sweep: unknown parameter '{param}'")
        node = node[k]
    if keys[-1] not in node:
        raise ScenarioError(f"--sweep: unknown parameter '{param}'")
    try:
        node[keys[-1]] = json.loads(value)
    except ValueError:
        node[keys[-1]] = value
    return normalize(raw)


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="nixie", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("run", "compare", "sweep", "validate"):
        p = sub.add_parser(name)
        p.add_argument("--scenario", required=True)
        if name != "validate":
            p.add_argument("--out")
            p.add_argument("--format", default="json")
            p.add_argument("--real", action="store_true", help="move the bytes on the GPU (CUDA engine)")
            p.add_argument("--log", choices=sorted(LOG_KINDS), help="keep these trace lines in each run")
        if name == "compare":
            p.add_argument("--policies", default="nixie,nixie_prefetch")
        if name == "sweep":
            p.add_argument("--sweep", required=True, help="param=v1,v2,...")
            p.add_argument("--policy", default="nixie")
        if name in ("run", "sweep"):
            p.add_argument("--seed", type=int)
    a = ap.parse_args(argv)
    try:
        sc = load_scenario(a.scenario)
        if getattr(a, "seed", None) is not None:
            sc["seed"] = a.seed
        if a.cmd == "validate":
            print(json.dumps(sc, sort_keys=True, indent=2))
            return 0
        if a.cmd == "run":
            rep = report(sc, [run_policy(sc, "nixie", a.real, a.log)])
        elif a.cmd == "compare":
            rep = report(sc, [run_policy(sc, p.strip(), a.real, a.log) for p in a.policies.split(",") if p.strip()])
        else:
            param, _, values = a.sweep.partition("=")
            if not values:
                raise ScenarioError("--sweep: expected param=v1,v2,...")
            runs = []
            for v in values.split(","):
                r = run_policy(_set_path(sc, param, v), a.policy, a.real, a.log)
                r["label"] = f"{param}={v}"
                runs.append(r)
            rep = report(sc, runs, sweep={"parameter": param, "values": values.split(",")})
        out = emit_report(rep, a.format, a.out)
        if not a.out:
            sys.stdout.write(out)
        return 0
    except ScenarioError as e:
        print(f"nixie: {e}", file=sys.stderr)
        return 1
    except Exception as e:  # the library's errors: scenario errors are 1, invariants 2
        kind = getattr(e, "kind", None)
        print(f"nixie: {kind or type(e).__name__}: {e}", file=sys.stderr)
        if kind in ("ParseError", "ValidationError", "InvalidScenario", "AppTooLarge", "CapacityExceeded",
                    "InsufficientEvictable", "UnknownApp", "UnknownChunk"):
            return 1
        return 2


if __name__ == "__main__":
    sys.exit(main())
