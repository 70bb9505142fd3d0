"""Benchmark of the Nixie context-switch swap path on B200 (BASELINE.json).

Metric: bidirectional swap GB/s per GPU (% of the measured simultaneous
H2D+D2H PCIe peak); p50/p99 context-switch latency.

Workload (BASELINE.json configs[1]): an interactive 16 GiB app and a 24 GiB
background app on one B200 capped at 32 GiB, 16 GiB pinned budget; the apps
alternate; a step is one steady-state context switch (8 GiB out of the GPU +
8 GiB in, both directions at once). The cold start from pageable memory and
the full scenario are parity-tested in tests/test_gpu_scale.py.

Lines printed by rank 0 (one JSON line):
  value  whole-job GB/s, device-timed (CUDA events around every PCIe launch
         of the timed switches; inputs resident, the first-hop copies are the
         path), summed over ranks / max-over-ranks time
  e2e    the same bytes through the public API call (plan_switch + real
         execute + commits, the C ABI nx_switch), host wall clock; h2d/d2h
         bytes per step are the switch's PCIe bytes
  roofline        the dominant kernel of the timed region (the K3 checksum
                  kernel on the copy-engine path: HBM-bound)
  link_roofline   the path's real bound: PCIe, against the same-run probe
  cpu_baseline    the reference's CPU implementation of the path (see below)

--impl reference: the unmodified reference's CPU path (oracle/_ref built from
/root/reference/proj/src): plan_switch + execute of the reference library for
the same switches plus the switch's bytes moved by host memcpy on all host
cores (the reference models no data), on a bounded sample.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
GIB, MIB = 1 << 30, 1 << 20
METRIC = "bidir swap GB/s per GPU (% of PCIe peak); p50/p99 context-switch latency"
WORKLOAD = ("c2_interactive_background: interactive 16 GiB + background 24 GiB apps alternating on one B200 "
            "capped at 32 GiB, 16 GiB pinned budget, steady-state switches (8 GiB out + 8 GiB in per switch)")


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


class Dist:
    """Host-side barrier / max / sum across ranks (gloo; no data-path collective)."""

    def __init__(self):
        self.rank, self.world, self.local = dist_env()
        self.pg = None
        if self.world > 1:
            import torch.distributed as td
            td.init_process_group("gloo")
            self.td = td

    def barrier(self):
        if self.world > 1:
            self.td.barrier()

    def reduce(self, value: float, op: str) -> float:
        if self.world == 1:
            return value
        import torch
        t = torch.tensor([value], dtype=torch.float64)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX if op == "max" else self.td.ReduceOp.SUM)
        return float(t.item())

    def gather(self, obj) -> list:
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self.td.all_gather_object(out, obj)
        return out

    def close(self):
        if self.world > 1:
            self.td.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for ln in f:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def pcie_link(device: int) -> dict:
    try:
        out = subprocess.run(["nvidia-smi", "-i", str(device), "--query-gpu=name,pcie.link.gen.current,pcie.link.gen.max,"
                              "pcie.link.width.current,pcie.link.width.max", "--format=csv,noheader"],
                             capture_output=True, text=True, timeout=20).stdout.strip()
        name, g, gm, w, wm = [p.strip() for p in out.split(",")]
        return {"gpu": name, "gen": int(g), "gen_max": int(gm), "width": int(w), "width_max": int(wm)}
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)[:80]}


class PcieCounters:
    """The GPU's own PCIe throughput during the timed region: the driver's
    nvmlDeviceGetPcieThroughput TX/RX (KB/s over its 20 ms window), sampled
    every 10 ms by a thread. A counter-level reading of what the copy engines
    moved, which ncu cannot see (it profiles kernels, not DMA). The readings
    include protocol overhead (TLP headers, the read requests of fetches on
    TX, completions on RX), so they sit above the algorithmic rates.
    TX = GPU -> host (evictions), RX = host -> GPU (fetches).
    (The NVML_FI_DEV_PCIE_COUNT_{TX,RX}_BYTES byte counters are 32-bit on these
    boards and, read every 10 ms, still under-count by ~15%: they update
    less often than they wrap at 50 GB/s. Not used.)"""

    def __init__(self, pci_bus_id: str):
        self.h = None
        self.err = None
        self.stop_ev = threading.Event()
        self.thread = None
        self.thr = []
        try:
            import pynvml
            self.nv = pynvml
            pynvml.nvmlInit()
            bus = pci_bus_id.upper()
            for cand in (bus, "0000" + bus if len(bus) == 12 else bus, bus[4:] if len(bus) == 16 else bus):
                try:
                    self.h = pynvml.nvmlDeviceGetHandleByPciBusId(cand)
                    break
                except Exception:  # noqa: BLE001
                    continue
            if self.h is None:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(0)
        except Exception as e:  # noqa: BLE001
            self.err = str(e)[:120]

    def _sample(self):
        nv = self.nv
        return (nv.nvmlDeviceGetPcieThroughput(self.h, nv.NVML_PCIE_UTIL_TX_BYTES),
                nv.nvmlDeviceGetPcieThroughput(self.h, nv.NVML_PCIE_UTIL_RX_BYTES))

    def _run(self):
        while not self.stop_ev.wait(0.01):
            try:
                self.thr.append(self._sample())
            except Exception as e:  # noqa: BLE001
                self.err = str(e)[:120]
                return

    def start(self):
        if self.h is None:
            return
        try:
            self._sample()
        except Exception as e:  # noqa: BLE001
            self.err = str(e)[:120]
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def stop(self, raw_gbs_per_direction: float = 0.0) -> dict:
        """Readings above the link's raw per-direction rate (Gen5 x16: 63.0
        GB/s) cannot be real traffic: on some boxes the NVML window is shorter
        than 20 ms under load and the KB/s figure over-reads. They stay in the
        sample list but not in the statistics."""
        if self.thread is None or not self.thr:
            if self.thread is not None:
                self.stop_ev.set()
                self.thread.join()
            return {"available": False, **({"error": self.err} if self.err else {})}
        self.stop_ev.set()
        self.thread.join()
        tx_all = [t * 1024 / 1e9 for t, _ in self.thr]
        rx_all = [r * 1024 / 1e9 for _, r in self.thr]
        ok = [i for i in range(len(self.thr))
              if raw_gbs_per_direction <= 0 or max(tx_all[i], rx_all[i]) <= raw_gbs_per_direction]
        out = {"available": True, "source": "nvmlDeviceGetPcieThroughput TX/RX (20 ms windows), sampled every 10 ms",
               "samples": len(self.thr), "samples_above_raw_link_rate": len(self.thr) - len(ok),
               "raw_gbs_per_direction": raw_gbs_per_direction,
               "tx_gbs_samples": [round(v, 1) for v in tx_all], "rx_gbs_samples": [round(v, 1) for v in rx_all]}
        if not ok:
            return {**out, "available": False, "error": "every reading exceeds the link's raw rate"}
        tx, rx = [tx_all[i] for i in ok], [rx_all[i] for i in ok]
        return {**out, "tx_gbs_mean": statistics.mean(tx), "rx_gbs_mean": statistics.mean(rx),
                "tx_gbs_p50": statistics.median(tx), "rx_gbs_p50": statistics.median(rx)}


def raw_link_gbs(link: dict) -> float:
    """The link's raw per-direction rate in GB/s from its generation and width (after line encoding)."""
    gt = {1: 2.5, 2: 5.0, 3: 8.0, 4: 16.0, 5: 32.0, 6: 64.0}.get(link.get("gen", 0), 0.0)
    enc = 0.8 if link.get("gen", 0) <= 2 else (242 / 256 if link.get("gen", 0) >= 6 else 128 / 130)
    return gt * link.get("width", 0) * enc / 8.0


def link_reference(device: int, bus_id: str, link: dict) -> dict:
    """An independent ceiling beside the same-run probe: the link's raw rate
    from its generation and width, and the TLP-payload bound from the max
    payload size (lspci); nvbandwidth when installed."""
    raw = raw_link_gbs(link)
    out = {"raw_gbs_per_direction": raw, "gen": link.get("gen"), "width": link.get("width")}
    try:
        txt = subprocess.run(["lspci", "-vvv", "-s", bus_id], capture_output=True, text=True, timeout=10).stdout
        import re
        m = re.search(r"DevCtl:.*?MaxPayload (\d+) bytes, MaxReadReq (\d+) bytes", txt, re.S)
        if m:
            mps, mrrs = int(m.group(1)), int(m.group(2))
            # per TLP: 4 B framing + 2 B sequence + 16 B header (64-bit address) + 4 B LCRC
            out.update(max_payload=mps, max_read_request=mrrs, tlp_payload_bound_gbs_per_direction=raw * mps / (mps + 26))
    except (OSError, subprocess.SubprocessError):
        pass
    import shutil
    out["nvbandwidth"] = "present" if shutil.which("nvbandwidth") else "absent from the image"
    return out


def topo_matrix() -> list:
    try:
        return subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True, timeout=20).stdout.strip().splitlines()
    except (OSError, subprocess.SubprocessError):
        return []


def pct(vals, q):
    s = sorted(vals)
    if not s:
        return None
    k = (len(s) - 1) * q
    lo = int(k)
    hi = min(lo + 1, len(s) - 1)
    return s[lo] + (s[hi] - s[lo]) * (k - lo)


def settle_host_link(eng, limit_s: float = 45.0) -> dict:
    """Before warm-up: short bidirectional CE probes until two consecutive
    readings agree within 3% at the link's level, i.e. the last one within 5%
    of the best reading so far (host-side background work, e.g. reclaim after
    a large free, or a neighbour's burst, has passed; two low readings that
    agree are a burst still running), at most `limit_s`. The readings are
    reported, and the run goes ahead after `limit_s` either way."""
    t0 = time.perf_counter()
    readings = []
    while time.perf_counter() - t0 < limit_s:
        readings.append(round(eng.probe_pcie(256 * MIB, 64 * MIB)["ce_bidir_total"], 2))
        if (len(readings) >= 2 and abs(readings[-1] - readings[-2]) <= 0.03 * readings[-1]
                and readings[-1] >= 0.95 * max(readings)):
            break
    return {"readings_gbps": readings, "secs": round(time.perf_counter() - t0, 2), "settled": len(readings) >= 2 and
            abs(readings[-1] - readings[-2]) <= 0.03 * readings[-1] and readings[-1] >= 0.95 * max(readings)}


def pinned_budget_for(dist: "Dist") -> int:
    """Config 2's pinned budget per rank: 16 GiB, the workload's figure. Each
    rank pins it plus ~2 GiB of probe and bounce buffers; when the host cannot
    hold that for every rank on the node, the budget shrinks (to no less than
    the 8.5 GiB the steady state needs: the victim's 8 GiB share plus the
    512 MiB streaming window) rather than drive the host out of memory. The
    bytes per switch do not change; the line reports the budget used."""
    try:
        with open("/proc/meminfo") as f:
            avail = {ln.split(":")[0]: int(ln.split()[1]) * 1024 for ln in f}.get("MemAvailable", 0)
    except OSError:
        return 16 * GIB
    per_node = int(os.environ.get("LOCAL_WORLD_SIZE", str(dist.world)))
    if not avail or avail >= per_node * 20 * GIB:
        return 16 * GIB
    fit = (avail // per_node - 3 * GIB) // (512 * MIB) * (512 * MIB)
    if fit < 17 * GIB // 2:
        raise SystemExit(f"bench: {per_node} ranks need >= {per_node * 11.5:.0f} GiB of host memory, "
                         f"{avail / GIB:.0f} GiB available")
    return int(fit)


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def ncu_traffic() -> dict:
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
    except OSError:
        return {}
    return d.get("current", d)  # the capture of the current build (older rounds keyed by round)


# ---------------------------------------------------------------------------------------------
# CPU baseline: the reference's own path on the host cores (bounded sample)
# ---------------------------------------------------------------------------------------------
def cpu_baseline(sample_switches: int = 2) -> dict:
    """Reference control path (unmodified reference library: plan_switch +
    execute, single-threaded by design) for the workload's switches, plus the
    switch's bytes moved by host memcpy on all host cores (the reference
    models no data; the paper's daemon copies with multiple host threads)."""
    ref = os.path.join(ROOT, "oracle", "_ref", "ref_trace")
    so = os.path.join(ROOT, "oracle", "_ref", "libswap_oracle.so")
    scn = os.path.join(ROOT, "paper_2601_11743_b200", "scenarios", "c2_interactive_background.scn")
    out = {"kind": "reference", "unit": "GB/s"}
    if not (os.path.exists(ref) and os.path.exists(so)):
        out.update(value=None, cores=0, sample="oracle/_ref not built")
        return out
    p = subprocess.run([ref, "--bench", scn, str(sample_switches)], capture_output=True, text=True, timeout=600)
    ctl_s, ctl_bytes = p.stdout.split()
    ctl_s, ctl_bytes = float(ctl_s), int(ctl_bytes)
    # Byte movement: each switch copies bytes_in + bytes_out; sample one
    # switch's worth (16 GiB) as 2 MiB blocks between two host buffers.
    lib = ctypes.CDLL(so)
    lib.so_copy_blocks.restype = ctypes.c_double
    lib.so_copy_blocks.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_int]
    cores = os.cpu_count() or 1
    per_switch = ctl_bytes // max(1, sample_switches)
    pool_bytes = min(per_switch, 4 * GIB)  # reuse a 4 GiB pool: bounded memory, same memcpy work
    nblk = pool_bytes // (2 * MIB)
    src = ctypes.create_string_buffer(pool_bytes)
    dst = ctypes.create_string_buffer(pool_bytes)
    ctypes.memset(src, 1, pool_bytes)
    ctypes.memset(dst, 2, pool_bytes)
    sp = (ctypes.c_void_p * nblk)(*[ctypes.addressof(src) + i * 2 * MIB for i in range(nblk)])
    dp = (ctypes.c_void_p * nblk)(*[ctypes.addressof(dst) + i * 2 * MIB for i in range(nblk)])
    reps = max(1, per_switch // pool_bytes)
    copy_s = sum(lib.so_copy_blocks(dp, sp, nblk, cores) for _ in range(reps)) * (per_switch / (reps * pool_bytes))
    per_switch_s = ctl_s / sample_switches + copy_s
    out.update(value=per_switch / per_switch_s / 1e9, cores=cores,
               sample=(f"{sample_switches} steady switches of the workload through the unmodified reference "
                       f"(plan_switch+execute, 1 thread: {ctl_s / sample_switches * 1e3:.1f} ms/switch) + one switch's "
                       f"{per_switch / GIB:.0f} GiB moved by memcpy on {cores} threads ({copy_s:.2f} s)"),
               ms_per_switch=per_switch_s * 1e3)
    return out


def run_reference(args, dist: Dist):
    if dist.rank != 0:
        return 0
    t0 = time.perf_counter()
    vals = []
    base = None
    for _ in range(args.warmup + args.steps):
        base = cpu_baseline(1)
        vals.append(base["value"])
    vals = vals[args.warmup:] if vals and vals[0] is not None else vals
    v = statistics.mean(vals) if vals and vals[0] is not None else None
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": base.get("ms_per_switch") if base else None, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOAD, "parallelism": "host cores (reference is single-threaded; memcpy on all cores)"},
            "cpu_baseline": {**(base or {}), "value": v},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t0}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
# Product arm
# ---------------------------------------------------------------------------------------------
def sm_path_switches(eng, step, n: int, path: int) -> dict:
    """The hand-written SM copy path on the same steady config-2 switches,
    after the timed region (not part of `value`): the engine's copy path is
    set to the SM kernel (K1T, the TMA pipeline on half the SMs) for `n`
    switches, every restore checksum-verified, then set back. DESIGN.md §3:
    the copy engines win on this link, which is why `calibrate()` keeps them."""
    eng.set_option("path", 1)
    try:
        sts = [step() for _ in range(n)]
    finally:
        eng.set_option("path", int(path))
    spans = [s["device_span_s"] for s in sts]
    gbs = [(s["bytes_in"] + s["bytes_out"]) / s["device_span_s"] / 1e9 for s in sts]
    return {"kernel": "K1T nx_swap_tma_kernel (cp.async.bulk ring, checksum fused; half the SMs per launch)",
            "switches": n, "gbs_p50": statistics.median(gbs), "device_span_ms_p50": statistics.median(spans) * 1e3,
            "mismatches": sum(s["mismatches"] for s in sts), "verified": sum(s["verified"] for s in sts),
            "k1_launches": sum(s["k1_launches"] for s in sts),
            "what": "same engine and workload as `value`, copy path forced to the SM kernel after the timed region"}


def x16_exchange(path: int, probes: list, switches: int = 20) -> dict:
    """North-star latency case: 16 GiB <-> 16 GiB exchange at a 16 GiB cap,
    `switches` times. Ideal = max(bytes / H2D-while-bidirectional, bytes /
    D2H-while-bidirectional) from the same-run probes, the
    most demanding of the probed shapes."""
    from paper_2601_11743_b200 import PlannerConfig, SwapEngine
    from paper_2601_11743_b200._lib import TIER_GPU, TIER_PINNED
    e = SwapEngine(gpu_capacity=16 * GIB, pinned_capacity=34 * GIB, paged_capacity=2 * GIB, path=path)
    try:
        e.allocate(0, 16 * GIB, TIER_GPU)
        e.allocate(1, 16 * GIB, TIER_PINNED)
        e.fill_pattern(0, 1)
        e.fill_pattern(1, 1)
        lat, dev = [], []
        nxt = 1
        for _ in range(switches):
            c0 = time.perf_counter()
            st = e.switch_to(nxt, PlannerConfig(victim_order=[1 - nxt]))
            lat.append(time.perf_counter() - c0)  # the whole public call
            assert st["mismatches"] == 0
            dev.append(st["device_span_s"])
            nxt = 1 - nxt
        bad = e.verify_pattern(0, 1) + e.verify_pattern(1, 1)
    finally:
        e.close()
    ideal = min(max(16 * GIB / (p["ce_bidir_h2d"] * 1e9), 16 * GIB / (p["ce_bidir_d2h"] * 1e9)) for p in probes)
    return {"bytes_each_way": 16 * GIB, "n": len(lat), "ideal_s": ideal,
            "p50_s": pct(lat, 0.5), "p99_s": pct(lat, 0.99), "max_s": max(lat),
            "p50_over_ideal": pct(lat, 0.5) / ideal, "p99_over_ideal": pct(lat, 0.99) / ideal, "target_over_ideal": 1.2,
            "device_span_p50_s": pct(dev, 0.5), "latency_s": [round(x, 4) for x in lat], "byte_exact": bad == 0}


def uvm_comparator(x16: dict | None, rounds: int = 2) -> dict:
    """The UVM comparator on the same exchange (reference
    claim Nixie/UVM ~2x): two 16 GiB
    cudaMallocManaged working sets round-robin on 17 GiB of usable device
    memory (tests/apps/uvm_rr.cu), fault-driven. Switch cost = kernel time
    with the other app resident minus the resident kernel time."""
    exe = os.path.join(ROOT, "paper_2601_11743_b200", "lib", "nx_uvm_rr")
    p = subprocess.run([exe, "--cap-gib", "17", "--ws-gib", "16", "--rounds", str(rounds), "--prefetch", "0"],
                       capture_output=True, text=True, timeout=600)
    try:
        d = json.loads(p.stdout.strip().splitlines()[-1])
    except (ValueError, IndexError):
        return {"error": (p.stderr or p.stdout)[-300:]}
    out = {"what": "cudaMallocManaged round-robin, 16 GiB <-> 16 GiB, demand faults (tests/apps/uvm_rr.cu)",
           "switch_ms_median": d["median_ms"], "switch_ms": d["switch_cost_ms"], "byte_exact": d.get("mismatches") == 0,
           "host_peak_rss_bytes": d.get("host_peak_rss_bytes")}
    if x16 and x16.get("p50_s"):
        out["engine_switch_ms_p50"] = x16["p50_s"] * 1e3
        out["engine_speedup"] = d["median_ms"] / (x16["p50_s"] * 1e3)
        out["reference_claim"] = "~2x (SPEC.md:563, PAPER.md:313)"
    return out


def interposer_c2(timeout_s: float = 240.0) -> dict:
    """The same workload (config 2) through the deployment path: two unmodified
    CUDA programs (16 + 24 GiB vecapps) under nixied + LD_PRELOAD shim on the
    32 GiB budget (tools/interposer_bench.py). Steady switches exchange 8 GiB
    each way; GB/s = both directions' bytes over the daemon's copy time."""
    for attempt in range(2):
        p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "interposer_bench.py"), "--iters", "10"],
                           capture_output=True, text=True, timeout=timeout_s)
        try:
            d = json.loads(p.stdout.strip().splitlines()[-1])
        except (ValueError, IndexError):
            return {"error": (p.stderr or p.stdout)[-300:]}
        # The scheduler decides when the apps alternate; a run where one app
        # finished before the other started competing has no steady switches.
        if (d.get("steady_switches") or 0) >= 5:
            break
    return {"value": d.get("copy_bidir_gbps_median"), "unit": "GB/s", "switch_ms": d.get("switch_total_ms"),
            "warmup_switch_ms": d.get("warmup_switch_ms"),
            "grant_ms_median": d.get("grant_ms_median"), "steady_switches": d.get("steady_switches"),
            "verified": d.get("verified"), "mismatches": d.get("mismatches"), "apps_ok": d.get("apps_ok"),
            "apps": "2 unmodified CUDA programs (tests/apps/vecapp.cu) under lib/nixied + LD_PRELOAD lib/libnixie_shim.so"}


def aggregate(ranks: list, steps: int) -> dict:
    """Whole-job numbers from the per-rank records (rank 0, after a gather).
    value: bytes of all ranks / device time, where the device time is the sum
    over steps of the slowest rank's CUDA-event span of that step (at N > 1
    every step starts on a barrier, so the ranks' switches overlap and the
    per-step max is the concurrent time). window: bytes / the sum over steps
    of (last rank's end - first rank's start) on the shared host clock, which
    also counts host gaps. e2e: bytes / the slowest rank's wall time of the
    timed public-API calls."""
    total = sum(r["bytes"] for r in ranks)
    dev = sum(max(r["spans"][i] for r in ranks) for i in range(steps))
    window = sum(max(r["windows"][i][1] for r in ranks) - min(r["windows"][i][0] for r in ranks) for i in range(steps))
    wall = max(r["wall_s"] for r in ranks)
    return {"total_bytes": total, "dev_max_s": dev, "window_s": window, "wall_max_s": wall,
            "value": total / dev / 1e9, "e2e": total / wall / 1e9,
            "window_gbs": total / window / 1e9 if window > 0 else None, "bad": sum(r["bad"] for r in ranks)}


def run_product(args, dist: Dist):
    from paper_2601_11743_b200 import PlannerConfig, SwapEngine, parse_path
    from paper_2601_11743_b200._lib import TIER_GPU, TIER_PINNED, device_info
    from paper_2601_11743_b200 import cuda_device_count
    ndev = max(1, cuda_device_count())
    # One GPU per rank. With fewer visible GPUs than ranks (a functional check
    # of the multi-rank path on a 1-GPU box) ranks share devices and the line
    # says so: its numbers are then not a scaling result.
    device = (dist.local % ndev) if args.gpus > 1 else 0
    shared_device = args.gpus > ndev
    peaks = measured_peaks()
    path = parse_path(args.path)
    pinned_budget = pinned_budget_for(dist)
    info = device_info(device)
    counters = PcieCounters(info["pci_bus_id"])
    extra = {"legs_per_launch": args.legs_per_launch} if args.legs_per_launch else {}
    eng = SwapEngine(device=device, gpu_capacity=32 * GIB, pinned_capacity=pinned_budget, paged_capacity=2 * GIB, path=path,
                     **extra)
    probe = eng.probe_pcie(1 * GIB, 64 * MIB)
    # Large copies lose less to the copy engines' per-call overhead
    # (profiles/r02_ce_bubble.txt: 256 MiB calls 99.6 GB/s vs 2 MiB calls 77):
    # the denominator takes the best shape measured, not the engine's own.
    probe_big = eng.probe_pcie(2 * GIB, 256 * MIB)
    # The engine's own paced shape (D2H held behind landed H2D,
    # EngineConfig::pace_lag_legs) moves more bytes per second than either
    # free-running shape on these links (profiles/r02_pcie_pace.txt), so it
    # is in the denominator too.
    probe_paced = max((eng.probe_pcie_paced(2 * GIB, c * MIB, k) for c, k in ((64, 2), (32, 3))),
                      key=lambda p: p["ce_bidir_total"])
    calib = eng.calibrate(256 * MIB) if path == 0 else None
    # Steady state only involves the GPU and the pinned ring, so the apps are
    # placed directly (no pageable cold start): the interactive app on the
    # GPU, the background app's 24 GiB as 16 GiB on the GPU + 8 GiB pinned.
    eng.allocate(0, 16 * GIB, TIER_GPU)
    eng.allocate(1, 16 * GIB, TIER_GPU)
    eng.allocate(1, 8 * GIB, TIER_PINNED)
    seed = 0x4E495849
    eng.fill_pattern(0, seed)
    eng.fill_pattern(1, seed)
    pc = PlannerConfig(streaming_window=512 * MIB, pinned_budget=pinned_budget)
    nxt = 0

    def step():
        nonlocal nxt
        pc.victim_order = [1 - nxt]
        c0 = time.perf_counter()
        st = eng.switch_to(nxt, pc)
        st["call_s"] = time.perf_counter() - c0  # the whole public call, as the application sees it
        nxt = 1 - nxt
        return st

    settle = settle_host_link(eng)
    for _ in range(max(3, args.warmup)):  # W warm-up switches (the first reaches the steady 8 <-> 8 GiB state)
        step()
    launches0 = eng.total_launches()
    sampler = ClockSampler(device)
    sampler.start()
    dist.barrier()
    counters.start()
    t0 = time.perf_counter()
    stats, windows = [], []
    for _ in range(args.steps):
        if dist.world > 1:
            dist.barrier()  # every rank switches at once: a common window per step
        w0 = time.time()
        stats.append(step())
        windows.append((w0, time.time()))
    wall = time.perf_counter() - t0
    lk = pcie_link(device)  # the idle link may have trained down already: bound by its maximum
    pcie = counters.stop(raw_link_gbs({"gen": lk.get("gen_max", 0), "width": lk.get("width_max", 0)}))
    dist.barrier()
    clocks = sampler.stop()
    launches = eng.total_launches() - launches0
    # Latency distribution: >= --latency-switches steady switches (the timed
    # ones included), independent of --steps (p50/p99 over >= 100).
    more = [step() for _ in range(max(0, args.latency_switches - args.steps))]
    sm_path = None
    if args.sm_switches > 0:
        try:
            sm_path = sm_path_switches(eng, step, args.sm_switches, path)
        except Exception as e:  # noqa: BLE001  (reported, never fatal to the bench line)
            sm_path = {"error": str(e)[-300:]}
    probe_after = eng.probe_pcie(1 * GIB, 64 * MIB)
    pinned_now, pinned_peak = eng.pinned_physical()
    pinned_extra = eng.pinned_overhead()
    bad = eng.verify_pattern(0, seed) + eng.verify_pattern(1, seed)
    eng.audit()
    eng.close()

    bytes_rank = sum(s["bytes_in"] + s["bytes_out"] for s in stats)
    dev_rank = sum(s["device_span_s"] for s in stats)
    lat = [s["call_s"] * 1e3 for s in stats + more]
    dev_lat = [s["device_span_s"] * 1e3 for s in stats + more]
    peak_rank = max(probe["ce_bidir_total"], probe["sm_bidir_total"], probe_after["ce_bidir_total"], probe_after["sm_bidir_total"],
                    probe_big["ce_bidir_total"], probe_paced["ce_bidir_total"])
    rank_rec = {"rank": dist.rank, "device": device, **info, "gbs": bytes_rank / dev_rank / 1e9, "pcie_peak_gbs": peak_rank,
                "pct_of_own_peak": bytes_rank / dev_rank / 1e9 / peak_rank * 100.0, "windows": windows,
                "bytes": bytes_rank, "dev_s": dev_rank, "wall_s": wall, "bad": bad,
                "spans": [s["device_span_s"] for s in stats]}
    ranks = dist.gather(rank_rec)
    x16 = x16_exchange(path, [probe, probe_big, probe_paced], args.x16_switches) if (args.x16 and dist.rank == 0) else None
    ip = None
    if args.interposer and args.gpus == 1 and dist.rank == 0:
        try:
            ip = interposer_c2()
        except Exception as e:  # noqa: BLE001  (reported, never fatal to the bench line)
            ip = {"error": str(e)[-300:]}
    uvm = None
    if args.uvm and dist.rank == 0 and args.gpus == 1:
        try:
            uvm = uvm_comparator(x16)
        except Exception as e:  # noqa: BLE001
            uvm = {"error": str(e)[-300:]}
    if dist.rank != 0:
        return 0

    agg = aggregate(ranks, args.steps)
    total_bytes, dev_max, wall_max, window = agg["total_bytes"], agg["dev_max_s"], agg["wall_max_s"], agg["window_s"]
    bad_all = agg["bad"]
    value = agg["value"]
    e2e = agg["e2e"]
    # Denominator: the better of the probes right before and right after the
    # timed region (shared hosts: neighbours' DRAM/PCIe load moves both).
    pcie_peak = peak_rank
    per_gpu = value / args.gpus
    k3_s = sum(s["k3_s"] for s in stats)
    k3_busy = sum(s["k3_busy_s"] for s in stats)
    k3_kernel = sum(s["k3_kernel_s"] for s in stats)
    k3_b = sum(s["k3_bytes"] for s in stats)
    k1_s = sum(s["k1_s"] for s in stats)
    k1_b = sum(s["k1_bytes"] for s in stats)
    k3_n = sum(s["k3_launches"] for s in stats)
    k1_n = sum(s["k1_launches"] for s in stats)
    traffic = ncu_traffic()
    if k1_s > k3_s:  # SM swap kernel dominates: PCIe-bound
        roof = {"kernel": "nx_swap_kernel (K1, fused checksum)", "bound": "pcie", "achieved": k1_b / k1_s / 1e9,
                "peak": pcie_peak, "unit": "GB/s", "launches": k1_n, "bytes_per_launch": k1_b / max(1, k1_n),
                "avg_launch_ms": k1_s / max(1, k1_n) * 1e3, "traffic": traffic.get("k1_dram_bytes_per_launch"),
                "peak_source": "same-run CE simultaneous H2D+D2H probe"}
    else:  # copy engines move the bytes; K3 checksum kernel reads HBM
        hbm = peaks.get("hbm_gbs", 6650.0)
        # K3 (TMA checksum pipeline over a device-resident leg table): one
        # switch-wide record launch for the departures plus grouped arrival
        # checks, all on one stream; achieved = bytes over the union of the
        # launch intervals (CUDA events on that stream).
        ratio = traffic.get("k3_dram_bytes_per_algorithmic_byte")
        roof = {"kernel": "nx_checksum_tma_kernel<SwapParamsTable> (K3 grouped record/verify)", "bound": "hbm",
                "achieved": k3_b / k3_busy / 1e9 if k3_busy else 0.0,
                "achieved_per_launch_avg": k3_b / k3_s / 1e9 if k3_s else 0.0,
                # in-kernel %globaltimer spans (first CTA start .. last CTA end): excludes
                # the stream/front-end delays the events include
                "achieved_kernel_clock": k3_b / k3_kernel / 1e9 if k3_kernel else None,
                "peak": hbm, "unit": "GB/s", "launches": k3_n, "bytes_per_launch": k3_b / max(1, k3_n),
                "avg_launch_ms": k3_s / max(1, k3_n) * 1e3, "busy_ms_per_step": k3_busy / args.steps * 1e3,
                "share_of_step": k3_busy / dev_rank if dev_rank else None,
                # ncu --set full (profiles/ncu_summary.json): DRAM bytes per
                # algorithmic byte of the K3 launches captured, scaled to this run's launches
                "traffic": ratio * k3_b / max(1, k3_n) if ratio else None,
                "traffic_source": traffic.get("source"),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"}
    roof["frac"] = roof["achieved"] / roof["peak"] if roof["peak"] else None
    base = cpu_baseline(2)
    st0 = stats[0]
    # Ideal switch: bytes / per-direction rate with the other direction
    # saturated, for each probed shape; the most demanding (smallest) one.
    ideal_ms = min(max(st0["bytes_in"] / (p["ce_bidir_h2d"] * 1e9), st0["bytes_out"] / (p["ce_bidir_d2h"] * 1e9)) * 1e3
                   for p in (probe, probe_big, probe_paced))
    link = pcie_link(device)
    alg_in = sum(s["bytes_in"] for s in stats)
    alg_out = sum(s["bytes_out"] for s in stats)
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dev_max / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic (splitmix64 pattern per 2 MiB block; every restore checksummed)",
        "config": {"workload": WORKLOAD, "gpu_cap_gib": 32, "pinned_budget_gib": pinned_budget / GIB, "apps_gib": [16, 24],
                   "bytes_per_step": bytes_rank / args.steps, "path": args.path,
                   "l2": "inputs (8 GiB per direction per step) far exceed the 126 MB L2",
                   "parallelism": f"{args.gpus} independent per-GPU instances, no collectives"},
        "per_gpu_gbps": per_gpu, "pct_of_pcie_peak": per_gpu / pcie_peak * 100.0,
        "switch_latency_ms": {"n": len(lat), "p50": pct(lat, 0.5), "p99": pct(lat, 0.99), "min": min(lat), "max": max(lat),
                              "ideal": ideal_ms, "p50_over_ideal": pct(lat, 0.5) / ideal_ms,
                              "p99_over_ideal": pct(lat, 0.99) / ideal_ms,
                              "device_span_p50": pct(dev_lat, 0.5), "device_span_p99": pct(dev_lat, 0.99),
                              "what": "host wall of the public call per steady switch (SwapEngine.switch_to through the C ABI: "
                                      "plan_switch + execute + commits + status read-back + stats); device span = first PCIe "
                                      "batch start .. last check end"},
        "ideal_latency_ms": ideal_ms,
        "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": alg_in / args.steps,
                "d2h_bytes_per_step": alg_out / args.steps},
        "roofline": roof,
        "link_roofline": {"bound": "pcie", "achieved": per_gpu, "peak": pcie_peak, "unit": "GB/s", "frac": per_gpu / pcie_peak,
                          "link": link, "peak_source": "same-run probes, best of: CE and SM at 1 GiB/direction in 64 MiB "
                                                       "calls before and after the timed region, CE at 2 GiB/direction in 256 MiB calls, "
                                                       "CE paced (D2H chunk i after H2D chunk i-k landed) at 2 GiB/direction in "
                                                       "64 MiB (k=2) and 32 MiB (k=3) calls"},
        "link_reference": link_reference(device, info["pci_bus_id"], link),
        "pcie_counters": {**pcie, **({"rx_over_algorithmic_h2d_rate": pcie["rx_gbs_mean"] / (alg_in / wall / 1e9),
                                      "tx_over_algorithmic_d2h_rate": pcie["tx_gbs_mean"] / (alg_out / wall / 1e9)}
                                     if pcie.get("available") else {})},
        "pcie_probe": {k: (round(v, 2) if isinstance(v, float) else v) for k, v in probe.items()},
        "pcie_probe_256mib": {k: round(probe_big[k], 2) for k in ("ce_bidir_total", "ce_bidir_h2d", "ce_bidir_d2h", "ce_h2d", "ce_d2h")},
        "pcie_probe_paced": {k: (round(v, 2) if isinstance(v, float) else v) for k, v in probe_paced.items()},
        "pcie_probe_after": {k: round(probe_after[k], 2) for k in ("ce_bidir_total", "ce_bidir_h2d", "ce_bidir_d2h", "sm_bidir_total")},
        "settle": settle,
        "calibration": calib,
        "sm_path": sm_path,
        # The paper's own data mechanism restated on the box (SURVEY.md §8d CPU-baseline item 2):
        # one cudaMemcpyAsync per 2 MiB block on two streams, both directions at once.
        "paper_mechanism_2mib_ce": ({"gbs": round(calib["ce_gbps"][0], 2), "what": "per-2 MiB cudaMemcpyAsync, one D2H and one "
                                     "H2D stream (calibrate(), 1 leg per call)", "engine_over_it": round(per_gpu / calib["ce_gbps"][0], 3)}
                                    if calib else None),
        "cpu_baseline": base,
        "gpu_launches": launches,
        "clocks": clocks,
        "byte_exact": bad_all == 0,
        "verified_restores": sum(s["verified"] for s in stats),
        "pinned": {"budget_bytes": 16 * GIB, "ring_bytes": 16 * GIB, "physical_peak_bytes": pinned_peak,
                   "out_of_budget_bytes": pinned_extra,
                   "out_of_budget_what": "128 MiB bounce buffer for pageable fills/compares (not on the swap path) + pinned "
                                         "stages of the K3 leg table and the frame table; probes allocate and free their own"},
        "x16_exchange": x16,
        "uvm": uvm,
        "interposer": ip,
        "multi_gpu": {"ranks": [{k: v for k, v in r.items() if k not in ("windows", "spans")} for r in ranks],
                      "concurrent_window_gbs": agg["window_gbs"],
                      "concurrent_window_what": "sum of bytes over ranks / sum over steps of (last rank's end - first "
                                                "rank's start), host clock, steps barrier-aligned at N > 1",
                      "topo": topo_matrix()},
        "shared_device": shared_device,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["product", "reference"], default="product")
    ap.add_argument("--path", choices=["auto", "sm", "ce"], default="auto")
    ap.add_argument("--no-x16", dest="x16", action="store_false")
    ap.add_argument("--x16-switches", type=int, default=20)
    ap.add_argument("--sm-switches", type=int, default=4,
                    help="steady switches on the SM copy kernel (K1T) after the timed region, reported as sm_path (0: skip)")
    ap.add_argument("--latency-switches", type=int, default=100,
                    help="steady switches sampled for p50/p99 (the timed ones included)")
    ap.add_argument("--no-uvm", dest="uvm", action="store_false", help="skip the cudaMallocManaged comparator")
    ap.add_argument("--legs-per-launch", type=int, default=0, help="CE batch / K3 launch size (0: engine default)")
    ap.add_argument("--no-interposer", dest="interposer", action="store_false",
                    help="skip the config-2 run through nixied + the LD_PRELOAD shim")
    args = ap.parse_args()
    dist = Dist()
    try:
        if args.impl == "reference":
            return run_reference(args, dist)
        return run_product(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    sys.exit(main())
