"""Reference-plan parity on the deployment path.

The interposer daemon (csrc/daemon/daemon.cpp) writes every registry mutation
and every executed plan to `--trace`. oracle/_ref/ref_replay replays the trace
on the UNMODIFIED reference (MemState::allocate/free_chunk,
proj/src/mem_model.cpp:48-116), recomputes plan_switch for each plan on the
same state with the same victim order (proj/src/planner.cpp:111-216), and
runs the daemon's plan through the reference executor (transfer.cpp:250-271).

* `--reference-victims`: the daemon's plans must equal the reference's line
  for line, and the real engine's per-lane leg order must equal the
  reference executor's.
* default (slab-aligned victim blocks, SlabPlacer::slab_victims): the
  documented delta. Same bytes in/out and same victim app order per switch;
  the victim blocks may differ. Per-lane order of the daemon's own plan must
  still equal the reference executor's.
"""
import collections
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REPLAY = os.path.join(ROOT, "oracle", "_ref", "ref_replay")

MIB = 1 << 20


def _replay(path):
    if not os.path.exists(REPLAY):
        pytest.skip("oracle/_ref/ref_replay not built (needs /root/reference at build time)")
    p = subprocess.run([REPLAY, path], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr
    return p.stdout.splitlines()


def _by_plan(lines, tags):
    """{k: {tag: [rest-of-line, ...]}} for lines whose first token is in `tags`."""
    out = collections.defaultdict(lambda: collections.defaultdict(list))
    for ln in lines:
        f = ln.split(" ", 2)
        if f[0] in tags and len(f) >= 2:
            out[int(f[1])][f[0]].append(f[2] if len(f) > 2 else "")
    return out


def _daemon_plans(trace_lines):
    plans = {}
    for ln in trace_lines:
        f = ln.split()
        if f and f[0] == "plan":
            plans[int(f[1])] = {"kind": f[2], "app": int(f[3]), "in": int(f[5]), "out": int(f[7])}
    return plans


def compare(trace_path, expect_identical):
    with open(trace_path) as f:
        tl = f.read().splitlines()
    ref = _replay(trace_path)
    mine = _by_plan(tl, ("P", "L", "Q"))
    theirs = _by_plan(ref, ("S", "P", "A", "L", "F"))
    plans = _daemon_plans(tl)
    assert plans and set(plans) <= set(theirs), (sorted(plans), sorted(theirs))
    # prefetch plans (plan_prefetch, planner.cpp:218-242) on the same registry
    prefetches = sorted(int(ln.split()[1]) for ln in tl if ln.startswith("prefetch "))
    for k in prefetches:
        assert mine[k]["Q"] == theirs[k]["F"], f"prefetch plan {k} differs from the reference's"
    differing = 0
    for k, p in sorted(plans.items()):
        s = theirs[k]["S"][0].split()
        assert (int(s[0]), int(s[1]), int(s[2])) == (p["app"], p["in"], p["out"]), (k, p, s)
        a = {ln.split()[0]: ln.split()[1:] for ln in theirs[k]["A"]}
        assert a["ref"] == a.get("daemon", []), (k, a)
        if expect_identical:
            assert mine[k]["P"] == theirs[k]["P"], f"plan {k}: daemon plan differs from the reference's"
        else:
            differing += mine[k]["P"] != theirs[k]["P"]
        # per lane, in start order: the real engine vs the reference executor on the same plan
        lanes = lambda rows: {ln: [r for r in rows if r.split()[0] == ln] for ln in {r.split()[0] for r in rows}}
        assert lanes(mine[k]["L"]) == lanes(theirs[k]["L"]), f"plan {k}: per-lane leg order differs"
    return {"plans": len(plans), "differing_plans": differing, "prefetches": len(prefetches),
            "moved": sum(p["in"] + p["out"] for p in plans.values())}


def test_ref_replay_pins_itself():
    """CPU: a hand-made trace whose daemon plan is the reference's own plan
    replays cleanly (audit passes, lanes come out), and a trace whose chunk
    ids disagree with the reference registry is rejected."""
    import tempfile
    head = ["capacity gpu 8388608", "capacity pinned 8388608", "capacity paged 67108864", "window 2097152",
            "budget 18446744073709551615", "victims reference", "alloc 0 8388608 gpu 0", "alloc 1 4194304 pinned 1",
            "alloc 1 2097152 paged 2", "plan 0 switch 1 in 6291456 out 6291456 victims 0"]
    d = tempfile.mkdtemp()
    t0 = os.path.join(d, "t0.trace")
    with open(t0, "w") as f:
        f.write("\n".join(head) + "\n")
    first = _replay(t0)
    pl = [ln for ln in first if ln.startswith("P 0 ")]
    assert len(pl) == 6 and "A 0 ref 0" in first
    t1 = os.path.join(d, "t1.trace")
    with open(t1, "w") as f:
        f.write("\n".join(head + pl + ["plan 1 switch 0 in 6291456 out 6291456 victims 1"]) + "\n")
    second = _replay(t1)
    assert [ln for ln in second if ln.startswith("P 0 ")] == pl
    assert "A 0 daemon 0" in second
    lanes0 = [ln for ln in second if ln.startswith("L 0 ")]
    assert len(lanes0) == 8  # 4 single-hop fetches/evictions + 2 two-hop moves
    assert "S 1 0 6291456 6291456" in second, second  # block 3 of app 0 never left
    bad = os.path.join(d, "bad.trace")
    with open(bad, "w") as f:
        f.write("\n".join(head[:6] + ["alloc 0 8388608 gpu 7"]) + "\n")
    p = subprocess.run([REPLAY, bad], capture_output=True, text=True)
    assert p.returncode == 1 and "chunk ids" in p.stderr


def _vec(mib, iters, think_ms, seed, name):
    from paper_2601_11743_b200.interpose import VECAPP
    return [VECAPP, "--mib", str(mib), "--buffers", "6", "--iters", str(iters), "--think-ms", str(think_ms),
            "--seed", str(seed), "--name", name]


def _run(mode, tmp_path):
    from paper_2601_11743_b200.interpose import Daemon, run_apps
    trace = str(tmp_path / f"daemon_{mode}.trace")
    extra = ["--trace", trace] + (["--reference-victims"] if mode in ("reference", "prefetch") else [])
    if mode == "prefetch":  # three apps on a small pinned budget: pageable blocks get prefetched
        with Daemon(gpu="4G", pinned="2G", paged="16G", prefetch=True, extra=extra) as d:
            res = run_apps(d, [_vec(2048, 5, 300, 41 + i, "abc"[i]) for i in range(3)], timeout=600)
            for r in res:
                assert r["rc"] == 0, (r["stderr"], d.stderr())
                assert r["out"]["device_errors"] == 0 and r["out"]["host_mismatch"] == 0
            sw = d.switches()
        assert len(sw) >= 3 and all(s["mismatches"] == 0 for s in sw)
        return trace
    with Daemon(gpu="4G", pinned="4G", paged="16G", extra=extra) as d:
        res = run_apps(d, [_vec(3072, 5, 250, 81, "a"), _vec(3072, 5, 250, 82, "b")], timeout=600)
        for r in res:
            assert r["rc"] == 0, (r["stderr"], d.stderr())
            assert r["out"]["device_errors"] == 0 and r["out"]["host_mismatch"] == 0
        sw = d.switches()
    assert len(sw) >= 3 and all(s["mismatches"] == 0 for s in sw)
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        import shutil
        shutil.copy(trace, os.path.join(out, f"daemon_parity_{mode}.trace"))
    return trace


@pytest.mark.gpu
def test_daemon_reference_victims_plans_equal_reference(tmp_path):
    """Two oversubscribed vecapps (2 x 3 GiB, 4 GiB budget) under
    `nixied --reference-victims`: every plan the daemon executed equals the
    reference planner's on the same registry, and the real engine's per-lane
    leg order equals the reference executor's."""
    st = compare(_run("reference", tmp_path), expect_identical=True)
    assert st["plans"] >= 3 and st["moved"] > 4 * 1024 * MIB, st


@pytest.mark.gpu
def test_daemon_slab_victims_documented_delta(tmp_path):
    """Default daemon (slab-aligned victims): per switch the same bytes in and
    out and the same victim app order as the reference planner; blocks may
    differ."""
    st = compare(_run("slab", tmp_path), expect_identical=False)
    assert st["plans"] >= 3 and st["moved"] > 4 * 1024 * MIB, st


@pytest.mark.gpu
def test_daemon_prefetch_plans_equal_reference(tmp_path):
    """`nixied --prefetch --reference-victims`: three apps on a 2 GiB pinned
    budget. Every prefetch plan the daemon started equals the reference's
    plan_prefetch on the replayed registry (prefetch commits are replayed as
    begin_move + commit_move), and every switch plan equals plan_switch."""
    st = compare(_run("prefetch", tmp_path), expect_identical=True)
    assert st["plans"] >= 3 and st["prefetches"] >= 1, st
