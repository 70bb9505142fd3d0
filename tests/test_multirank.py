"""N>1 host logic on CPU: bench.py's per-rank aggregation (barrier, sum of
bytes, max of time) over gloo with world_size 2, as torchrun would launch it.
The swap path itself has no collective: each rank is an independent Nixie
instance."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import json, os, sys
sys.path.insert(0, %r)
import bench
d = bench.Dist()
d.barrier()
r = d.rank
out = {"rank": r, "world": d.world, "sum": d.reduce(10.0 + r, "sum"), "max": d.reduce(1.5 * (r + 1), "max")}
# bench.run_product's aggregation over gathered synthetic per-rank records:
# rank r moves 16 GiB per step in spans of (0.2 + 0.1 r) s, step windows on
# the host clock start 0.01 s apart per rank.
GB = 16 * (1 << 30)
rec = {"rank": r, "bytes": 3 * GB, "spans": [0.2 + 0.1 * r] * 3, "wall_s": 1.0 + r, "bad": 0,
       "windows": [(10.0 * i + 0.01 * r, 10.0 * i + 0.01 * r + 0.25 + 0.1 * r) for i in range(3)]}
ranks = d.gather(rec)
out["gathered"] = [x["rank"] for x in ranks]
out["agg"] = bench.aggregate(ranks, 3)
d.barrier()
d.close()
print(json.dumps(out))
""" % ROOT


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_aggregation_over_gloo():
    port = free_port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER], env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                      text=True))
    outs = []
    for p in procs:
        o, e = p.communicate(timeout=240)
        assert p.returncode == 0, e[-2000:]
        outs.append(json.loads(o.strip().splitlines()[-1]))
    GB = 16 * (1 << 30)
    for o in outs:
        assert o["world"] == 2
        assert o["sum"] == 21.0 and o["max"] == 3.0
        assert o["gathered"] == [0, 1]
        a = o["agg"]
        assert a["total_bytes"] == 6 * GB
        # per step the slower rank (0.3 s) bounds the concurrent device time
        assert abs(a["dev_max_s"] - 0.9) < 1e-9 and abs(a["value"] - 6 * GB / 0.9 / 1e9) < 1e-6
        # common window per step: rank 0 starts at 0.00, rank 1 ends at 0.01 + 0.35
        assert abs(a["window_s"] - 3 * 0.36) < 1e-9
        assert abs(a["e2e"] - 6 * GB / 2.0 / 1e9) < 1e-6 and a["bad"] == 0


def test_reference_arm_nonzero_ranks_exit_cleanly():
    """Under torchrun only rank 0 runs the reference arm; others exit 0."""
    port = free_port()
    env = dict(os.environ, RANK="1", WORLD_SIZE="1", LOCAL_RANK="1", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    # WORLD_SIZE=1 keeps the process group out of the way; rank 1 must print nothing.
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       env=env, capture_output=True, text=True, timeout=240)
    assert p.returncode == 0 and p.stdout.strip() == ""
