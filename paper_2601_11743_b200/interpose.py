"""Running unmodified CUDA applications under Nixie (the interposer path).

    with Daemon(gpu="4G", pinned="4G") as d:
        procs = [d.spawn([VECAPP, "--mib", "3072"]) for _ in range(2)]
        ...
    d.records()  # the daemon's JSON-lines log: hello / switch / bye / sched

`Daemon` starts `lib/nixied` (csrc/daemon/daemon.cpp) on a private socket;
`Daemon.spawn` runs a command with `LD_PRELOAD=lib/libnixie_shim.so` and
`NIXIE_SOCKET` set (csrc/shim/shim.cpp), exactly how a user runs an
application under Nixie. Nothing here touches application
data: the daemon moves the bytes, the shim maps and gates.
"""
from __future__ import annotations

import json
import os
import signal
import subprocess
import tempfile
import time
from typing import Dict, List, Optional, Sequence

PKG = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(PKG, "lib")
NIXIED = os.path.join(LIB, "nixied")
SHIM = os.path.join(LIB, "libnixie_shim.so")
VECAPP = os.path.join(LIB, "nx_vecapp")


class Daemon:
    def __init__(self, gpu: str = "32G", pinned: str = "16G", paged: str = "96G", window: Optional[str] = None,
                 path: str = "ce", idle_ms: Optional[float] = None, tick_ms: Optional[float] = None,
                 allot_s: Optional[float] = None, preempt_s: Optional[float] = None, host_threads: Optional[int] = None,
                 log: Optional[str] = None, prefetch: bool = False, slab_mib: Optional[int] = None,
                 extra: Sequence[str] = ()):
        for f in (NIXIED, SHIM):
            if not os.path.exists(f):
                raise RuntimeError(f"{f} is not built (python -c 'import __graft_entry__ as g; g.build()')")
        self.tmp = tempfile.mkdtemp(prefix="nixie-")
        self.sock = os.path.join(self.tmp, "nixie.sock")
        self.log = log or os.path.join(self.tmp, "daemon.jsonl")
        args = [NIXIED, "--socket", self.sock, "--gpu", gpu, "--pinned", pinned, "--paged", paged, "--path", path,
                "--log", self.log]
        for flag, v in (("--window", window), ("--idle-ms", idle_ms), ("--tick-ms", tick_ms), ("--allot-s", allot_s),
                        ("--preempt-s", preempt_s), ("--host-threads", host_threads), ("--slab-mib", slab_mib)):
            if v is not None:
                args += [flag, str(v)]
        self.args = args + (["--prefetch"] if prefetch else []) + list(extra)
        self.proc: Optional[subprocess.Popen] = None
        self.stderr_path = os.path.join(self.tmp, "daemon.err")

    def __enter__(self) -> "Daemon":
        self.start()
        return self

    def __exit__(self, *exc) -> None:
        self.stop()

    def start(self, timeout: float = 120.0) -> None:
        self._err = open(self.stderr_path, "w")
        self.proc = subprocess.Popen(self.args, stdout=self._err, stderr=subprocess.STDOUT, start_new_session=True)
        t0 = time.time()
        while not os.path.exists(self.sock):
            if self.proc.poll() is not None:
                raise RuntimeError(f"nixied exited rc={self.proc.returncode}: {self.stderr()}")
            if time.time() - t0 > timeout:
                self.stop()
                raise RuntimeError("nixied did not come up")
            time.sleep(0.05)

    def stderr(self) -> str:
        try:
            with open(self.stderr_path) as f:
                return f.read()
        except OSError:
            return ""

    def env(self, base: Optional[Dict[str, str]] = None) -> Dict[str, str]:
        e = dict(os.environ if base is None else base)
        e["LD_PRELOAD"] = SHIM + (":" + e["LD_PRELOAD"] if e.get("LD_PRELOAD") else "")
        e["NIXIE_SOCKET"] = self.sock
        return e

    def spawn(self, cmd: List[str], **kw) -> subprocess.Popen:
        return subprocess.Popen(cmd, env=self.env(), stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, **kw)

    def stop(self, timeout: float = 60.0) -> int:
        if self.proc is None:
            return 0
        if self.proc.poll() is None:
            self.proc.send_signal(signal.SIGTERM)
            try:
                self.proc.wait(timeout)
            except subprocess.TimeoutExpired:
                os.killpg(self.proc.pid, signal.SIGKILL)
                self.proc.wait()
        self._err.close()
        rc = self.proc.returncode
        self.proc = None
        return rc

    def records(self) -> List[dict]:
        out = []
        if os.path.exists(self.log):
            with open(self.log) as f:
                for line in f:
                    line = line.strip()
                    if line:
                        out.append(json.loads(line))
        return out

    def switches(self) -> List[dict]:
        return [r for r in self.records() if r.get("event") == "switch"]


def run_apps(daemon: Daemon, cmds: List[List[str]], timeout: float = 600.0, stagger_s: float = 0.0) -> List[dict]:
    """Runs the commands concurrently under the daemon; returns per app
    {rc, out (last JSON line parsed when possible), stderr}."""
    procs = []
    for c in cmds:
        procs.append(daemon.spawn(c))
        if stagger_s:
            time.sleep(stagger_s)
    res = []
    deadline = time.time() + timeout
    for p in procs:
        try:
            out, err = p.communicate(timeout=max(1.0, deadline - time.time()))
        except subprocess.TimeoutExpired:
            p.kill()
            out, err = p.communicate()
        parsed = None
        for line in reversed(out.strip().splitlines()):
            try:
                parsed = json.loads(line)
                break
            except ValueError:
                continue
        res.append({"rc": p.returncode, "out": parsed, "stdout": out, "stderr": err[-4000:]})
    return res
