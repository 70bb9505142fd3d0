"""Host-side checks of the interposer (no GPU): the shim exports exactly the
CUDA entry points it interposes (include/nixie_shim.h) and nothing of its
statically linked C++ runtime, is inert without NIXIE_SOCKET, and the daemon
binary parses its command line."""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2601_11743_b200.interpose import NIXIED, SHIM, VECAPP  # noqa: E402

INTERPOSED = {
    "cudaMalloc", "cudaFree", "cudaMallocAsync", "cudaFreeAsync", "cuMemAlloc_v2", "cuMemFree_v2", "cudaMemGetInfo",
    "cudaLaunchKernel", "cudaLaunchKernel_ptsz", "cudaLaunchKernelExC", "cudaLaunchKernelExC_ptsz",
    "cudaLaunchCooperativeKernel", "cudaLaunchCooperativeKernel_ptsz", "cudaGraphLaunch", "cudaGraphLaunch_ptsz",
    "cuLaunchKernel", "cudaMemcpy", "cudaMemcpyAsync", "cudaMemcpyAsync_ptsz", "cudaMemcpy2D", "cudaMemcpy2DAsync",
    "cudaMemset", "cudaMemsetAsync", "cudaMemsetAsync_ptsz",
    "cudaDeviceSynchronize", "cudaStreamSynchronize", "cudaEventSynchronize",
    "cudaStreamBeginCapture", "cudaStreamEndCapture",
    "cublasLtMatmul", "cublasGemmEx", "cublasGemmStridedBatchedEx", "cublasSgemm_v2", "cublasSgemmStridedBatched",
    "cudnnBackendExecute",
    # allocation breadth
    "cudaMallocAsync_ptsz", "cudaMallocPitch", "cudaMalloc3D", "cuMemAllocPitch_v2", "cuMemAllocAsync", "cuMemFreeAsync",
    # implicitly allocating APIs
    "cudaStreamCreate", "cudaStreamCreateWithFlags", "cudaStreamCreateWithPriority", "cudaStreamDestroy",
    "cudaGraphInstantiate", "cudaGraphInstantiateWithFlags", "cudaGraphExecDestroy", "cudaDeviceSetLimit",
    "cuStreamCreate", "cuStreamCreateWithPriority", "cuStreamDestroy_v2", "cublasCreate_v2", "cublasDestroy_v2",
    "cublasLtCreate", "cublasLtDestroy", "cudnnCreate", "cudnnDestroy",
    # every copy / memset that can touch device memory
    "cudaMemcpy_ptds", "cudaMemcpy2D_ptds", "cudaMemcpy2DAsync_ptsz", "cudaMemcpy3D", "cudaMemcpy3D_ptds",
    "cudaMemcpy3DAsync", "cudaMemcpy3DAsync_ptsz", "cudaMemcpyPeer", "cudaMemcpyPeerAsync", "cudaMemcpy3DPeer",
    "cudaMemcpy3DPeer_ptds", "cudaMemcpy3DPeerAsync", "cudaMemcpy3DPeerAsync_ptsz", 
    "cudaMemset_ptds",
    "cudaMemset2D", "cudaMemset2D_ptds", "cudaMemset2DAsync", "cudaMemset2DAsync_ptsz", "cudaMemset3D",
    "cudaMemset3D_ptds", "cudaMemset3DAsync", "cudaMemset3DAsync_ptsz",
    "cuLaunchKernelEx", "cuLaunchCooperativeKernel", "cuGraphLaunch", "cuMemcpy", "cuMemcpyAsync", "cuMemcpyHtoD_v2",
    "cuMemcpyDtoH_v2", "cuMemcpyDtoD_v2", "cuMemcpyHtoDAsync_v2", "cuMemcpyDtoHAsync_v2", "cuMemcpyDtoDAsync_v2",
    "cuMemcpy2D_v2", "cuMemcpy2DUnaligned_v2", "cuMemcpy2DAsync_v2", "cuMemcpy3D_v2", "cuMemcpy3DAsync_v2",
    "cuMemcpyPeer", "cuMemcpyPeerAsync", "cuMemsetD8_v2", "cuMemsetD16_v2", "cuMemsetD32_v2", "cuMemsetD8Async",
    "cuMemsetD16Async", "cuMemsetD32Async", "cuMemsetD2D8_v2", "cuMemsetD2D16_v2", "cuMemsetD2D32_v2",
}


def exported(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return {ln.split()[-1] for ln in out.splitlines() if re.search(r" [TW] ", ln)}


def test_shim_exports_exactly_the_interposed_api():
    syms = exported(SHIM)
    want = INTERPOSED | {"nixie_shim_active", "nixie_shim_app", "dlsym"}
    assert syms == want, sorted(syms ^ want)
    header = open(os.path.join(ROOT, "include", "nixie_shim.h")).read()
    for s in INTERPOSED:
        base = s.replace("_ptsz", "").replace("_ptds", "")
        assert base in header, f"{s} not documented in include/nixie_shim.h"


def test_shim_is_inert_without_a_daemon():
    code = ("import ctypes, os; os.environ.pop('NIXIE_SOCKET', None); "
            f"s = ctypes.CDLL({SHIM!r}); s.nixie_shim_app.restype = ctypes.c_uint; "
            "print(s.nixie_shim_active(), s.nixie_shim_app())")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    assert out.stdout.split() == ["0", str(0xFFFFFFFF)]


def test_daemon_cli():
    r = subprocess.run([NIXIED, "--help"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "--socket" in r.stderr and "--phys-slack" in r.stderr
    r = subprocess.run([NIXIED, "--bogus"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 1
    # --slab-mib is validated as given: no truncation of 1 or 3 into a default or a neighbour
    for bad in ("1", "3", "5", "2048", "x", "64m"):
        r = subprocess.run([NIXIED, "--slab-mib", bad, "--help"], capture_output=True, text=True, timeout=60)
        assert r.returncode == 1 and "power of two" in r.stderr, (bad, r.stderr)
    r = subprocess.run([NIXIED, "--help"], capture_output=True, text=True, timeout=60)
    assert "--trace" in r.stderr


def test_test_app_links_the_shared_runtime():
    """LD_PRELOAD can only interpose a dynamically linked CUDA runtime."""
    out = subprocess.run(["readelf", "-d", VECAPP], capture_output=True, text=True, check=True).stdout
    assert "libcudart.so" in out


def test_placement_unit_tests():
    """SlabPlacer (daemon) and RangeAlloc (shim) host-only unit tests."""
    exe = os.path.join(ROOT, "paper_2601_11743_b200", "lib", "nx_unit_tests")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
