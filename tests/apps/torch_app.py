"""An ordinary PyTorch program used to test the interposer: it allocates
device tensors, runs elementwise kernels, synchronises, thinks, and checks
its tensors at the end. It knows nothing about Nixie (run it with
LD_PRELOAD=libnixie_shim.so NIXIE_SOCKET=...). Prints one JSON line."""
import json
import sys
import time

import torch


def main():
    mib = float(sys.argv[1]) if len(sys.argv) > 1 else 1024
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    think = float(sys.argv[3]) if len(sys.argv) > 3 else 0.2
    bufs = 4
    n = int(mib * (1 << 20) / 4 / bufs)
    free_b, total_b = torch.cuda.mem_get_info()
    xs = [torch.full((n,), k * 1000, dtype=torch.int32, device="cuda") for k in range(bufs)]
    # cuBLAS work: its kernels reach the driver through cuGetProcAddress, not
    # the runtime's PLT entry points (the shim gates them too).
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(2048, 2048, device="cuda", generator=g)
    b = torch.randn(2048, 2048, device="cuda", generator=g)
    ref = (a @ b).double().sum().item()
    # cuDNN work (convolution through cudnnBackendExecute)
    img = torch.randn(8, 16, 64, 64, device="cuda", generator=g)
    wgt = torch.randn(32, 16, 3, 3, device="cuda", generator=g)
    conv_ref = torch.nn.functional.conv2d(img, wgt, padding=1).double().sum().item()
    mm_bad = 0
    lat = []
    for it in range(iters):
        t0 = time.perf_counter()
        for x in xs:
            x.add_(1)
        c = a @ b
        y = torch.nn.functional.conv2d(img, wgt, padding=1)
        torch.cuda.synchronize()
        mm_bad += int(abs(c.double().sum().item() - ref) > 1e-6 * max(1.0, abs(ref)))
        mm_bad += int(abs(y.double().sum().item() - conv_ref) > 1e-6 * max(1.0, abs(conv_ref)))
        lat.append((time.perf_counter() - t0) * 1e3)
        time.sleep(think)
    bad = 0
    for k, x in enumerate(xs):
        bad += int((x != k * 1000 + iters).sum().item())
    print(json.dumps({"name": "torch_app", "bytes": n * 4 * bufs, "iters": iters, "mismatch": bad, "matmul_mismatch": mm_bad,
                      "memgetinfo": [free_b, total_b], "iter_ms_max": max(lat)}))
    return 0 if bad == 0 and mm_bad == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
