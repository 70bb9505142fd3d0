import sys, json
sys.path.insert(0, '.')
from paper_2601_11743_b200 import SwapEngine, GIB, MIB
from paper_2601_11743_b200._lib import lib, check
import ctypes
e = SwapEngine(gpu_capacity=64 * MIB, pinned_capacity=64 * MIB, paged_capacity=64 * MIB)
for variant, ctas_list in ((10, (37, 74, 148)), (11, (37, 74, 148)), (0, (16, 32, 64, 96, 128, 200))):
    for ctas in ctas_list:
        out = (ctypes.c_double * 3)()
        check(lib.nx_probe_copy_variant(e._h, variant, 1 * GIB, ctas, out))
        print(f"variant {variant} ctas {ctas}: h2d {out[0]:.1f} d2h {out[1]:.1f} bidir {out[2]:.1f}", flush=True)
