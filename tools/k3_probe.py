import ctypes, sys
sys.path.insert(0, '.')
from paper_2601_11743_b200 import SwapEngine, MIB
from paper_2601_11743_b200._lib import lib, check
e = SwapEngine(gpu_capacity=64 * MIB, pinned_capacity=64 * MIB, paged_capacity=64 * MIB)
us = (ctypes.c_double * 16)()
for load in (0, 1):
    print("under PCIe load" if load else "idle link")
    check(lib.nx_probe_checksum_launch_ex(e._h, load, us))
    for k in range(8):
        n = 1 << k
        mb = n * 2.097152
        print(f"legs {n:4d}: TMA {us[2*k]:8.2f} us ({mb/us[2*k]:.2f} TB/s)   {'GRAPH' if load else 'LDG'} {us[2*k+1]:8.2f} us ({mb/us[2*k+1]:.2f} TB/s)")
