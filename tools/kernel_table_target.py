"""Every kernel of the library once, for the per-kernel ncu table (PCIe read
and write bytes/s and DRAM GB/s per launch; tools/kernel_table.py builds the
table against the same box's per-direction link peak):
  K4 nx_pattern_kernel        fill (record) and compare of a GPU-resident app
  K1T nx_swap_tma_kernel      SM-path switches with the default kernel
  K1 nx_swap_kernel           SM-path switches with sm_tma_ctas = 0 (split and fused-launch engines;
                              on this full-GPU shape the departures all go out
                              before any fetch, so the launches move one direction)
  K3 nx_checksum_tma_kernel   CE-path switch: grouped record + arrival checks
  nx_table_upload_kernel      the K3 descriptor upload
Shape: 1 GiB on a full 1 GiB GPU exchanged with 1 GiB in the pinned ring.
With --probe (no ncu) it prints the same run's link probe instead."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11743_b200 import GIB, MIB, PlannerConfig, SwapEngine  # noqa: E402
from paper_2601_11743_b200._lib import PATH_CE, PATH_SM, TIER_GPU, TIER_PINNED  # noqa: E402


def exchange(sm_tma_ctas=-1, **opts):
    with SwapEngine(gpu_capacity=1 * GIB, pinned_capacity=2 * GIB, paged_capacity=64 * MIB, **opts) as e:
        e.set_option("sm_tma_ctas", sm_tma_ctas)  # -1: K1T on half the SMs (default), 0: K1
        e.allocate(0, 1 * GIB, TIER_GPU)
        e.allocate(1, 1 * GIB, TIER_PINNED)
        e.fill_pattern(0, 5)  # K4 fill (GPU tier: record on the device)
        e.fill_pattern(1, 5)
        nxt = 1
        for _ in range(2):
            st = e.switch_to(nxt, PlannerConfig(streaming_window=64 * MIB, victim_order=[1 - nxt]))
            assert st["mismatches"] == 0
            nxt = 1 - nxt
        assert e.verify_pattern(0, 5) == 0  # K4 compare
        assert e.verify_pattern(1, 5) == 0


if __name__ == "__main__":
    if "--probe" in sys.argv:
        with SwapEngine(gpu_capacity=64 * MIB, pinned_capacity=64 * MIB, paged_capacity=64 * MIB) as e:
            print(json.dumps(e.probe_pcie(1 * GIB, 64 * MIB)))
        sys.exit(0)
    exchange(path=PATH_SM)                      # K1T split launches (the SM path's default kernel)
    exchange(path=PATH_SM, sm_tma_ctas=0)       # K1 split launches
    exchange(path=PATH_SM, sm_tma_ctas=0, fused_launch=True)   # K1 fused launches
    exchange(path=PATH_CE)                      # K3 + table upload
    print("done")
