"""Does the host buffer size change the bidirectional link rate? (IOMMU /
host-DRAM locality check for the 16 GiB pinned ring.) Free-running and paced
copy-engine probes at 1..8 GiB per direction, alternating, best of 3 each."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_11743_b200 import GIB, MIB, SwapEngine  # noqa: E402

e = SwapEngine(gpu_capacity=2 * GIB, pinned_capacity=64 * MIB, paged_capacity=64 * MIB)
for rep in range(2):
    for g in (1, 2, 4, 8):
        free = e.probe_pcie(g * GIB, 64 * MIB)
        paced = e.probe_pcie_paced(g * GIB, 64 * MIB, 2)
        print(json.dumps({"rep": rep, "gib_per_direction": g, "free_64mib": round(free["ce_bidir_total"], 2),
                          "free_h2d": round(free["ce_bidir_h2d"], 2), "free_d2h": round(free["ce_bidir_d2h"], 2),
                          "paced_64mib": round(paced["ce_bidir_total"], 2), "paced_h2d": round(paced["ce_bidir_h2d"], 2),
                          "paced_d2h": round(paced["ce_bidir_d2h"], 2)}), flush=True)
e.close()
