"""K1 vs K1T in SwapEngine.calibrate(): SM-path vs copy-engine GB/s with both
directions running, per batch size, for the LDG kernel (sm_tma_ctas=0) and
the TMA kernel at a few grid sizes. One JSON line per setting."""
import json
import sys

sys.path.insert(0, ".")
from paper_2601_11743_b200 import GIB, SwapEngine  # noqa: E402

e = SwapEngine(gpu_capacity=2 * GIB, pinned_capacity=1 * GIB, paged_capacity=1 * GIB)
e.probe_pcie(1 * GIB)  # settle
for ctas in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,8,16,32,74").split(",")]:
    e.set_option("sm_tma_ctas", ctas)
    c = e.calibrate()
    print(json.dumps({"sm_tma_ctas": ctas, "legs": c["legs"], "sm_gbps": [round(x, 1) for x in c["sm_gbps"]],
                      "ce_gbps": [round(x, 1) for x in c["ce_gbps"]]}), flush=True)
e.close()
