"""Per-kernel table from an ncu --metrics CSV (tools/kernel_table_target.py):
for every kernel kind, launches, mean duration, PCIe read/write GB/s and DRAM
GB/s per launch, set against the same box's per-direction link peak (the CE
probe printed by `kernel_table_target.py --probe`) and the link generation.

ncu's pcie__read_bytes / pcie__write_bytes count the GPU's PCIe traffic from
the device's side: read = bytes the GPU read from the host (H2D payload plus
completions), write = bytes it wrote (D2H payload plus read requests).
Under ncu kernels run one at a time, so a split K1 launch has the link to
itself: its rate is set against the one-direction peak; a fused launch
(both directions) against the simultaneous peak.

Usage: python tools/kernel_table.py launches.csv probe.json smi.txt > table.json"""
import collections
import csv
import json
import re
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9,
        "usecond": 1e-6, "msecond": 1e-3, "second": 1, "s": 1}


def load(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[i + 1:]:
        if len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1)
        per[d["ID"]][d["Metric Name"]] = v
        names[d["ID"]] = d["Kernel Name"]
    return per, names


def kind(name, m):
    for k, label in (("nx_swap_tma_kernel", "K1T nx_swap_tma_kernel, "), ("nx_swap_kernel", "K1 nx_swap_kernel, ")):
        if k in name:
            # what the launch moved: one direction or both (fused warp groups)
            rd, wr = m.get("pcie__read_bytes.sum", 0.0), m.get("pcie__write_bytes.sum", 0.0)
            d = "H2D" if wr < 0.25 * rd else ("D2H" if rd < 0.25 * wr else "H2D+D2H (fused)")
            return label + d
    for k in ("nx_checksum_tma_kernel", "nx_pattern_kernel<0>", "nx_pattern_kernel<1>", "nx_table_upload_kernel"):
        if k in name:
            return {"nx_checksum_tma_kernel": "K3 nx_checksum_tma_kernel", "nx_pattern_kernel<0>": "K4 fill nx_pattern_kernel<0>",
                    "nx_pattern_kernel<1>": "K4 compare nx_pattern_kernel<1>"}.get(k, k)
    return name[:60]


def main():
    per, names = load(sys.argv[1])
    probe = json.load(open(sys.argv[2]))
    smi = open(sys.argv[3]).read() if len(sys.argv) > 3 else ""
    agg = collections.defaultdict(lambda: collections.Counter())
    for i, m in per.items():
        a = agg[kind(names[i], m)]
        a["launches"] += 1
        for k in ("gpu__time_duration.sum", "pcie__read_bytes.sum", "pcie__write_bytes.sum", "dram__bytes_read.sum",
                  "dram__bytes_write.sum"):
            a[k] += m.get(k, 0.0)
    rows = []
    for k, a in sorted(agg.items()):
        t = a["gpu__time_duration.sum"]
        rows.append({"kernel": k, "launches": a["launches"], "mean_us": round(t / a["launches"] * 1e6, 2),
                     "pcie_read_gbs": round(a["pcie__read_bytes.sum"] / t / 1e9, 2),
                     "pcie_write_gbs": round(a["pcie__write_bytes.sum"] / t / 1e9, 2),
                     "dram_read_gbs": round(a["dram__bytes_read.sum"] / t / 1e9, 1),
                     "dram_write_gbs": round(a["dram__bytes_write.sum"] / t / 1e9, 1),
                     "pcie_read_mb_per_launch": round(a["pcie__read_bytes.sum"] / a["launches"] / 1e6, 2),
                     "pcie_write_mb_per_launch": round(a["pcie__write_bytes.sum"] / a["launches"] / 1e6, 2)})
    last = smi.strip().splitlines()[-1].split(",") if smi.strip() else []
    gen = re.match(r"\s*(\d)", last[1]) if len(last) > 1 else None
    out = {"link": {"probe_ce_h2d_gbs": round(probe["ce_h2d"], 2), "probe_ce_d2h_gbs": round(probe["ce_d2h"], 2),
                    "probe_ce_bidir_h2d_gbs": round(probe["ce_bidir_h2d"], 2),
                    "probe_ce_bidir_d2h_gbs": round(probe["ce_bidir_d2h"], 2),
                    "probe_sm_h2d_gbs": round(probe["sm_h2d"], 2), "probe_sm_d2h_gbs": round(probe["sm_d2h"], 2),
                    "nvidia_smi": smi.strip().splitlines()[-1] if smi.strip() else None,
                    "gen": int(gen.group(1)) if gen else None,
                    "width": int(last[3]) if len(last) > 3 and last[3].strip().isdigit() else None},
           "kernels": rows}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
