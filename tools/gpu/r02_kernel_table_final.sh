#!/bin/bash
# Per-kernel ncu table (north star: PCIe read/write bytes/s and DRAM GB/s per
# kernel against the measured per-direction link peak and the link generation).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current --format=csv > gpurun_out/r02_ktf_smi.txt
python tools/kernel_table_target.py --probe > gpurun_out/r02_ktf_probe.json
timeout 1200 ncu --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/r02_ktf_launches.csv python tools/kernel_table_target.py > gpurun_out/r02_kt.log 2>&1
tail -n 2 gpurun_out/r02_kt.log
python tools/kernel_table.py gpurun_out/r02_ktf_launches.csv gpurun_out/r02_ktf_probe.json gpurun_out/r02_ktf_smi.txt > gpurun_out/r02_kernel_table_final.json
cat gpurun_out/r02_kernel_table_final.json
