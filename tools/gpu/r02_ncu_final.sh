#!/bin/bash
# Round 2 ncu evidence for the current build: the bench's launch list
# (gpu__time_duration per launch) and a --set full capture of the K3 launches
# of one steady config-2 switch (record launches + arrival checks).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench_final.csv \
  python bench.py --steps 2 --warmup 3 --no-x16 --no-interposer --no-uvm --latency-switches 2 > gpurun_out/ncu_bench.log 2>&1
tail -n 2 gpurun_out/ncu_bench.log | cut -c1-200
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:nx_checksum_tma -s 30 -c 10 \
  -o gpurun_out/r02_prof_k3_c2_final python tools/ncu_target.py ce 8 c2 > gpurun_out/r02_prof_k3_c2_final.log 2>&1
tail -n 3 gpurun_out/r02_prof_k3_c2_final.log
ncu -i gpurun_out/r02_prof_k3_c2_final.ncu-rep --page raw --csv > gpurun_out/r02_ncu_k3_c2_final_raw.csv 2>&1
ls -la gpurun_out | head -40
