#!/bin/bash
# ncu --set full of K1T (the SM copy path's default kernel) on the kernel
# table's 1 GiB full-GPU exchange: two D2H and two H2D launches.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nx_swap_tma -c 4 \
  -o gpurun_out/r02_prof_k1t python tools/kernel_table_target.py > gpurun_out/r02_prof_k1t.log 2>&1
tail -n 3 gpurun_out/r02_prof_k1t.log
ncu -i gpurun_out/r02_prof_k1t.ncu-rep --page raw --csv > gpurun_out/r02_ncu_k1t_raw.csv 2>&1
ncu -i gpurun_out/r02_prof_k1t.ncu-rep --page details --csv > gpurun_out/r02_ncu_k1t_details.csv 2>&1
ls -la gpurun_out | grep k1t
