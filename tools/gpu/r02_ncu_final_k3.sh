#!/bin/bash
# ncu --set full of K3 on steady config-2 switches of the final build. With
# 4096-leg arrival groups a switch issues 6 K3 launches, so 8 switches are run
# and the 10 launches after the first 30 (switches 6-7, steady) are captured.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:nx_checksum_tma -s 30 -c 10 \
  -o gpurun_out/r02_prof_k3_c2_final python tools/ncu_target.py ce 8 c2 > gpurun_out/r02_prof_k3_c2_final.log 2>&1
tail -n 3 gpurun_out/r02_prof_k3_c2_final.log
ncu -i gpurun_out/r02_prof_k3_c2_final.ncu-rep --page raw --csv > gpurun_out/r02_ncu_k3_c2_final_raw.csv 2>&1
ncu -i gpurun_out/r02_prof_k3_c2_final.ncu-rep --page details --csv > gpurun_out/r02_ncu_k3_c2_final_details.csv 2>&1
ls -la gpurun_out | head -20
