mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nx_checksum_tma -c 24 -o gpurun_out/prof_k3table_all python tools/ncu_target.py ce 2 > gpurun_out/prof_k3table_all.log 2>&1; tail -n 3 gpurun_out/prof_k3table_all.log
