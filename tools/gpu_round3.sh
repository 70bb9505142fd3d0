set -x
mkdir -p gpurun_out
timeout 900 python tools/explore2.py 2>&1 | tail -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nx_swap_kernel -s 40 -c 3 -o gpurun_out/prof_ce python tools/ncu_target.py ce 4 > gpurun_out/prof_ce.log 2>&1
tail -n 3 gpurun_out/prof_ce.log
