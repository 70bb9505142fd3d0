set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ce.csv python tools/ncu_target.py ce 4 > gpurun_out/ncu_ce.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sm.csv python tools/ncu_target.py sm 4 > gpurun_out/ncu_sm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nx_swap_kernel -s 40 -c 3 -o gpurun_out/prof_ce python tools/ncu_target.py ce 4 > gpurun_out/prof_ce.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nx_swap_kernel -s 20 -c 3 --metrics pcie__read_bytes,pcie__write_bytes,pcie__throughput -o gpurun_out/prof_sm python tools/ncu_target.py sm 3 > gpurun_out/prof_sm.log 2>&1
ls -la gpurun_out; tail -5 gpurun_out/*.log
