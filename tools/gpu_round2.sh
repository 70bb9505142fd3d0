set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 2>&1 | tail -15
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 2000 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ce.csv python tools/ncu_target.py ce 4 > gpurun_out/ncu_ce.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nx_swap_kernel -s 40 -c 3 -o gpurun_out/prof_ce python tools/ncu_target.py ce 4 > gpurun_out/prof_ce.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nx_swap_kernel -s 20 -c 2 --metrics pcie__read_bytes.sum,pcie__write_bytes.sum -o gpurun_out/prof_sm python tools/ncu_target.py sm 3 > gpurun_out/prof_sm.log 2>&1
cat gpurun_out/bench.json
for f in gpurun_out/ncu_ce.log gpurun_out/prof_ce.log gpurun_out/prof_sm.log; do tail -n 4 $f; done
