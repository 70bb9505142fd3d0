mkdir -p gpurun_out
nvidia-smi --query-gpu=name,pcie.link.gen.current,pcie.link.width.current,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.err
python3 -c "import json; d=json.load(open('gpurun_out/bench.json')); print({k: d[k] for k in ('value','pct_of_pcie_peak','switch_latency_ms','e2e','gpu_launches','byte_exact')}); print(d['roofline']); print(d.get('x16_exchange')); print(d.get('clocks'))"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; cut -c1-300 gpurun_out/bench_ref.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-x16 --no-interposer > gpurun_out/ncu_bench.log 2>&1; tail -n 2 gpurun_out/ncu_bench.log | cut -c1-200
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nx_checksum_tma -s 6 -c 3 -o gpurun_out/prof_k3table python tools/ncu_target.py ce 4 > gpurun_out/prof_k3table.log 2>&1; tail -n 3 gpurun_out/prof_k3table.log
ls -la gpurun_out/
