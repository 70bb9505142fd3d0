mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_scale.py tests/test_gpu_workload.py -q -m gpu -x --timeout 600 > gpurun_out/pytest_eng.txt 2>&1; tail -3 gpurun_out/pytest_eng.txt
for cfg in "1 0" "1 1"; do timeout 300 python tools/k3_inengine.py $cfg 2>&1 | grep -v "^\[(" | tail -5; done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.err
python3 -c "import json; d=json.load(open('gpurun_out/bench.json')); print({k: d[k] for k in ('value','pct_of_pcie_peak','switch_latency_ms','e2e','gpu_launches','byte_exact')}); print(d['roofline']); print(d.get('x16_exchange'))"
