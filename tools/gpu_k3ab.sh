mkdir -p gpurun_out
for one in 0 1; do timeout 300 python tools/k3_inengine.py $one 2>&1 | grep -v "^\[(" | tail -12; done
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 400 gpurun_out/bench.err
python3 -c "import json; d=json.load(open('gpurun_out/bench.json')); print({k: d[k] for k in ('value','pct_of_pcie_peak','switch_latency_ms','e2e','gpu_launches','byte_exact')}); print(d['roofline'])"
