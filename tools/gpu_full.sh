mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; tail -4 gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1000 gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1
python3 -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print({k: d[k] for k in ('value','pct_of_pcie_peak','switch_latency_ms','ideal_latency_ms','gpu_launches','byte_exact','settle')})
print(d['e2e']); print(d['roofline']); print(d['pcie_probe']['ce_bidir_total'], d['pcie_probe_after']); print(d['x16_exchange']); print(d['clocks'])
r=json.load(open('gpurun_out/bench_ref.json')); print('ref', r['value'], r['cpu_baseline']['sample'])"
