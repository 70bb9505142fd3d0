mkdir -p gpurun_out
nvidia-smi --query-gpu=name,pcie.link.gen.current,pcie.link.width.current,clocks.sm,clocks.max.sm --format=csv,noheader
T0=$(date +%s); python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench wall s: $(( $(date +%s) - T0 ))"
python3 -c "import json; d=json.load(open('gpurun_out/bench.json')); print({k: d[k] for k in ('value','pct_of_pcie_peak','switch_latency_ms','e2e','gpu_launches','byte_exact')}); r=d['roofline']; print(round(r['achieved']), round(r['frac'],3), r['traffic']); print(d.get('x16_exchange')); print(d.get('interposer')); print(d.get('clocks')); print(d['cpu_baseline'])"
