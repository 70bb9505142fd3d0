mkdir -p gpurun_out
for i in 1 2; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-x16 > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err
python3 -c "import json; d=json.load(open('gpurun_out/bench_$i.json')); p=d['pcie_probe']; print(round(d['value'],1), round(d['pct_of_pcie_peak'],1), d['switch_latency_ms']['p50'], p['ce_bidir_total'], p['ce_h2d'], p['ce_bidir_h2d'], d['cpu_baseline']['ms_per_switch'])"
done
