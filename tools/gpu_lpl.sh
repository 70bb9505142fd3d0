mkdir -p gpurun_out
for lpl in 128 256; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-x16 --legs-per-launch $lpl > gpurun_out/bench_lpl$lpl.json 2> gpurun_out/bench_lpl$lpl.err
python3 -c "import json; d=json.load(open('gpurun_out/bench_lpl$lpl.json')); r=d['roofline']; print($lpl, round(d['value'],1), round(d['pct_of_pcie_peak'],1), d['switch_latency_ms']['p50'], 'k3', round(r['achieved']), round(r['frac'],3), round(r['achieved_kernel_clock']), r['launches'], round(r['avg_launch_ms']*1e3,1))"
done
