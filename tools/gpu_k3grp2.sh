mkdir -p gpurun_out
for cfg in "1 0" "1 1" "1 0" "1 1"; do timeout 300 python tools/k3_inengine.py $cfg 2>&1 | grep "span ms\|TB/s events\|k3_one" | tr '\n' ' '; echo; done
timeout 900 python bench.py --steps 10 --warmup 3 --no-x16 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.err
python3 -c "import json; d=json.load(open('gpurun_out/bench.json')); print({k: d[k] for k in ('value','pct_of_pcie_peak','switch_latency_ms','gpu_launches','byte_exact')}); r=d['roofline']; print(round(r['achieved']), round(r['frac'],3), r['launches'], round(r['avg_launch_ms']*1e3,1))"
