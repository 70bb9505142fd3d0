#!/bin/bash
# Round-2 checkpoint on the streaming-store build: GPU tests in the driver's
# form (-x), smoke, bench, reference arm.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,pcie.link.gen.current,pcie.link.width.current,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -x -q -m gpu -rA --timeout 600 > gpurun_out/v3_pytest_gpu.txt 2>&1; tail -3 gpurun_out/v3_pytest_gpu.txt
timeout 300 python __graft_entry__.py > gpurun_out/v3_smoke.txt 2>&1; tail -1 gpurun_out/v3_smoke.txt
timeout 900 python bench.py > gpurun_out/v3_bench.json 2> gpurun_out/v3_bench.err; tail -c 300 gpurun_out/v3_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v3_bench_ref.json 2> gpurun_out/v3_bench_ref.err; cut -c1-400 gpurun_out/v3_bench_ref.json
python3 -c "import json; d=json.load(open('gpurun_out/v3_bench.json')); print({k: d[k] for k in ('value','pct_of_pcie_peak','e2e','gpu_launches','byte_exact')}); print(d['link_roofline']['peak'], d['pcie_probe_paced'], d['pcie_probe_256mib']); print(d['switch_latency_ms']); print(d['roofline']['frac'])"
