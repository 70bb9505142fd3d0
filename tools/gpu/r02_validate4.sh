#!/bin/bash
# Checkpoint after k3_verify_group 1024 -> 4096: engine/scale/workload GPU
# tests, smoke, default bench.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,pcie.link.gen.current,pcie.link.width.current,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_scale.py tests/test_gpu_budget.py tests/test_gpu_workload.py -x -q -m gpu -rA --timeout 600 > gpurun_out/v4_pytest_gpu.txt 2>&1; tail -2 gpurun_out/v4_pytest_gpu.txt
timeout 300 python __graft_entry__.py > gpurun_out/v4_smoke.txt 2>&1; tail -1 gpurun_out/v4_smoke.txt
timeout 900 python bench.py > gpurun_out/v4_bench.json 2> gpurun_out/v4_bench.err; tail -c 300 gpurun_out/v4_bench.err
python3 -c "import json; d=json.load(open('gpurun_out/v4_bench.json')); print({k: d[k] for k in ('value','pct_of_pcie_peak','e2e','gpu_launches','byte_exact')}); print(d['link_roofline']['peak'], d['pcie_probe_paced'], d['pcie_probe_256mib']); print(d['switch_latency_ms']); print(d['roofline'])"
