#!/bin/bash
# Config 4 (budget sweep with the UVM series), the budget/UVM gates, and the bench line.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -rA --timeout 900 -m gpu tests/test_gpu_engine.py tests/test_gpu_budget.py tests/test_gpu_uvm.py > gpurun_out/pytest_c4.txt 2>&1; tail -8 gpurun_out/pytest_c4.txt
timeout 1500 python tools/budget_sweep.py > gpurun_out/r02_budget_sweep.jsonl 2> gpurun_out/budget_sweep.err; tail -3 gpurun_out/r02_budget_sweep.jsonl | cut -c1-600; tail -3 gpurun_out/budget_sweep.err
timeout 300 python __graft_entry__.py 2>&1 | tail -1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 400 gpurun_out/bench.err
python3 -c "import json; d=json.load(open('gpurun_out/bench.json')); print({k: d[k] for k in ('value','pct_of_pcie_peak','e2e','gpu_launches','byte_exact')}); print(d['link_roofline']['peak'], d['pcie_probe_256mib']); print(d['pcie_counters']); print(d['switch_latency_ms']); print(d.get('x16_exchange',{}).get('p50_over_ideal'))"
