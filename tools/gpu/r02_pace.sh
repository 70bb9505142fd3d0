#!/bin/bash
# Round 2, D2H pacing: GPU tests, bench, config-2 timeline and config-4 A/B.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rA > gpurun_out/pace_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pace_pytest_gpu.txt
python bench.py > gpurun_out/pace_bench.json 2> gpurun_out/pace_bench.err; echo "bench rc=$?"
timeout 300 python tools/timeline.py --switches 5 --out gpurun_out/timeline_pace.json > gpurun_out/timeline_pace.txt 2>&1
timeout 900 python tools/ab_c4.py --budgets 2,8 --rounds 3 base pace_lag_legs=-1 > gpurun_out/ab_c4_pace.txt 2>&1; echo "c4 rc=$?"
tail -2 gpurun_out/pace_pytest_gpu.txt
