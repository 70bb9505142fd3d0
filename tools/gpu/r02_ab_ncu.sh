#!/bin/bash
# Paired A/B of the fetch/eviction coupling modes, the capture-deadlock test, ncu of this round's kernels, the bench line.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python tools/ab_switch.py --rounds 10 --out gpurun_out/ab_raw.json base d2h_commit_legs=128 d2h_commit_legs=64 \
  early_frame_release=0,d2h_commit_legs=0 early_frame_release=0,d2h_commit_legs=32 > gpurun_out/ab_switch.jsonl 2> gpurun_out/ab_switch.err
cat gpurun_out/ab_switch.jsonl | cut -c1-330; tail -2 gpurun_out/ab_switch.err
timeout 600 python -m pytest -q -rA --timeout 300 -m gpu "tests/test_gpu_interposer.py::test_pause_during_a_capture_with_an_allocation_does_not_deadlock" > gpurun_out/pytest_capture.txt 2>&1; tail -4 gpurun_out/pytest_capture.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-x16 --no-interposer --no-uvm --latency-switches 2 > gpurun_out/ncu_bench.log 2>&1; tail -n 2 gpurun_out/ncu_bench.log | cut -c1-200
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nx_checksum_tma -s 6 -c 3 -o gpurun_out/r02_prof_k3 python tools/ncu_target.py ce 4 > gpurun_out/r02_prof_k3.log 2>&1; tail -n 3 gpurun_out/r02_prof_k3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nx_table_upload -s 4 -c 2 -o gpurun_out/r02_prof_upload python tools/ncu_target.py ce 4 > gpurun_out/r02_prof_upload.log 2>&1; tail -n 3 gpurun_out/r02_prof_upload.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 400 gpurun_out/bench.err
python3 -c "import json; d=json.load(open('gpurun_out/bench.json')); print({k: d[k] for k in ('value','pct_of_pcie_peak','e2e','gpu_launches','byte_exact')}); print(d['link_roofline']['peak'], d['pcie_probe_256mib']); print(d['pcie_counters']); print(d['switch_latency_ms']); print(d.get('x16_exchange',{}).get('p50_over_ideal')); print(d['roofline'])"
