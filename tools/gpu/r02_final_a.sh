#!/bin/bash
# Round-2 validation: the whole GPU suite, a paired A/B of the flush interleave, config 3 on hardware,
# ncu of K1 (SM path, PCIe bytes), K4 and the large K3 launches, the config-4 sweep, the bench line.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,pcie.link.gen.current,pcie.link.width.current,clocks.sm,clocks.max.sm,memory.total --format=csv
grep -E "MemTotal|MemAvailable" /proc/meminfo
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -rA > gpurun_out/pytest_gpu_full.txt 2>&1; tail -4 gpurun_out/pytest_gpu_full.txt
timeout 600 python tools/ab_switch.py --rounds 12 base early_frame_release=0,d2h_commit_legs=0 > gpurun_out/ab3_switch.jsonl 2> gpurun_out/ab3.err; cut -c1-300 gpurun_out/ab3_switch.jsonl
timeout 900 python tools/config3.py 20 > gpurun_out/r02_config3_mlfq_mix.jsonl 2> gpurun_out/config3.err; python3 -c "
import json
for l in open('gpurun_out/r02_config3_mlfq_mix.jsonl'):
    d=json.loads(l); print(d.get('interval_s'), {k: v for k, v in d.items() if k in ('switches','byte_exact','interactive_latency_s','latency')})" 2>&1 | cut -c1-400; tail -2 gpurun_out/config3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nx_swap_kernel -s 2 -c 4 -o gpurun_out/r02_prof_k1 python tools/ncu_target.py sm 3 > gpurun_out/r02_prof_k1.log 2>&1; tail -n 2 gpurun_out/r02_prof_k1.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nx_pattern_kernel -c 4 -o gpurun_out/r02_prof_k4 python tools/ncu_target.py ce 1 > gpurun_out/r02_prof_k4.log 2>&1; tail -n 2 gpurun_out/r02_prof_k4.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:nx_checksum_tma -c 30 -o gpurun_out/r02_prof_k3_all python tools/ncu_target.py ce 3 > gpurun_out/r02_prof_k3_all.log 2>&1; tail -n 2 gpurun_out/r02_prof_k3_all.log
timeout 1500 python tools/budget_sweep.py > gpurun_out/r02_budget_sweep_2.jsonl 2> gpurun_out/budget_sweep_2.err; tail -1 gpurun_out/r02_budget_sweep_2.jsonl; tail -2 gpurun_out/budget_sweep_2.err
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.err
python3 -c "import json; d=json.load(open('gpurun_out/bench.json')); print({k: d[k] for k in ('value','pct_of_pcie_peak','e2e','gpu_launches','byte_exact')}); print(d['link_roofline']['peak'], d['switch_latency_ms']['p50_over_ideal'], d.get('x16_exchange',{}).get('p50_over_ideal'), d['roofline']['frac'], d.get('paper_mechanism_2mib_ce'))"
