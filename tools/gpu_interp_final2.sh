mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_interposer.py -q --timeout 400 > gpurun_out/ip.txt 2>&1; tail -1 gpurun_out/ip.txt
timeout 900 python tools/interposer_bench.py --out gpurun_out/interposer_c2.jsonl 2>&1 | tail -1 > gpurun_out/interposer_c2_summary.json; python3 -c "import json; d=json.load(open('gpurun_out/interposer_c2_summary.json')); print({k:d.get(k) for k in ('steady_switches','copy_bidir_gbps_median','switch_total_ms','grant_ms_median','verified','mismatches')})"
for iv in 1 3 6; do timeout 900 python tools/interposer_c3.py --interval $iv --horizon 45 --out gpurun_out/ic3_$iv.jsonl 2>&1 | tail -1; done > gpurun_out/interposer_c3.jsonl
python3 -c "
import json
for l in open('gpurun_out/interposer_c3.jsonl'):
    d=json.loads(l); print(d['interval_s'], d['switches'], d['grant_ms'], d['switch_ms'], d['per_app']['code-completion']['request_ms'], d['mismatches'], d['apps_ok'])"
