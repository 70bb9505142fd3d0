mkdir -p gpurun_out
timeout 900 python tools/interposer_llm_c2.py 12 gpurun_out/llm_c2.jsonl > gpurun_out/llm_c2.out 2>&1
tail -1 gpurun_out/llm_c2.out | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d.get(k) for k in ('apps_ok','slabs_grown','slabs_dropped','live_slabs_after_switches','steady_switches','copy_bidir_gbps_median','switch_ms','grant_ms_p50','mismatches','errors')}, [a['logit_mismatch'] for a in d['apps'] if a])"
python3 - <<'P'
import json
recs=[json.loads(l) for l in open('gpurun_out/llm_c2.jsonl') if l.strip()]
sw=[r for r in recs if r.get('event')=='switch']
print('partial', [r.get('partial_slabs') for r in sw], 'live', [r.get('live_slabs') for r in sw])
P
timeout 900 python -m pytest tests/test_gpu_interposer.py -q --timeout 400 -x > gpurun_out/ip.txt 2>&1; tail -2 gpurun_out/ip.txt
