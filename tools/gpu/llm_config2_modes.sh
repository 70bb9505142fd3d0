# LLM config 2 through the interposer: the default (slab-aligned victims,
# stale mappings kept, descending evictions), then --isolate-victims.
mkdir -p gpurun_out
for v in ${VARIANTS:-def isolate}; do
  f=""; [ "$v" = isolate ] && f="slab,isolate"
  timeout 900 python tools/interposer_llm_c2.py 12 gpurun_out/llm_c2_$v.jsonl 0 $f > gpurun_out/llm_c2_$v.out 2>&1
  tail -1 gpurun_out/llm_c2_$v.out | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', {k: d.get(k) for k in ('apps_ok','slabs_grown','live_slabs_after_switches','steady_switches','copy_bidir_gbps_median','switch_ms','grant_ms_p50','mismatches','errors')})"
  python3 - "$v" <<'P'
import json,sys
sw=[json.loads(l) for l in open(f'gpurun_out/llm_c2_{sys.argv[1]}.jsonl') if l.strip()]
sw=[r for r in sw if r.get('event')=='switch']
print('premaps', [r['premap_calls'] for r in sw], 'total', [round(r['total_ms']) for r in sw])
P
done
timeout 900 python -m pytest tests/test_gpu_interposer.py -q --timeout 400 -x -k two_vecapps > gpurun_out/ip_modes.txt 2>&1; tail -2 gpurun_out/ip_modes.txt
