# LLM config 2 through the interposer: slab-aligned victims at the default
# slack and at 18 slack slabs (what the reference victim order grew to).
mkdir -p gpurun_out
for sl in def 18; do
  if [ "$sl" = def ]; then timeout 900 python tools/interposer_llm_c2.py 12 gpurun_out/llm_c2_$sl.jsonl > gpurun_out/llm_c2_$sl.out 2>&1
  else timeout 900 python tools/interposer_llm_c2.py 12 gpurun_out/llm_c2_$sl.jsonl 0 slab $sl > gpurun_out/llm_c2_$sl.out 2>&1; fi
  tail -1 gpurun_out/llm_c2_$sl.out | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sl', {k: d.get(k) for k in ('apps_ok','slabs_grown','live_slabs_after_switches','steady_switches','copy_bidir_gbps_median','switch_ms','grant_ms_p50','mismatches')})"
  python3 - "$sl" <<'P'
import json,sys
sw=[json.loads(l) for l in open(f'gpurun_out/llm_c2_{sys.argv[1]}.jsonl') if l.strip()]
sw=[r for r in sw if r.get('event')=='switch']
print('premaps', [r['premap_calls'] for r in sw], 'total', [round(r['total_ms']) for r in sw])
P
done
