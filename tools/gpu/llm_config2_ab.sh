# LLM pair (config 2): default vs --isolate-victims, alternating, same box.
mkdir -p gpurun_out
for v in def isolate def isolate; do
  f=""; [ "$v" = isolate ] && f="slab,isolate"
  timeout 900 python tools/interposer_llm_c2.py 12 gpurun_out/llm_ab_$v.jsonl 0 $f > gpurun_out/llm_ab_$v.out 2>&1
  tail -1 gpurun_out/llm_ab_$v.out | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', {k: d.get(k) for k in ('apps_ok','steady_switches','copy_bidir_gbps_median','switch_ms','mismatches')})"
done
