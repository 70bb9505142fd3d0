mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_interposer.py -q -x --timeout 400 > gpurun_out/interp.txt 2>&1; tail -2 gpurun_out/interp.txt
timeout 900 python tools/interposer_bench.py --out gpurun_out/interposer_c2.jsonl 2>&1 | tail -1 | cut -c1-200
python3 - <<'PY'
import json
sw=[json.loads(l) for l in open('gpurun_out/interposer_c2.jsonl') if '"switch"' in l]
print('c2 switches', len(sw), 'map calls', [s['map_calls'] for s in sw][:20], 'grant ms', [round(s['grant_ms'],1) for s in sw][:20])
PY
timeout 900 python tools/interposer_c3.py --interval 3 --horizon 45 --out gpurun_out/ic3_3.jsonl 2>&1 | tail -1 | tee gpurun_out/interposer_c3_aff.jsonl | cut -c1-400
python3 - <<'PY'
import json
sw=[json.loads(l) for l in open('gpurun_out/ic3_3.jsonl') if '"switch"' in l]
sw.sort(key=lambda d:-d['total_ms'])
for d in sw[:5]: print(d['from'],d['to'],'in',d['bytes_in']>>30,'copy',d['copy_ms'],'grant',d['grant_ms'],'total',d['total_ms'])
byes=[json.loads(l) for l in open('gpurun_out/ic3_3.jsonl') if '"bye"' in l]
print([(b['app'], b['map_ms']) for b in byes])
PY
