mkdir -p gpurun_out
timeout 900 python tools/interposer_bench.py --out gpurun_out/interposer_c2.jsonl 2>&1 | tail -1 | cut -c1-100
python3 - <<'PY'
import json
sw=[json.loads(l) for l in open('gpurun_out/interposer_c2.jsonl') if '"switch"' in l]
for d in sw: print(d['from'],d['to'],'copy',round(d['copy_ms']),'grant',round(d['grant_ms'],1),'recv',round(d['grant_recv_ms'],1),'premap',round(d['premap_ms'],1),d['premap_calls'],'unmap',round(d['premap_unmap_ms'],1),'map',round(d['map_ms'],1),d['map_calls'],'total',round(d['total_ms']))
PY
