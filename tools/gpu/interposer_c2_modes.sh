# Config 2 through the interposer (two vecapps), daemon logs kept: the default
# mapping mode twice, then --isolate-victims.
mkdir -p gpurun_out
for v in def1 def2 isolate; do
  x=""; [ "$v" = isolate ] && x="--daemon-arg=--isolate-victims"
  timeout 900 python tools/interposer_bench.py --iters 10 --out gpurun_out/ipc2_$v.jsonl $x > gpurun_out/ipc2_$v.json 2>&1
  python3 - "$v" <<'P'
import json,sys
v=sys.argv[1]
d=json.loads(open(f'gpurun_out/ipc2_{v}.json').read().strip().splitlines()[-1])
print(v, d.get('switch_total_ms'), d.get('copy_bidir_gbps_median'))
sw=[json.loads(l) for l in open(f'gpurun_out/ipc2_{v}.jsonl') if l.strip()]
for r in sw:
    if r.get('event')=='switch' and r['pcie_h2d']>0:
        print(' ', r['from'],'->',r['to'], round(r['total_ms']), 'copy', round(r['copy_ms']), 'grant', round(r['grant_ms'],1), 'premap', r['premap_calls'], round(r['premap_ms']), 'unmap', round(r['premap_unmap_ms']), 'recv', round(r['grant_recv_ms'],1), 'map', r['map_calls'], round(r['map_ms'],1))
P
done
