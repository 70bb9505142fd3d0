#!/bin/bash
# Does D2H pacing help or hurt the interposer path? The LLM pair (config 2
# with PyTorch programs, slab-aligned victims) and the vecapp pair, paced vs
# unpaced (nixied --pace-lag -1), alternating.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for r in 1 2; do
  for v in pace nopace; do
    timeout 900 python tools/interposer_llm_c2.py 12 "" 0 "$v" > gpurun_out/r02_llm_${v}_$r.txt 2>&1
    echo "llm $v $r: $(tail -1 gpurun_out/r02_llm_${v}_$r.txt | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["copy_bidir_gbps_median"], d["switch_ms"], d["steady_switches"], d["mismatches"])')"
    extra=""; [ "$v" = nopace ] && extra="--daemon-arg=--pace-lag --daemon-arg=-1"
    timeout 600 python tools/interposer_bench.py $extra > gpurun_out/r02_vec_${v}_$r.json 2>/dev/null
    echo "vec $v $r: $(python3 -c 'import json; d=json.load(open("gpurun_out/r02_vec_'${v}'_'$r'.json")); print(round(d["copy_bidir_gbps_median"],2), d["switch_total_ms"], d["mismatches"])')"
  done
done
