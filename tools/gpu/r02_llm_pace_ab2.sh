#!/bin/bash
# LLM pair through the interposer, paced vs unpaced, after contiguous pinned slots.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for r in 1 2 3; do
  for v in pace nopace; do
    timeout 900 python tools/interposer_llm_c2.py 12 "" 0 "$v" > gpurun_out/r02_llm2_${v}_$r.txt 2>&1
    echo "llm $v $r: $(tail -1 gpurun_out/r02_llm2_${v}_$r.txt | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["copy_bidir_gbps_median"], d["switch_ms"], d["steady_switches"], d["mismatches"])')"
  done
done
