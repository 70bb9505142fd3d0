#!/bin/bash
# Config-2 switch timelines: D2H commit groups (EngineConfig::d2h_commit_legs) vs whole-batch commits.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x --timeout 600 -m gpu tests/test_gpu_engine.py tests/test_gpu_scale.py > gpurun_out/pytest_engine.txt 2>&1; tail -3 gpurun_out/pytest_engine.txt
for v in "d2h_commit_legs=0" "" "d2h_commit_legs=16" "d2h_commit_legs=64" "first_batch_legs=4" "d2h_commit_legs=0 first_batch_legs=2" "d2h_commit_legs=0" "" ; do
  tag=$(echo "${v:-default}" | tr '= ' '_-')
  timeout 300 python tools/timeline.py --switches 8 --out gpurun_out/tl_$tag.json $v > gpurun_out/tl_$tag.txt 2>&1
  echo "== $tag rc=$?"; python3 - "$tag" <<'PY'
import json,sys,statistics as st
d=json.load(open(f"gpurun_out/tl_{sys.argv[1]}.json"))["summary"]
sw=d["switches"]; sp=[s["span_ms"] for s in sw]
print({"span_p50": round(st.median(sp),2), "span_min": round(min(sp),2), "span_max": round(max(sp),2),
       "h2d_only": round(st.median([s["h2d_only_ms"] for s in sw]),2), "d2h_only": round(st.median([s["d2h_only_ms"] for s in sw]),2),
       "h2d_rate": round(st.median([s["h2d_rate_gbs"] for s in sw]),2), "probe": round(d["probe"]["ce_bidir_total"],2), "exact": d["byte_exact"]})
PY
done
