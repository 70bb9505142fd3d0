#!/bin/bash
# Early frame release: parity/byte-exactness gates, then config-2 timelines with it on and off.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x --timeout 900 -m gpu tests/test_gpu_engine.py tests/test_gpu_scale.py tests/test_gpu_budget.py \
  tests/test_gpu_workload.py "tests/test_gpu_interposer.py::test_two_vecapps_oversubscribed" > gpurun_out/pytest_early.txt 2>&1; tail -4 gpurun_out/pytest_early.txt
timeout 300 python __graft_entry__.py 2>&1 | tail -1
for v in "" "early_frame_release=0 d2h_commit_legs=0" "d2h_commit_legs=64" "d2h_commit_legs=16" "" "early_frame_release=0 d2h_commit_legs=0"; do
  tag=$(echo "${v:-early}" | tr '= ' '_-')
  timeout 300 python tools/timeline.py --switches 8 --out gpurun_out/tle_$tag.json $v > gpurun_out/tle_$tag.txt 2>&1
  echo "== $tag rc=$?"; tail -2 gpurun_out/tle_$tag.txt | cut -c1-300; python3 - "$tag" <<'PY'
import json,sys,statistics as st
try:
    d=json.load(open(f"gpurun_out/tle_{sys.argv[1]}.json"))["summary"]
except Exception as e:
    print("no json", e); sys.exit(0)
sw=d["switches"]; sp=[s["span_ms"] for s in sw]
print({"span_p50": round(st.median(sp),2), "span_min": round(min(sp),2), "span_max": round(max(sp),2),
       "h2d_only": round(st.median([s["h2d_only_ms"] for s in sw]),2), "d2h_only": round(st.median([s["d2h_only_ms"] for s in sw]),2),
       "h2d_rate": round(st.median([s["h2d_rate_gbs"] for s in sw]),2), "probe": round(d["probe"]["ce_bidir_total"],2), "exact": d["byte_exact"]})
PY
done
timeout 1500 python tools/budget_sweep.py > gpurun_out/r02_budget_sweep.jsonl 2> gpurun_out/budget_sweep.err; tail -1 gpurun_out/r02_budget_sweep.jsonl; tail -2 gpurun_out/budget_sweep.err
