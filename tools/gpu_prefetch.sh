mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_engine.py -q -m gpu -k "prefetch or full_gpu" --timeout 300 2>&1 | tail -3
timeout 900 python tools/prefetch_ab.py 30 8 3 > gpurun_out/prefetch_ab.jsonl 2> gpurun_out/prefetch_ab.err; tail -3 gpurun_out/prefetch_ab.err
python3 - <<'PY'
import json
for l in open("gpurun_out/prefetch_ab.jsonl"):
    d = json.loads(l)
    print("prefetch", d["prefetch"], "switches", d["switches"], "prefetched GiB", round(d["prefetched_bytes"]/2**30, 1), "exact", d["byte_exact"], d["errors"])
    for k, v in d["per_app"].items(): print("  ", k, v)
PY
