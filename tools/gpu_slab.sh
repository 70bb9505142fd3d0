mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_interposer.py -q -x --timeout 400 > gpurun_out/interp.txt 2>&1; tail -1 gpurun_out/interp.txt
for sm in 128 512 1024; do timeout 900 python tools/interposer_c3.py --interval 3 --horizon 40 --slab-mib $sm 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['slab_mib'], d['switches'], d['grant_ms'], d['switch_ms'], d['per_app']['code-completion']['request_ms'], d['mismatches'], d['apps_ok'])"; done
