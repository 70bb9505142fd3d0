mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.used,memory.total --format=csv
timeout 900 python -m pytest tests/test_gpu_interposer.py -x -q -s --timeout 400 > gpurun_out/interp.txt 2>&1; tail -40 gpurun_out/interp.txt
for f in gpurun_out/interposer_*.jsonl; do echo "== $f"; grep -v '"sched"' $f | cut -c1-400 | head -20; done
