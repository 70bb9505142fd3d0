mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_interposer.py tests/test_gpu_engine.py -q -m gpu -k "prefetch or interposer or vecapps or driver or torch or memgetinfo" --timeout 400 > gpurun_out/interp.txt 2>&1; tail -4 gpurun_out/interp.txt
grep -h '"prefetch"\|bye' gpurun_out/interposer_prefetch.jsonl | cut -c1-200 | head -12
