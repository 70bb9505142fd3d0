mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_interposer.py -x -q -s --timeout 400 > gpurun_out/interp.txt 2>&1; tail -3 gpurun_out/interp.txt
timeout 900 python tools/interposer_bench.py --out gpurun_out/interposer_c2.jsonl 2>&1 | tail -3
