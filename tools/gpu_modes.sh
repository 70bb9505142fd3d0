# Interposer after the victim/mapping defaults changed: GPU interposer tests,
# config 2 (vecapps) as the bench runs it, the LLM pair in both mapping modes.
mkdir -p gpurun_out
timeout 900 python tools/interposer_bench.py --iters 10 > gpurun_out/ipbench.json 2> gpurun_out/ipbench.err; tail -c 600 gpurun_out/ipbench.json
bash tools/gpu_stale.sh
timeout 1200 python -m pytest tests/test_gpu_interposer.py -q --timeout 400 > gpurun_out/ip_all.txt 2>&1; tail -2 gpurun_out/ip_all.txt
