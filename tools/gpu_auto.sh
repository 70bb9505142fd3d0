# Stale-mapping policy "auto" (keep while two apps hold memory): config 3
# through the interposer (3 apps), the LLM pair (2 apps), interposer tests.
mkdir -p gpurun_out
bash tools/gpu_ic3.sh | cut -c1-200
VARIANTS=def bash tools/gpu_stale.sh
timeout 1200 python -m pytest tests/test_gpu_interposer.py -q --timeout 400 > gpurun_out/ip_all.txt 2>&1; tail -2 gpurun_out/ip_all.txt
