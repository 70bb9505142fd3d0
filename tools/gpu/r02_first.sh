mkdir -p gpurun_out
nvidia-smi --query-gpu=name,pcie.link.gen.current,pcie.link.width.current,clocks.sm,clocks.max.sm --format=csv
timeout 2000 python -m pytest tests -q -m gpu --timeout 900 -rA > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py 2>&1 | tail -1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.err
bash tools/gpu/r02_timeline.sh
