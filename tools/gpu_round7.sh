mkdir -p gpurun_out
timeout 1200 python tools/budget_sweep.py 8 > gpurun_out/budget8.txt 2>&1; cat gpurun_out/budget8.txt
timeout 1200 python tools/budget_sweep.py 16 > gpurun_out/budget16.txt 2>&1; cat gpurun_out/budget16.txt
