mkdir -p gpurun_out
timeout 300 python tools/k3_probe.py > gpurun_out/k3_probe.txt 2>&1; tail -8 gpurun_out/k3_probe.txt
timeout 1500 python tools/scale_check.py > gpurun_out/scale.txt 2>&1; cat gpurun_out/scale.txt | cut -c1-400
