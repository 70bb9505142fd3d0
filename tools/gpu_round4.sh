set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
timeout 900 python tools/explore2.py > gpurun_out/explore2.txt 2>&1; cat gpurun_out/explore2.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nx_checksum_tma -s 40 -c 3 -o gpurun_out/prof_k3tma python tools/ncu_target.py ce 4 > gpurun_out/prof_k3tma.log 2>&1
tail -n 3 gpurun_out/prof_k3tma.log
