set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py -q -m gpu --timeout 300 -k "corrupt or byte_exact" > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nx_checksum_tma -s 40 -c 3 -o gpurun_out/prof_k3tma python tools/ncu_target.py ce 4 > gpurun_out/prof_k3tma.log 2>&1
tail -n 3 gpurun_out/prof_k3tma.log
