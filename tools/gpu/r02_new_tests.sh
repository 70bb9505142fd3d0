#!/bin/bash
# Round-2 additions on the GPU: daemon plan parity, UVM gate, interposer breadth, CE bubble probe.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -rA --timeout 600 -m gpu tests/test_gpu_daemon_parity.py tests/test_gpu_uvm.py \
  "tests/test_gpu_interposer.py::test_interposer_api_breadth" "tests/test_gpu_interposer.py::test_implicit_allocations_count_against_the_budget" \
  > gpurun_out/pytest_new.txt 2>&1; tail -25 gpurun_out/pytest_new.txt
timeout 300 ./tools/ce_bubble > gpurun_out/ce_bubble.txt 2>&1; cat gpurun_out/ce_bubble.txt
