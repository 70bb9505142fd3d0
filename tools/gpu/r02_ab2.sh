#!/bin/bash
# Longer paired A/B of the coupling modes; config-4 lane concurrency grid.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python tools/ab_switch.py --rounds 25 --out gpurun_out/ab2_raw.json base d2h_commit_legs=128 early_frame_release=0,d2h_commit_legs=0 \
  > gpurun_out/ab2_switch.jsonl 2> gpurun_out/ab2_switch.err; cut -c1-330 gpurun_out/ab2_switch.jsonl; tail -2 gpurun_out/ab2_switch.err
timeout 1200 python tools/c4_lanes.py 2,4,8 16,64 256,1024 > gpurun_out/c4_lanes.jsonl 2> gpurun_out/c4_lanes.err; cat gpurun_out/c4_lanes.jsonl; tail -2 gpurun_out/c4_lanes.err
