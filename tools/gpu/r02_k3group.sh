#!/bin/bash
# K3 arrival-check group size A/B (switch span and event-timed K3 rate) and a
# config-2 timeline of the current build.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 300 python tools/timeline.py --switches 5 --out gpurun_out/timeline_now.json > gpurun_out/timeline_now.txt 2>&1; echo "timeline rc=$?"; tail -4 gpurun_out/timeline_now.txt
timeout 900 python tools/ab_switch.py --rounds 10 --out gpurun_out/ab_k3group.json base k3_verify_group=2048 k3_verify_group=4096 > gpurun_out/ab_k3group.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/ab_k3group.txt | cut -c1-900
