#!/bin/bash
# Config-2 switch timelines under engine variants (tools/timeline.py).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nvidia-smi -q | grep -iE "numa|Link Width|Generation|PCIe" | head -20 > gpurun_out/smi_pcie.txt
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
for v in "" "first_batch_legs=2" "legs_per_launch=64" "legs_per_launch=256" ; do
  tag=$(echo "${v:-default}" | tr '=' '_')
  timeout 300 python tools/timeline.py --switches 5 --out gpurun_out/timeline_$tag.json $v > gpurun_out/timeline_$tag.txt 2>&1
  echo "== $tag rc=$?"; tail -4 gpurun_out/timeline_$tag.txt
done
