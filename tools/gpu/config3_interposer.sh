mkdir -p gpurun_out
for iv in 1 3 6; do timeout 900 python tools/interposer_c3.py --interval $iv --horizon 45 --out gpurun_out/ic3_$iv.jsonl 2>&1 | tail -1; done | tee gpurun_out/interposer_c3.jsonl
