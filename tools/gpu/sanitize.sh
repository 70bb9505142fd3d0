mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --leak-check full --print-limit 50 python tools/sanitize_target.py > gpurun_out/sanitize_memcheck.txt 2>&1; tail -4 gpurun_out/sanitize_memcheck.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_target.py > gpurun_out/sanitize_synccheck.txt 2>&1; tail -3 gpurun_out/sanitize_synccheck.txt
timeout 900 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 50 python tools/sanitize_target.py > gpurun_out/sanitize_racecheck.txt 2>&1; tail -4 gpurun_out/sanitize_racecheck.txt
