mkdir -p gpurun_out
cd /root/repo
python - <<'PY' > gpurun_out/shimdbg.txt 2>&1
import os, subprocess, sys
sys.path.insert(0, ".")
from paper_2601_11743_b200.interpose import Daemon
with Daemon(gpu="5G", pinned="2G", paged="8G") as d:
    env = d.env(); env["NIXIE_SHIM_DEBUG"] = "1"
    r = subprocess.run([sys.executable, "tests/apps/torch_app.py", "256", "2", "0.05"], env=env, capture_output=True, text=True, timeout=300)
    print("rc", r.returncode); print(r.stdout[-500:]); open("gpurun_out/shim_gpa.txt","w").write(r.stderr)
    env2 = dict(os.environ); env2["LD_DEBUG"]="bindings"; env2["LD_PRELOAD"]=env["LD_PRELOAD"]
    r = subprocess.run([sys.executable, "-c", "import torch; a=torch.randn(64,64,device='cuda'); print((a@a).sum().item())"], env=env2, capture_output=True, text=True, timeout=300)
    import re
    lines=[l for l in r.stderr.splitlines() if "dlsym" in l and ("cublas" in l or "cudart" in l or "nixie" in l)]
    print("\n".join(lines[:40]))
print(open(d.log).read()[-1500:])
PY
tail -60 gpurun_out/shimdbg.txt
