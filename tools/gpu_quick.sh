set -x
nvidia-smi --query-gpu=name,pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,pcie.link.width.max --format=csv
nproc; free -g | head -2; nvidia-smi topo -m | head -20
timeout 300 python __graft_entry__.py 2>&1 | tail -20
timeout 300 python -c "
from paper_2601_11743_b200 import SwapEngine, GIB, MIB
e=SwapEngine(gpu_capacity=1*GIB, pinned_capacity=1*GIB, paged_capacity=1*GIB)
for ch in (2*MIB, 16*MIB, 64*MIB):
    print(ch>>20, 'MiB', {k:(round(v,2) if isinstance(v,float) else v) for k,v in e.probe_pcie(1*GIB, ch).items()})
" 2>&1 | tail -10
