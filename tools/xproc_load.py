"""Background bidirectional PCIe load from another process (for VMM probes)."""
import sys, time
import torch
secs = float(sys.argv[1]) if len(sys.argv) > 1 else 20
h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
d = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
d2 = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
t0 = time.time()
print("load start", flush=True)
while time.time() - t0 < secs:
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
print("load done", flush=True)
