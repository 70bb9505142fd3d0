"""Seeded random small workloads (workload_sim.hpp grammar) for differential
parity tests against the reference (shared by tests and golden generation)."""
import random


def random_workload(seed: int) -> str:
    r = random.Random(seed)
    gpu = r.choice([64, 96, 128, 192])        # MiB
    pinned = r.choice([32, 64, 128, 256])
    n = r.randint(2, 4)
    lines = [f"capacity gpu {gpu}MiB", f"capacity pinned {pinned}MiB", "capacity paged 4GiB",
             f"link 0 {r.choice([1, 4, 16])}GiB/s {r.choice([1, 4, 16])}GiB/s full",
             f"link 1 {r.choice([1, 2, 8])}GiB/s {r.choice([1, 2, 8])}GiB/s full",
             f"dispatch {r.choice(['0', '5e-6', '1e-4'])}",
             f"window {r.choice([4, 8, 16])}MiB",
             f"mlfq {r.randint(2, 4)} {r.choice([1, 2])} {r.choice([0.25, 0.5])} {r.choice([0.02, 0.05, 0.1])} 0.01",
             f"seed {r.randint(0, 1 << 30)}", f"horizon {r.choice([4, 6, 8])}",
             f"prefetch {r.choice(['on', 'off'])}"]
    for a in range(n):
        size = r.choice([16, 32, 48, 64]) * (1 << 20)
        size = min(size, gpu << 20)
        tier = r.choice(["paged", "pinned", "gpu"]) if a == 0 else r.choice(["paged", "paged", "pinned"])
        if tier == "pinned" and size > pinned << 19:  # keep the initial placement feasible most of the time
            tier = "paged"
        if r.random() < 0.6:
            lines.append(f"interactive {a} {size} {tier} {r.uniform(0, 1):.3f} {r.choice([0.2, 0.5, 1.0, 2.0])} "
                         f"{r.randint(1, 6)} {r.choice([0.005, 0.02, 0.05])} {r.choice([0, 0.1, 0.3])}")
        else:
            lines.append(f"batch {a} {size} {tier} {r.uniform(0, 1):.3f} {r.choice([0.01, 0.03])} {r.randint(1, 8)}")
    return "\n".join(lines) + "\n"
