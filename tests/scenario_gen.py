"""Seeded random scenario generator shared by the golden-fixture script and
the parity tests (small instances the reference finishes in milliseconds)."""
import random

MIB = 1 << 20


def random_scenario(seed: int) -> str:
    r = random.Random(seed)
    blk = 2 * MIB
    caps = {"gpu": r.randint(2, 12) * blk, "pinned": r.randint(1, 10) * blk, "paged": r.randint(8, 40) * blk}
    lines = [f"capacity gpu {caps['gpu']}", f"capacity pinned {caps['pinned']}", f"capacity paged {caps['paged']}",
             "capacity disk 0", f"window {r.choice([1, 1, 2, 4]) * blk}"]
    if r.random() < 0.3:
        lines.append(f"budget {r.randint(1, 10) * blk}")
    if r.random() < 0.2:
        lines.append(f"link 0 {r.choice([16, 32, 64])}GiB/s {r.choice([16, 32, 64])}GiB/s {r.choice(['full', 'full', 'half'])}")
    if r.random() < 0.2:
        lines.append(f"link 1 {r.choice([8, 32])}GiB/s {r.choice([8, 32])}GiB/s full")
    used = {"gpu": 0, "pinned": 0, "paged": 0}
    napps = r.randint(2, 4)
    apps = []
    for a in range(napps):
        size = r.randint(1, max(1, caps["gpu"] // MIB)) * MIB  # may be unaligned, never above the GPU cap
        fp = -(-size // blk) * blk
        order = ["gpu", "pinned", "paged"]
        r.shuffle(order)
        for t in order:
            if used[t] + fp <= caps[t]:
                used[t] += fp
                lines.append(f"app {a} {size} {t}")
                apps.append(a)
                break
    t = 0.0
    prev = None
    for _ in range(r.randint(2, 7)):
        choices = [a for a in apps if a != prev]
        if not choices:
            break
        nxt = r.choice(choices)
        t += r.choice([0.0, 0.001, 0.5, 3.0, 20.0])
        lines.append(f"switch {t} {nxt} {r.choice([0.0, 0.01, 1.0, 9.0])}")
        prev = nxt
    return "\n".join(lines) + "\n"
