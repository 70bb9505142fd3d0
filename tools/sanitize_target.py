"""Small swap workload for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel family on tiny sizes. K1 (SM swap, fused
checksum), K3 per-batch and grouped table launches (CE path), K4 fill /
compare, prefetch; restores verified byte-exact."""
import sys
sys.path.insert(0, ".")
from paper_2601_11743_b200 import MIB, PlannerConfig, SwapEngine
from paper_2601_11743_b200._lib import PATH_CE, PATH_SM, TIER_GPU, TIER_PAGED, TIER_PINNED

for opts in (dict(path=PATH_SM), dict(path=PATH_CE, k3_grouped=False), dict(path=PATH_CE, k3_grouped=True),
             dict(path=PATH_CE, pace_lag_legs=2, first_batch_legs=1, d2h_commit_legs=1)):  # paced, tiny groups
    with SwapEngine(gpu_capacity=32 * MIB, pinned_capacity=48 * MIB, paged_capacity=64 * MIB, **opts) as e:
        e.allocate(0, 32 * MIB, TIER_GPU)
        e.allocate(1, 24 * MIB, TIER_PINNED)
        e.allocate(2, 16 * MIB, TIER_PAGED)
        for a in (0, 1, 2):
            e.fill_pattern(a, 7)
        pc = PlannerConfig(streaming_window=4 * MIB)
        for to, victims in ((1, [0, 2]), (2, [0, 1]), (0, [1, 2])):
            pc.victim_order = victims
            st = e.switch_to(to, pc)
            assert st["mismatches"] == 0, st
        e.prefetch_begin(1, pc)
        pc.victim_order = [0, 2]
        e.switch_to(1, pc)
        for a in (0, 1, 2):
            assert e.verify_pattern(a, 7) == 0
        print(opts, "ok", flush=True)
