# BASELINE.json configs[2] with MLFQ prefetch (PAPER.md:273): 3-app mix on one GPU capped at 32 GiB, MLFQ with
# the paper's constants (K=4, T[1]=8 s, S[1]=4 s, idle 100 ms, tick 10 ms).
#   app 0 code completion: 16 GiB (Qwen3-8B bf16-sized), a request every 3 s
#         (+-10%), 5 kernels of 20 ms each (SPEC.md:479 Interactive archetype)
#   app 1 image generation: 24 GiB (FLUX-sized), a request every 12 s, 40 kernels of 50 ms
#   app 2 batch OCR: 12 GiB, never thinks, 16 kernels of 40 ms between syncs
# Links: PCIe 64 GiB/s per direction full duplex (the reference's default
# modeled link), host pinned<->pageable 32 GiB/s (transfer.hpp:27-28).
capacity gpu 32GiB
capacity pinned 16GiB
capacity paged 256GiB
link 0 64GiB/s 64GiB/s full
link 1 32GiB/s 32GiB/s full
dispatch 5e-6
mlfq 4 8 4 0.1 0.01
seed 0x4E495849
horizon 60
prefetch on
interactive 0 16GiB paged 0.0 3 5 0.02 0.1
interactive 1 24GiB paged 0.3 12 40 0.05 0.1
batch 2 12GiB paged 0.6 0.04 16
