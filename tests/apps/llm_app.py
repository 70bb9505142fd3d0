"""An ordinary PyTorch LLM-inference program (Llama-architecture model,
random weights, bf16) used to test the interposer with a real model stack:
cuBLASLt GEMMs, attention, RMSNorm, rotary embeddings, the caching
allocator. Each request is a forward pass over a fixed prompt; the logits
must equal the first request's bit for bit (same inputs, same kernels), so a
byte lost or misplaced by a context switch shows up. Knows nothing about
Nixie. Prints one JSON line.
Usage: llm_app.py <requests> <think_s> <seed>"""
import json
import sys
import time

import torch
from transformers import LlamaConfig, LlamaForCausalLM


def main():
    requests = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    think = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
    seed = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    torch.manual_seed(seed)
    cfg = LlamaConfig(hidden_size=2048, intermediate_size=5632, num_hidden_layers=12, num_attention_heads=16,
                      num_key_value_heads=16, vocab_size=32000, max_position_embeddings=1024)
    model = LlamaForCausalLM(cfg).to(device="cuda", dtype=torch.bfloat16).eval()
    params = sum(p.numel() for p in model.parameters())
    ids = torch.randint(0, cfg.vocab_size, (2, 256), device="cuda", generator=torch.Generator(device="cuda").manual_seed(seed))
    ref = None
    bad = 0
    lat = []
    with torch.no_grad():
        for r in range(requests):
            t0 = time.perf_counter()
            logits = model(ids).logits.float()
            torch.cuda.synchronize()
            lat.append((time.perf_counter() - t0) * 1e3)
            if ref is None:
                ref = logits.clone()
            else:
                bad += int(not torch.equal(logits, ref))
            time.sleep(think)
    print(json.dumps({"name": "llm_app", "params": params, "requests": requests, "logit_mismatch": bad,
                      "request_ms": {"max": max(lat), "median": sorted(lat)[len(lat) // 2]},
                      "max_memory_allocated": torch.cuda.max_memory_allocated()}))
    return 0 if bad == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
