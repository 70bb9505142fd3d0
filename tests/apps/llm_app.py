"""An ordinary PyTorch LLM-inference program (Llama-architecture model,
random weights, bf16) used to test the interposer with a real model stack:
cuBLASLt GEMMs, attention, RMSNorm, rotary embeddings, the caching
allocator. Each request is a forward pass over a fixed prompt; the logits
must equal the first request's bit for bit (same inputs, same kernels), so a
byte lost or misplaced by a context switch shows up. Knows nothing about
Nixie. Prints one JSON line.

Usage: llm_app.py <requests> <think_s> <seed> [preset] [batch] [seq]
  presets: small (0.75B), qwen3-8b (8.2B ~ 16 GiB bf16, the BASELINE config-2
  interactive app), flux-12b (12.8B ~ 24 GiB bf16, the config-2 background
  app's size)"""
import json
import sys
import time

import torch
from transformers import LlamaConfig, LlamaForCausalLM

PRESETS = {
    "small": dict(hidden_size=2048, intermediate_size=5632, num_hidden_layers=12, num_attention_heads=16,
                  num_key_value_heads=16, vocab_size=32000),
    "qwen3-8b": dict(hidden_size=4096, intermediate_size=12288, num_hidden_layers=36, num_attention_heads=32,
                     num_key_value_heads=8, vocab_size=151936),
    "flux-12b": dict(hidden_size=5120, intermediate_size=13824, num_hidden_layers=38, num_attention_heads=40,
                     num_key_value_heads=40, vocab_size=32000),
}


def main():
    requests = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    think = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
    seed = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    preset = sys.argv[4] if len(sys.argv) > 4 else "small"
    batch = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    seq = int(sys.argv[6]) if len(sys.argv) > 6 else 256
    torch.manual_seed(seed)
    cfg = LlamaConfig(max_position_embeddings=4096, **PRESETS[preset])
    t_init = time.perf_counter()
    torch.set_default_dtype(torch.bfloat16)
    with torch.device("cuda"):
        model = LlamaForCausalLM(cfg).eval()
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t_init
    params = sum(p.numel() for p in model.parameters())
    ids = torch.randint(0, cfg.vocab_size, (batch, seq), device="cuda", generator=torch.Generator(device="cuda").manual_seed(seed))
    ref = None
    bad = 0
    lat = []
    with torch.no_grad():
        for r in range(requests):
            t0 = time.perf_counter()
            logits = model(ids).logits[:, -1, :].float()
            torch.cuda.synchronize()
            lat.append((time.perf_counter() - t0) * 1e3)
            if ref is None:
                ref = logits.clone()
            else:
                bad += int(not torch.equal(logits, ref))
            time.sleep(think)
    s = sorted(lat)
    print(json.dumps({"name": f"llm_app:{preset}", "params": params, "weights_gib": round(params * 2 / 2**30, 2),
                      "requests": requests, "logit_mismatch": bad, "init_s": round(init_s, 2),
                      "request_ms": {"p50": s[len(s) // 2], "max": s[-1], "mean": sum(s) / len(s),
                                     "first": lat[0]},
                      "max_memory_allocated_gib": round(torch.cuda.max_memory_allocated() / 2**30, 2)}))
    return 0 if bad == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
