"""Measurement tool: a few asr_sample calls (batch 64, LLaMA-3 vocabulary) for ncu."""
import torch

import gen
from paper_2512_11221_b200 import asr_sample

B, V = 64, 128256
g = gen.GenParams(seed=7, L=1, Hq=2, Hkv=2, d=16, vocab=V)
lg = torch.empty((B, V), dtype=torch.bfloat16, device="cuda")
gen.dev_logits(g, B, 5, lg)
u = torch.rand(B, device="cuda")
tok = torch.empty(B, dtype=torch.int32, device="cuda")
for _ in range(3):
    asr_sample(lg, u, tok, temperature=1.0, top_k=0, top_p=0.95)
torch.cuda.synchronize()
print("ok", tok[:4].tolist())
