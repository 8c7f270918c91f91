"""Measurement tool: a few asr_sample calls at the LLaMA-3 vocabulary for ncu.
Usage: python tools/sample_probe.py [batch] [temperature] [top_k] [top_p]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import gen  # noqa: E402
from paper_2512_11221_b200 import asr_sample  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
T = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
K = int(sys.argv[3]) if len(sys.argv) > 3 else 0
P = float(sys.argv[4]) if len(sys.argv) > 4 else 0.95
V = 128256
g = gen.GenParams(seed=7, L=1, Hq=2, Hkv=2, d=16, vocab=V)
lg = torch.empty((B, V), dtype=torch.bfloat16, device="cuda")
gen.dev_logits(g, B, 5, lg)
u = torch.rand(B, device="cuda")
tok = torch.empty(B, dtype=torch.int32, device="cuda")
for _ in range(3):
    asr_sample(lg, u, tok, temperature=T, top_k=K, top_p=P)
torch.cuda.synchronize()
print("ok", tok[:4].tolist())
