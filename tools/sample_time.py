"""Measurement tool: asr_sample / asr_sample_entropy per-call time, back to back from Python (host
launch path included) vs replayed from a CUDA graph of 20 calls (device time per call)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import gen
from paper_2512_11221_b200 import asr_sample, asr_sample_entropy

V = 128256
for B in (1, 64):
    g = gen.GenParams(seed=7, L=1, Hq=2, Hkv=2, d=16, vocab=V)
    lg = torch.empty((B, V), dtype=torch.bfloat16, device="cuda")
    gen.dev_logits(g, B, 5, lg)
    u = torch.rand(B, device="cuda")
    tok = torch.empty(B, dtype=torch.int32, device="cuda")
    ent = torch.empty(B, dtype=torch.float32, device="cuda")
    for name, (T, k, P) in {"greedy": (0.0, 0, 1.0), "T0.8_k50_p0.9": (0.8, 50, 0.9), "T1_p0.95": (1.0, 0, 0.95)}.items():
        for fused in (False, True):
            def call():
                if fused:
                    asr_sample_entropy(lg, u, tok, ent, temperature=T, top_k=k, top_p=P)
                else:
                    asr_sample(lg, u, tok, temperature=T, top_k=k, top_p=P)
            for _ in range(3):
                call()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                call()
            e1.record()
            torch.cuda.synchronize()
            host = e0.elapsed_time(e1) * 1000 / 20
            s = torch.cuda.Stream()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(gr, stream=s):
                    for _ in range(20):
                        call()
            torch.cuda.synchronize()
            gr.replay()
            torch.cuda.synchronize()
            e0.record()
            gr.replay()
            e1.record()
            torch.cuda.synchronize()
            dev = e0.elapsed_time(e1) * 1000 / 20
            print(f"B={B} {name}{'+ent' if fused else ''}: back-to-back {host:.2f} us/call, graph {dev:.2f} us/call")
