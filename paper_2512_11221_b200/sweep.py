"""NEXT-2: a (tau, K, k, W) sensitivity sweep over one relevance trace by policy
replay — PAPER.md §6 "Threshold Sensitivity. Performance depends on hyperparameters tau, K, and k"
(P:199); SPEC run_sweep: one replay per grid cell on a fixed trace, a table of
(parameters -> mean compression, max absence, recovery count), cells independent.

Every cell is one context of the C ABI (asr_create with the cell's window / tau / softness /
history_window) stepped with asr_step_policy: Alg. 1 lines 3-15 + the step-boundary recovery on the
GPU with the trace's scores instead of attention (no K/V).  Host code here only loops and reads the
per-step statistics; the cells' contexts step in lockstep, each on its own CUDA stream.
"""
from __future__ import annotations

import itertools

from .asr import Config, Context


def run_sweep(grid: dict, scores, steps: int, prompt: int, logits=None, vocab: int = 0, device: int = 0,
              base: Config | None = None) -> list[dict]:
    """grid: {"tau": [...], "window": [...], "softness": [...], "history_window": [...]} (missing keys: the
    base config's value); scores: fp32 CUDA tensor [batch][prompt + steps + 1] (s_j per position, the
    trace); logits: optional callable step -> bf16 CUDA tensor [batch][vocab] (the entropy detector's
    input, e.g. planted spikes), vocab its width.  Returns one row per cell: the parameters, mean
    compression over the steps (1 - active/total after each step, mean over sequences), the largest
    remaining absence seen (max timer of the final ledgers), recovery actions (count over sequences),
    the final active / total of sequence 0 and its post-step active count after every step."""
    import torch
    keys = ("tau", "window", "softness", "history_window")
    base = base or Config(n_layers=1, n_q_heads=2, n_kv_heads=2, head_dim=16, vocab=vocab, host_mirror=0)
    B = int(scores.shape[0])
    cap = prompt + steps + 1
    assert scores.shape[1] >= cap, "scores must cover every position the steps append"
    cells = list(itertools.product(*[grid.get(k, [getattr(base, k)]) for k in keys]))
    ctxs, streams = [], []
    zeros = torch.zeros((B, max(prompt, 1), base.n_layers, base.n_kv_heads, base.head_dim), dtype=torch.bfloat16,
                        device=f"cuda:{device}")
    for cell in cells:
        kw = {**{f: getattr(base, f) for f in base.__dataclass_fields__}, **dict(zip(keys, cell))}
        kw.update(batch=B, max_context=cap, device=device, vocab=vocab if logits is not None else 0, host_mirror=0,
                  wr_window=None)
        ctxs.append(Context(Config(**kw), zeros, zeros, [prompt] * B))
        streams.append(torch.cuda.Stream(device=device))
    rows = [{"tau": c[0], "window": c[1], "softness": c[2], "history_window": c[3], "compression_sum": 0.0,
             "recoveries": 0, "active_trace": []} for c in cells]
    sc = scores[:, :cap].contiguous()   # rows of max_context (asr_step_policy's layout)
    for i in range(steps):
        lg = logits(i - 1) if (logits is not None and i > 0) else None
        for ctx, st in zip(ctxs, streams):
            with torch.cuda.stream(st):
                ctx.step_policy(sc, logits_prev=lg)
        for ctx, row in zip(ctxs, rows):
            for b in range(B):
                s = ctx.stats(b)
                row["compression_sum"] += s["compression"] / B
                row["recoveries"] += int(s["recovery_action"] > 0)
                if b == 0:
                    row["active_trace"].append(int(s["active"]))
    for ctx, row in zip(ctxs, rows):
        led = [ctx.stats(b, detail=True)["ledger"] for b in range(B)]
        row["mean_compression"] = row.pop("compression_sum") / steps
        row["max_absence"] = int(max(int(l["timer"].max()) for l in led))
        s0 = ctx.stats(0)
        row["final_active"], row["final_total"] = int(s0["active"]), int(s0["total"])
        ctx.close()
    return rows
