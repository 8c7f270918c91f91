"""Parity harness: drives the CUDA path (through the C ABI) and the fp64 oracle on the same seeded
inputs, step by step, and compares them element by element.

Bars (BASELINE.json north_star):
- attended index lists, ledgers (residency, timer, count, freeze step) and per-step counters:
  bit-exact;
- Eq. 2 scores: exactly equal on LAT inputs (exact in fp32 in any summation order);
- attention O: max over (b, l, h) of max_e |o - o*| / max_e |o*|  <= 2e-3 (bf16 KV) / 1e-5 (fp32 KV);
- entropy: |H - H*| <= 1e-4 nats.
"""
from __future__ import annotations

import dataclasses

import numpy as np

import gen
import oracle

TOL_O = {"bf16": 2e-3, "f32": 1e-5}
TOL_H = 1e-4


@dataclasses.dataclass
class Case:
    L: int = 1
    Hq: int = 2
    Hkv: int = 2
    d: int = 16
    B: int = 1
    prompt: tuple = (32,)
    steps: int = 32
    window: int = 16
    tau: float = 0.5
    softness: float = 2.0
    dtype: str = "bf16"
    seed: int = 1001
    family: int = gen.LAT
    hot_permille: int = 0
    a_hot: int = 4
    vocab: int = 0
    spike_first: int = -1
    spike_period: int = 0
    spike_count: int = 0
    needle_pos: int = -1
    query_first: int = -1
    query_count: int = 0
    tick_order: int = 0
    score_mode: int = 0
    pinned_prefix: int = 0
    wr_window: int | None = None
    host_io: bool = False          # pass host (numpy) buffers through the C ABI
    restore_at: dict = dataclasses.field(default_factory=dict)  # step -> (seq, level) explicit restore
    max_context: int = 0
    pool_tokens: int = 0           # > 0: pressure mode (device slot pool, eviction / prefetch / demand)
    evict_min: int = 2
    evict_policy: int = 0          # 0 Belady under pressure, 1 evict at freeze (round-1 policy)
    pool_reserve: int = 0
    nccl_world1: bool = False      # attach a one-rank NCCL communicator (attend -> all-reduce -> decide)
    logits_dtype: str = "bf16"     # "f32": the same (bf16-exact) logits passed as fp32
    history_window: int = 0        # W (NEXT-3): 0 = lifetime counts
    time_attention_at: tuple = ()  # steps before which asr_time_attention runs (must leave no trace)
    fr_clear_counts: int = 0       # FR also clears the detection counts (SPEC S:391 reading)
    entropy_given: bool = False    # H taken by asr_sample_entropy (with a draw) and passed to the step
    mirror_bits: int = 0           # 8: the INT8 frozen tier (restored tokens come back dequantised)

    def gen_params(self) -> gen.GenParams:
        return gen.GenParams(seed=self.seed, family=self.family, L=self.L, Hq=self.Hq, Hkv=self.Hkv, d=self.d,
                             hot_permille=self.hot_permille, a_hot=self.a_hot, needle_pos=self.needle_pos,
                             query_first=self.query_first, query_count=self.query_count, vocab=self.vocab,
                             spike_first=self.spike_first, spike_period=self.spike_period,
                             spike_count=self.spike_count)

    def capacity(self) -> int:
        return self.max_context or (max(self.prompt) + self.steps + 1)


def orc_cfg(c: Case) -> oracle.OrcCfg:
    return oracle.OrcCfg(L=c.L, Hq=c.Hq, Hkv=c.Hkv, d=c.d, window=c.window, tau=c.tau, softness=c.softness,
                         pinned_prefix=c.pinned_prefix, score_scaled=c.score_mode, tick_skip_new=c.tick_order,
                         vocab=c.vocab, wr_window=c.wr_window, history_window=c.history_window,
                         fr_clear_counts=c.fr_clear_counts)


def asr_cfg(c: Case):
    from paper_2512_11221_b200 import Config, KV_BF16, KV_F32
    return Config(n_layers=c.L, n_q_heads=c.Hq, n_kv_heads=c.Hkv, head_dim=c.d, batch=c.B,
                  max_context=c.capacity(), kv_dtype=KV_BF16 if c.dtype == "bf16" else KV_F32,
                  window=c.window, tau=c.tau, softness=c.softness, pinned_prefix=c.pinned_prefix,
                  score_mode=c.score_mode, tick_order=c.tick_order, vocab=c.vocab, wr_window=c.wr_window,
                  pool_tokens=c.pool_tokens, evict_min_absence=c.evict_min, history_window=c.history_window,
                  fr_clear_counts=c.fr_clear_counts, evict_policy=c.evict_policy, pool_reserve=c.pool_reserve,
                  mirror_bits=c.mirror_bits)


def o_rel_err(o: np.ndarray, o_ref: np.ndarray) -> float:
    """max over rows (b, l, h) of max_e |o - o*| / max_e |o*|."""
    num = np.abs(o.astype(np.float64) - o_ref).max(-1)
    den = np.abs(o_ref).max(-1)
    return float((num / den).max())


def run(c: Case, check_o: bool = True) -> dict:
    """Run c.steps steps on GPU and oracle; assert parity at every step.  Returns a summary."""
    import torch
    from paper_2512_11221_b200 import Context

    p = c.gen_params()
    cap = c.capacity()
    P = list(c.prompt)
    assert len(P) == c.B
    Pmax = max(P)
    npd = np.uint16 if c.dtype == "bf16" else np.float32
    tdt = torch.bfloat16 if c.dtype == "bf16" else torch.float32
    # full K/V per sequence (positions beyond n are unused until appended)
    KV = [gen.kv(p, b, 0, cap, c.dtype) for b in range(c.B)]
    pk = np.zeros((c.B, max(Pmax, 1), c.L, c.Hkv, c.d), npd)
    pv = np.zeros_like(pk)
    for b in range(c.B):
        pk[b, :P[b]] = KV[b][0][:P[b]]
        pv[b, :P[b]] = KV[b][1][:P[b]]

    def to_t(a):
        t = torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a)
        t = t.view(torch.bfloat16) if a.dtype == np.uint16 else t
        return t if c.host_io else t.cuda()

    ctx = Context(asr_cfg(c), to_t(pk), to_t(pv), P)
    # INT8 tier: a token copied back from the quantised mirror is attended with its R-quant
    # dequantised rows (oracle/quant.py); the oracle is given exactly those values for the tokens the
    # device flags (asr_ledger_view.dequantized), the appended values for all others
    KVq, KVo = None, KV
    if c.mirror_bits == 8:
        from oracle import quant

        def deq(a):   # [n][L][Hkv][d] bf16 bits -> the same, every row through R-quant INT8
            rows = a.reshape(-1, c.d)
            codes, scales = quant.quantize(rows, 8)
            return quant.dequantize(codes, scales).reshape(a.shape)
        KVq = [(deq(KV[b][0]), deq(KV[b][1])) for b in range(c.B)]
        KVo = [(KV[b][0].copy(), KV[b][1].copy()) for b in range(c.B)]
    if c.nccl_world1:
        from paper_2512_11221_b200 import asr_nccl_unique_id
        ctx.attach_nccl(asr_nccl_unique_id(), 1, 0)
    orc = [oracle.OracleSeq(orc_cfg(c), cap, P[b]) for b in range(c.B)]
    worst_o, worst_h, frozen_total, restored_total = 0.0, 0.0, 0, 0
    evicted_total = prefetched_total = demand_total = 0
    recoveries = 0
    tiles = []
    for i in range(c.steps):
        if i in c.time_attention_at:
            ctx.time_attention(2)
        if i in c.restore_at:
            seq, level = c.restore_at[i]
            ctx.restore(seq, level)
            for b in range(c.B):
                if seq < 0 or seq == b:
                    orc[b].restore(level)
        q = np.stack([gen.q(p, b, i, c.dtype) for b in range(c.B)])
        kn = np.stack([KV[b][0][P[b] + i] for b in range(c.B)])
        vn = np.stack([KV[b][1][P[b] + i] for b in range(c.B)])
        lg = np.stack([gen.logits(p, b, i - 1, c.logits_dtype) for b in range(c.B)]) if (c.vocab and i > 0) else None
        if c.host_io:
            o = np.zeros((c.B, c.L, c.Hq, c.d), np.float32)
            ent = np.zeros(c.B, np.float32)
            ctx.step(q, kn, vn, o, logits_prev=lg, entropy=ent)
        elif c.entropy_given and lg is not None:
            # NEXT-1 fused with (a6): one read of each logits row yields the next token and H
            from paper_2512_11221_b200 import asr_sample_entropy
            o_t = torch.zeros((c.B, c.L, c.Hq, c.d), dtype=torch.float32, device="cuda")
            e_t = torch.zeros(c.B, dtype=torch.float32, device="cuda")
            h_t = torch.empty(c.B, dtype=torch.float32, device="cuda")
            tok = torch.empty(c.B, dtype=torch.int32, device="cuda")
            asr_sample_entropy(to_t(lg), torch.full((c.B,), 0.5, device="cuda"), tok, h_t, temperature=0.8, top_k=50,
                               top_p=0.9)
            ctx.step(to_t(q), to_t(kn), to_t(vn), o_t, logits_prev=h_t, entropy=e_t, entropy_given=True)
        else:
            o_t = torch.zeros((c.B, c.L, c.Hq, c.d), dtype=torch.float32, device="cuda")
            e_t = torch.zeros(c.B, dtype=torch.float32, device="cuda")
            ctx.step(to_t(q), to_t(kn), to_t(vn), o_t, logits_prev=None if lg is None else to_t(lg),
                     entropy=e_t)
        stats = [ctx.stats(b, detail=True) for b in range(c.B)]
        tiles.append(sum(c.L * ((g["attended"] + 15) // 16) for g in stats))   # the attention's work items
        if not c.host_io:
            o = o_t.cpu().numpy()
            ent = e_t.cpu().numpy()
        for b in range(c.B):
            if KVq is not None:   # the tokens the device now holds dequantised
                fl = np.flatnonzero(stats[b]["dequantized"])
                KVo[b][0][fl], KVo[b][1][fl] = KVq[b][0][fl], KVq[b][1][fl]
            Ob, act, scores, out = orc[b].step(q[b], KVo[b][0], KVo[b][1], None if lg is None else lg[b])
            g = stats[b]
            where = f"step {i} seq {b}"
            np.testing.assert_array_equal(g["active_list"], act, err_msg=where)
            # the sums are exact on LAT inputs; the mean is one correctly rounded fp32 division
            sc32 = scores.astype(np.float32)
            assert np.array_equal(g["scores"], sc32), \
                f"{where}: scores differ at {np.flatnonzero(g['scores'] != sc32)[:5]}"
            led = orc[b].ledger()
            for key in ("residency", "timer", "count", "freeze_step"):
                np.testing.assert_array_equal(g["ledger"][key], led[key], err_msg=f"{where} {key}")
            assert g["total"] == out["n"] and g["attended"] == out["attended"], where
            assert g["active"] == out["active_post"] and g["frozen"] == out["frozen_post"], where
            assert g["frozen_this_step"] == out["frozen_this_step"], where
            assert g["restored_this_step"] == out["restored_this_step"], (where, g, out)
            assert g["recovery_action"] == out["recovery_action"], where
            recoveries += out["recovery_action"] > 0
            assert g["rewalk_requested"] == out["rewalk_requested"], where
            assert g["device_error"] == 0
            if out["entropy_valid"]:
                assert g["entropy_valid"] == 1
                dh = abs(float(g["entropy"]) - out["entropy"])
                assert dh <= TOL_H, (where, dh)
                assert abs(float(ent[b]) - out["entropy"]) <= TOL_H
                worst_h = max(worst_h, dh)
            if check_o:
                err = o_rel_err(o[b], Ob)
                assert err <= TOL_O[c.dtype], (where, err)
                worst_o = max(worst_o, err)
            frozen_total += out["frozen_this_step"]
            restored_total += out["restored_this_step"]
            if c.pool_tokens:
                assert g["resident"] <= c.pool_tokens, where
                # every attended token held a device slot (else the device would have latched an error)
                assert g["resident"] >= g["active"], where
                evicted_total += g["evicted_this_step"]
                assert g["free_slots"] >= 0, where
                prefetched_total += g["prefetched_this_step"]
                demand_total += g["demand_restored_this_step"]
    # exact restoration ("no permanent information loss"): every stored token's bytes, on the
    # device (resident tokens, including ones evicted and copied back) and in the host mirror, equal
    # what was appended
    for b in range(c.B):
        n = P[b] + c.steps
        led = ctx.stats(b, detail=True)["ledger"]
        mir = KVq[b] if KVq is not None else KV[b]   # INT8 tier: the mirror holds R-quant rows exactly
        for j in range(n):
            km, vm = ctx.read_kv(b, j, from_mirror=True)
            np.testing.assert_array_equal(km, mir[0][j], err_msg=f"mirror K seq {b} pos {j}")
            np.testing.assert_array_equal(vm, mir[1][j], err_msg=f"mirror V seq {b} pos {j}")
            try:
                kd, vd = ctx.read_kv(b, j)
            except Exception:
                assert c.pool_tokens and led["residency"][j] == 0, (b, j)   # only frozen tokens may be evicted
                continue
            np.testing.assert_array_equal(kd, KVo[b][0][j], err_msg=f"device K seq {b} pos {j}")
            np.testing.assert_array_equal(vd, KVo[b][1][j], err_msg=f"device V seq {b} pos {j}")
    summary = {"worst_o": worst_o, "worst_h": worst_h, "frozen": frozen_total, "restored": restored_total,
               "recoveries": recoveries, "tiles": tiles,
               "evicted": evicted_total, "prefetched": prefetched_total, "demand": demand_total,
               "final": [ctx.stats(b) for b in range(c.B)]}
    ctx.close()
    return summary
