"""NEXT-2 parity: the GPU policy-replay step (asr_step_policy: Alg. 1 lines 3-15 and the step-boundary
recovery with caller-supplied scores, no attention) against the oracle's policy-only step
(orc_step_policy), bitwise on lists and ledgers, over random below-tau traces, several (tau, K, k, W)
settings and planted entropy spikes."""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K,k,W,tick", [(8, 2.0, 0, 0), (16, 3.0, 0, 0), (4, 2.0, 32, 0), (8, 1.5, 0, 1)])
def test_policy_replay_matches_oracle(K, k, W, tick):
    import torch
    from paper_2512_11221_b200 import Config, Context
    B, P, steps, V = 3, 20, 180, 4096
    cap = P + steps + 1
    rng = np.random.default_rng(100 + K + W)
    gp = gen.GenParams(seed=51, L=1, Hq=2, Hkv=2, d=16, vocab=V, spike_first=60, spike_period=17, spike_count=4)
    cfg = Config(n_layers=1, n_q_heads=2, n_kv_heads=2, head_dim=16, batch=B, max_context=cap, window=K, tau=0.5,
                 softness=k, vocab=V, history_window=W, tick_order=tick, host_mirror=0)
    pk = torch.zeros((B, P, 1, 2, 16), dtype=torch.bfloat16, device="cuda")
    ctx = Context(cfg, pk, pk.clone(), [P] * B)
    orc = [oracle.OracleSeq(oracle.OrcCfg(L=1, Hq=2, Hkv=2, d=16, window=K, softness=k, vocab=V,
                                          history_window=W, tick_skip_new=tick), cap, P) for _ in range(B)]
    maxc = ctx.cfg.max_context
    for i in range(steps):
        below = (rng.random((B, cap)) < 0.75).astype(np.uint8)
        scores = np.where(below, 0.25, 1.0).astype(np.float32)          # |s - tau| = 0.25: no ambiguity
        sc = np.zeros((B, maxc), np.float32)   # rows of max_context (the ABI's layout)
        sc[:, :cap] = scores
        st = torch.from_numpy(sc).cuda()
        lg = None
        if i > 0:
            lg_np = np.stack([gen.logits(gp, b, i - 1) for b in range(B)])
            lg = torch.from_numpy(lg_np.view(np.int16)).view(torch.bfloat16).cuda()
        ent = torch.zeros(B, dtype=torch.float32, device="cuda")
        ctx.step_policy(st, logits_prev=lg, entropy=ent)
        for b in range(B):
            H = None if lg is None else oracle.entropy(lg_np[b])
            act, out = orc[b].step_policy(below[b], H)
            g = ctx.stats(b, detail=True)
            where = f"step {i} seq {b}"
            np.testing.assert_array_equal(g["active_list"], act, err_msg=where)
            led = orc[b].ledger()
            for key in ("residency", "timer", "count", "freeze_step"):
                np.testing.assert_array_equal(g["ledger"][key], led[key], err_msg=f"{where} {key}")
            assert g["active"] == out["active_post"] and g["frozen_this_step"] == out["frozen_this_step"], where
            assert g["recovery_action"] == out["recovery_action"], where


def test_policy_replay_full_size():
    """bench.py's replay point as it runs it: 1024 sequences grown from 512 to 8192 tokens on the
    all-cold trace (every score 0.25 < tau), K = 512, k = 2; sampled sequences' final ledgers and lists
    bit-exact against the oracle's policy replay (1349 active of 8192, the closed form of
    tests/test_oracle_policy.py), and every sequence's counts equal."""
    import torch
    from paper_2512_11221_b200 import Config, Context
    B, ctxlen, P = 1024, 8192, 512
    cfg = Config(n_layers=1, n_q_heads=2, n_kv_heads=2, head_dim=16, batch=B, max_context=ctxlen + 32 + 8,
                 window=512, tau=0.5, softness=2.0, vocab=0, host_mirror=0)
    pk = torch.zeros((B, P, 1, 2, 16), dtype=torch.bfloat16, device="cuda")
    ctx = Context(cfg, pk, pk.clone(), [P] * B)
    scores = torch.full((B, cfg.max_context), 0.25, dtype=torch.float32, device="cuda")
    s = oracle.OracleSeq(oracle.OrcCfg(L=1, Hq=2, Hkv=2, d=16, window=512, softness=2.0), cfg.max_context, P)
    below = np.ones(cfg.max_context, np.uint8)
    for _ in range(ctxlen - P):
        ctx.step_policy(scores)
        act, out = s.step_policy(below[:s.n + 1])
    torch.cuda.synchronize()
    assert out["n"] == ctxlen and out["active_post"] == 1349
    led = s.ledger()
    for b in (0, 1, 511, 1023):
        g = ctx.stats(b, detail=True)
        np.testing.assert_array_equal(g["active_list"], act, err_msg=f"seq {b}")
        for key in ("residency", "timer", "count", "freeze_step"):
            np.testing.assert_array_equal(g["ledger"][key], led[key], err_msg=f"seq {b} {key}")
        assert g["device_error"] == 0
    for b in range(B):
        g = ctx.stats(b)
        assert (g["total"], g["active"], g["attended"]) == (ctxlen, out["active_post"], out["attended"]), b
    ctx.close()
