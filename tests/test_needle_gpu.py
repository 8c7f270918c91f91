"""BASELINE.json configs[3] analogue: 32K context, prefill state, needle-in-haystack restore pattern
with entropy-triggered recovery, checked against the oracle.

The whole 32K prompt is Active at step 0 (prefill, R-prefill), so the prompt cohort freezes and
returns in lockstep.  The needle is a prompt token at position 16384 (LAT needle key
k[1] = 128).  q = the first step whose tick leaves the needle frozen with timer >= 2 — the oracle's
policy replay finds it; a spike planted in logits_q makes step q+1's detector fire SR, which restores
the needle at the q/q+1 boundary (needle in A_{q+1}) while the retrieval queries (q[1] = 7/16) of steps
q+1 .. q+8 give it a score far above tau.  Further spikes every 16 steps climb WR, FR, RR.

Reduced shape for the oracle's sake: 2 layers of the LLaMA head layout (32 q / 8 KV heads, d=128 —
the MMA attention path), batch 2.  Ledgers and lists are compared bitwise at every step (oracle
policy replay, whose class labels the LAT construction guarantees); attention outputs are compared
with full fp64 oracle steps on the steps around q.
"""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu

CTX, K, NEEDLE, V = 32768, 512, 16384, 128256
L, HQ, HKV, D, B = 2, 32, 8, 128, 2


def find_q(P):
    cfg = oracle.OrcCfg(L=L, Hq=HQ, Hkv=HKV, d=D, window=K)
    s = oracle.OracleSeq(cfg, P + 400, P)
    below = np.ones(P + 400, np.uint8)
    for i in range(300):
        s.step_policy(below)
        led = s.ledger()
        if led["residency"][NEEDLE] == 0 and led["timer"][NEEDLE] >= 2:
            return i
    raise AssertionError("needle never frozen for >= 2 steps")


@pytest.mark.parametrize("pool", [0, 1])
def test_needle_restore_ladder_32k(pool):
    import torch
    from paper_2512_11221_b200 import Config, Context

    P = CTX - 256
    q = find_q(P)
    assert q == 55   # SURVEY A.6 (prefill lockstep, d = 3 from c = 36): bench.py's configs[3] point relies on it
    steps = q + 56
    p = gen.GenParams(seed=4001, L=L, Hq=HQ, Hkv=HKV, d=D, needle_pos=NEEDLE, query_first=q + 1, query_count=8,
                      vocab=V, spike_first=q, spike_period=16, spike_count=4)
    cap = P + steps + 1
    KVs = [gen.kv(p, b, 0, cap) for b in range(B)]
    to_t = lambda a: torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda()
    pk = torch.stack([to_t(KVs[b][0][:P]) for b in range(B)])
    pv = torch.stack([to_t(KVs[b][1][:P]) for b in range(B)])
    cfg = Config(n_layers=L, n_q_heads=HQ, n_kv_heads=HKV, head_dim=D, batch=B, max_context=cap, window=K, vocab=V,
                 pool_tokens=(B * cap + 4 * B) if pool else 0, evict_min_absence=2,
                 evict_policy=1)   # at-freeze eviction: the pool holds everything, Belady would evict nothing
    ctx = Context(cfg, pk, pv, [P] * B)
    del pk, pv
    ocfg = oracle.OrcCfg(L=L, Hq=HQ, Hkv=HKV, d=D, window=K, vocab=V)
    orc = [oracle.OracleSeq(ocfg, cap, P) for _ in range(B)]
    o_t = torch.zeros((B, L, HQ, D), dtype=torch.float32, device="cuda")
    actions, needle_in, needle_state = [], {}, {}
    full_steps = {q, q + 1, q + 2}
    demand = 0
    for i in range(steps):
        qn = np.stack([gen.q(p, b, i) for b in range(B)])
        kn = np.stack([KVs[b][0][P + i] for b in range(B)])
        vn = np.stack([KVs[b][1][P + i] for b in range(B)])
        lg = np.stack([gen.logits(p, b, i - 1) for b in range(B)]) if i > 0 else None
        ctx.step(to_t(qn), to_t(kn), to_t(vn), o_t, logits_prev=None if lg is None else to_t(lg))
        o = o_t.cpu().numpy()
        for b in range(B):
            g = ctx.stats(b, detail=True)
            if i in full_steps:
                O, act, scores, out = orc[b].step(qn[b], KVs[b][0], KVs[b][1], None if lg is None else lg[b])
                rel = (np.abs(o[b] - O).max(-1) / np.abs(O).max(-1)).max()
                assert rel <= 2e-3, (i, b, rel)
                np.testing.assert_array_equal(g["scores"], scores.astype(np.float32))
            else:
                H = oracle.entropy(lg[b]) if lg is not None else None
                # class labels of the LAT construction: every eligible token scores below tau except the
                # needle on its retrieval steps
                below = np.ones(cap, np.uint8)
                if gen.is_query_step(p, i):
                    below[NEEDLE] = 0
                act, out = orc[b].step_policy(below, H)
            np.testing.assert_array_equal(g["active_list"], act, err_msg=f"step {i} seq {b}")
            led = orc[b].ledger()
            for key in ("residency", "timer", "count", "freeze_step"):
                np.testing.assert_array_equal(g["ledger"][key], led[key], err_msg=f"step {i} seq {b} {key}")
            assert g["recovery_action"] == out["recovery_action"] and g["attended"] == out["attended"]
            assert g["device_error"] == 0
            if b == 0:
                needle_in[i] = bool(np.isin(NEEDLE, act))
                needle_state[i] = (int(g["ledger"]["residency"][NEEDLE]), int(g["ledger"]["timer"][NEEDLE]))
                if out["recovery_action"]:
                    actions.append((i, out["recovery_action"]))
            demand += g["demand_restored_this_step"]
    # after step q the needle is frozen with timer >= 2 (it would miss step q+1); SR at the q/q+1
    # boundary restores it, so it is attended at q+1 and scores far above tau on its retrieval steps
    assert needle_state[q][0] == 0 and needle_state[q][1] >= 2
    assert needle_in[q + 1] and needle_state[q + 1] == (1, 0)
    assert actions == [(q + 1, 1), (q + 17, 2), (q + 33, 3), (q + 49, 4)]
    if pool:
        assert demand > 0   # SR / WR / FR copied evicted tokens back from the host mirror
    ctx.close()


def test_needle_full_depth_32_layers():
    """configs[3] at full depth: 32 layers of the LLaMA-3-8B shape, batch 2, the 32K prefill with the
    needle, bench.py's launch (device-generated prompt and inputs).  Ledgers and attended lists of
    every step bit-exact against the oracle's policy replay (LAT classes; the needle scores high on
    its retrieval steps only); O of sampled (layer, head) rows at steps q, q+1 (SR restores the
    needle's cohort: |A| jumps to the whole context) and q+2 against oracle.attend_head."""
    import torch
    from paper_2512_11221_b200 import Config, Context

    L32 = 32
    P = CTX - 256
    q = find_q(P)
    steps = q + 20
    p = gen.GenParams(seed=4002, L=L32, Hq=HQ, Hkv=HKV, d=D, needle_pos=NEEDLE, query_first=q + 1, query_count=8,
                      vocab=V, spike_first=q, spike_period=16, spike_count=2)
    cap = P + steps + 1
    cfg = Config(n_layers=L32, n_q_heads=HQ, n_kv_heads=HKV, head_dim=D, batch=B, max_context=cap, window=K, vocab=V,
                 host_mirror=0)
    bf = torch.bfloat16
    pk = torch.empty((B, P, L32, HKV, D), dtype=bf, device="cuda")
    pv = torch.empty_like(pk)
    gen.dev_kv(p, B, 0, P, pk, pv)
    torch.cuda.synchronize()
    ctx = Context(cfg, pk, pv, [P] * B)
    del pk, pv
    torch.cuda.empty_cache()
    qd = torch.empty((B, L32, HQ, D), dtype=bf, device="cuda")
    kn = torch.empty((B, L32, HKV, D), dtype=bf, device="cuda")
    vn = torch.empty_like(kn)
    lg = torch.empty((B, V), dtype=bf, device="cuda")
    o = torch.empty((B, L32, HQ, D), dtype=torch.float32, device="cuda")
    pos = torch.full((B,), P, dtype=torch.int32, device="cuda")
    ocfg = oracle.OrcCfg(L=L32, Hq=HQ, Hkv=HKV, d=D, window=K, vocab=V)
    orc = [oracle.OracleSeq(ocfg, cap, P) for _ in range(B)]
    checks = {q: None, q + 1: None, q + 2: None}
    kv_host = {}
    actions = []
    rng = np.random.default_rng(7)
    for i in range(steps):
        gen.dev_q(p, B, i, qd)
        gen.dev_kv(p, B, 0, 1, kn, vn, pos0_dev=pos + i)
        gen.dev_logits(p, B, i - 1, lg)
        ctx.step(qd, kn, vn, o, logits_prev=lg if i > 0 else None)
        O = o.cpu().numpy() if i in checks else None
        for b in range(B):
            H = oracle.entropy(gen.logits(p, b, i - 1)) if i > 0 else None
            below = np.ones(cap, np.uint8)
            if gen.is_query_step(p, i):
                below[NEEDLE] = 0
            act, out = orc[b].step_policy(below, H)
            g = ctx.stats(b, detail=True)
            np.testing.assert_array_equal(g["active_list"], act, err_msg=f"step {i} seq {b}")
            led = orc[b].ledger()
            for key in ("residency", "timer", "count", "freeze_step"):
                np.testing.assert_array_equal(g["ledger"][key], led[key], err_msg=f"step {i} seq {b} {key}")
            assert g["recovery_action"] == out["recovery_action"] and g["device_error"] == 0
            if b == 0 and out["recovery_action"]:
                actions.append((i, out["recovery_action"]))
            if O is not None:
                qb = gen.q(p, b, i)
                if b not in kv_host:   # every position's K/V rows, host build of the generator (4.3 GB)
                    kv_host[b] = gen.kv(p, b, 0, cap)
                Kb, Vb = kv_host[b][0][act], kv_host[b][1][act]
                rows = {(0, 0), (L32 - 1, HQ - 1), *[(int(x), int(y)) for x, y in rng.integers(0, [L32, HQ], (14, 2))]}
                for l, h in sorted(rows):
                    kvh = h // (HQ // HKV)
                    ref = oracle.attend_head(qb[l, h], Kb[:, l, kvh], Vb[:, l, kvh])
                    err = float(np.max(np.abs(O[b, l, h] - ref)) / np.max(np.abs(ref)))
                    assert err <= 2e-3, (i, b, l, h, err)
                if b == 0 and i == q + 1:
                    assert NEEDLE in act   # SR at the q/q+1 boundary restored the needle
    assert actions == [(q + 1, 1), (q + 17, 2)]
    ctx.close()
