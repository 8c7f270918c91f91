"""Pins for the oracle's attention (Eq. 1, over A_i per Alg. 1 line 1) and score
(Eq. 2).

Pinned against: SPEC worked examples, textbook special cases (singleton
softmax = identity, equal logits = mean, two-token softmax = logistic of the scaled logit gap),
an independent formulation (full attention over all positions with frozen logits at -inf,
S:287, written in numpy), affine equivariance of attention in V, head-permutation invariance and
homogeneity of Eq. 2, the GQA mapping, and the LAT generator's provable score bounds.
"""
import json
import math
import os

import numpy as np
import pytest

import gen
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def f32(a):
    return np.ascontiguousarray(np.asarray(a, np.float32))


def one_step(cfg, K, V, q, P):
    """Prefill P tokens from K/V[:P], then one step appending position P; returns outputs."""
    cap = K.shape[0]
    s = oracle.OracleSeq(cfg, cap, P)
    return s.step(f32(q), f32(K), f32(V))


def test_spec_score_examples():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))["score_raw"]
    for case in g["cases"]:
        H = case["H"]
        d = len(case["q"][0])
        cfg = oracle.OrcCfg(L=1, Hq=H, Hkv=H, d=d, window=1, tau=-1.0)
        # position 0 holds the example key; position 1 is the new token (protected)
        K = np.zeros((2, 1, H, d), np.float32)
        K[0, 0] = np.array(case["k"], np.float32)
        V = np.zeros_like(K)
        q = np.array(case["q"], np.float32)[None]
        O, act, scores, out = one_step(cfg, K, V, q, 1)
        assert list(act) == [0, 1]
        assert scores[0] == case["s"]


def test_score_invariants_and_gqa():
    rng = np.random.default_rng(3)
    L, Hq, Hkv, d, n = 2, 8, 2, 16, 12
    cfg = oracle.OrcCfg(L=L, Hq=Hq, Hkv=Hkv, d=d, window=1, tau=-1.0)
    K = rng.integers(-8, 9, (n, L, Hkv, d)).astype(np.float32) / 16
    V = rng.standard_normal((n, L, Hkv, d)).astype(np.float32)
    q = rng.integers(-8, 9, (L, Hq, d)).astype(np.float32) / 16
    _, _, s0, _ = one_step(cfg, K, V, q, n - 1)
    # homogeneity: s(alpha q) = alpha s(q)
    _, _, s2, _ = one_step(cfg, K, V, 2 * q, n - 1)
    np.testing.assert_array_equal(s2, 2 * s0)
    # permuting query heads inside a GQA group leaves every s_j unchanged
    perm = np.arange(Hq).reshape(Hkv, -1)[:, ::-1].ravel()
    _, _, s3, _ = one_step(cfg, K, V, q[:, perm], n - 1)
    np.testing.assert_array_equal(s3, s0)
    # GQA map: only KV head 1 nonzero -> only query heads 4..7 contribute; with q = 1/16 and
    # k = 1/16 on every coordinate each dot is d/256, so s = (4 heads * L layers * d/256)/(L*Hq)
    K1 = np.zeros_like(K)
    K1[:, :, 1, :] = 1 / 16
    q1 = np.full_like(q, 1 / 16)
    _, _, s4, _ = one_step(cfg, K1, V, q1, n - 1)
    np.testing.assert_array_equal(s4, np.full(n, (4 * L * d / 256) / (L * Hq)))
    # scaled mode is raw / sqrt(d)
    cfg2 = oracle.OrcCfg(L=L, Hq=Hq, Hkv=Hkv, d=d, window=1, tau=-1.0, score_scaled=1)
    _, _, s5, _ = one_step(cfg2, K, V, q, n - 1)
    np.testing.assert_allclose(s5, s0 / math.sqrt(d), rtol=1e-15)


def test_attention_special_cases():
    d = 8
    cfg = oracle.OrcCfg(L=1, Hq=1, Hkv=1, d=d, window=1, tau=-1.0)
    rng = np.random.default_rng(0)
    # singleton active set -> O = V exactly
    K = rng.standard_normal((1, 1, 1, d)).astype(np.float32)
    V = rng.standard_normal((1, 1, 1, d)).astype(np.float32)
    O, act, _, _ = one_step(cfg, K, V, rng.standard_normal((1, 1, d)), 0)
    np.testing.assert_array_equal(O[0, 0], V[0, 0, 0].astype(np.float64))
    # equal logits -> mean of V
    K = np.zeros((3, 1, 1, d), np.float32)
    V = rng.standard_normal((3, 1, 1, d)).astype(np.float32)
    O, _, _, _ = one_step(cfg, K, V, rng.standard_normal((1, 1, d)), 2)
    np.testing.assert_allclose(O[0, 0], V[:, 0, 0].astype(np.float64).mean(0), rtol=0, atol=1e-15)
    # two tokens: weights are the logistic of the logit gap / sqrt(d) (Eq. 1 scale)
    K = np.zeros((2, 1, 1, d), np.float32)
    K[0, 0, 0, 0] = 3.0
    V = np.zeros((2, 1, 1, d), np.float32)
    V[0, 0, 0, 0] = 1.0
    q = np.zeros((1, 1, d), np.float32)
    q[0, 0, 0] = 2.0
    O, _, _, _ = one_step(cfg, K, V, q, 1)
    gap = 6.0 / math.sqrt(d)
    assert abs(O[0, 0, 0] - 1 / (1 + math.exp(-gap))) < 1e-15


def masked_full_attention(q, K, V, active, d):
    """Independent formulation: attention over ALL positions with frozen logits = -inf."""
    L, Hq, _ = q.shape
    Hkv = K.shape[2]
    g = Hq // Hkv
    O = np.zeros((L, Hq, d))
    for l in range(L):
        for h in range(Hq):
            logits = K[:, l, h // g, :].astype(np.float64) @ q[l, h].astype(np.float64) / np.sqrt(d)
            logits = np.where(active, logits, -np.inf)
            w = np.exp(logits - logits.max())
            w /= w.sum()
            O[l, h] = w @ V[:, l, h // g, :].astype(np.float64)
    return O


def test_masked_equivalence_and_affine_v():
    # LAT all-cold tiny config: run steps with real decisions and compare every step's O with
    # the masked full attention over the oracle's own residency before the step.
    p = gen.GenParams(seed=11, L=2, Hq=4, Hkv=2, d=16)
    K_, P, steps = 4, 6, 40
    cap = P + steps
    cfg = oracle.OrcCfg(L=2, Hq=4, Hkv=2, d=16, window=K_)
    K, V = gen.kv(p, 0, 0, cap, "f32")
    s = oracle.OracleSeq(cfg, cap, P)
    frozen_seen = 0
    for i in range(steps):
        q = gen.q(p, 0, i, "f32")
        O, act, scores, out = s.step(q, K, V)
        active = np.zeros(cap, bool)
        active[act] = True
        np.testing.assert_allclose(O, masked_full_attention(q, K, V, active, 16), rtol=0, atol=1e-13)
        frozen_seen += out["frozen_post"]
    assert frozen_seen > 0
    # affine equivariance: O(a V + b) = a O(V) + b (softmax weights sum to 1)
    s1 = oracle.OracleSeq(cfg, cap, cap - 1)
    s2 = oracle.OracleSeq(cfg, cap, cap - 1)
    q = gen.q(p, 0, 0, "f32")
    O1, *_ = s1.step(q, K, V)
    O2, *_ = s2.step(q, K, (2.0 * V + 0.5).astype(np.float32))
    np.testing.assert_allclose(O2, 2.0 * O1 + 0.5, rtol=0, atol=1e-12)


def test_lat_scores_respect_guard_band():
    # LAT construction: cold tokens score <= 7/16, hot (a=4) tokens >= 1.3125 (DESIGN.md input recipe)
    p = gen.GenParams(seed=5, L=2, Hq=8, Hkv=2, d=32, hot_permille=300, a_hot=4)
    cap = 200
    K, V = gen.kv(p, 0, 0, cap)
    cfg = oracle.OrcCfg(L=2, Hq=8, Hkv=2, d=32, window=8, tau=0.5)
    s = oracle.OracleSeq(cfg, cap, 100)
    for i in range(20):
        O, act, scores, out = s.step(gen.q(p, 0, i), K, V)
        hot = np.array([gen.is_hot(p, 0, int(j)) for j in act])
        assert np.all(scores[~hot] <= 7 / 16) and np.all(scores[hot] >= 1.3125)
        assert np.all(np.abs(scores - 0.5) > 1e-3)
        # lattice exactness: every score is a multiple of 2^-8 / (L*Hq)
        units = scores * 256 * 16
        np.testing.assert_array_equal(units, np.round(units))


def test_tau_zero_is_full_attention():
    # tau = 0: no s_j < 0, so every token stays active and O is full attention
    p = gen.GenParams(seed=2, family=gen.GAUSS, L=1, Hq=4, Hkv=1, d=16)
    cap = 50
    K, V = gen.kv(p, 0, 0, cap, "f32")
    cfg = oracle.OrcCfg(L=1, Hq=4, Hkv=1, d=16, window=2, tau=0.0)
    s = oracle.OracleSeq(cfg, cap, 10)
    for i in range(30):
        q = gen.q(p, 0, i, "f32")
        O, act, _, out = s.step(q, K, V)
        assert out["attended"] == out["n"] and out["frozen_post"] == 0
        active = np.zeros(cap, bool)
        active[: out["n"]] = True
        np.testing.assert_allclose(O, masked_full_attention(q, K, V, active, 16), rtol=0, atol=1e-13)


def test_full_step_matches_policy_replay_on_lat():
    # with real attention + Eq. 2 scores on LAT inputs, the ledger follows exactly the all-cold
    # class labels (cold -> flagged), i.e. the closed form of test_oracle_policy
    p = gen.GenParams(seed=9, L=1, Hq=2, Hkv=2, d=16)
    cfg = oracle.OrcCfg(window=16)
    cap = 32 + 32
    K, V = gen.kv(p, 0, 0, cap)
    s_full = oracle.OracleSeq(cfg, cap, 32)
    s_pol = oracle.OracleSeq(cfg, cap, 32)
    below = np.ones(cap, np.uint8)
    for i in range(32):
        _, act1, _, o1 = s_full.step(gen.q(p, 0, i), K, V)
        act2, o2 = s_pol.step_policy(below)
        np.testing.assert_array_equal(act1, act2)
        assert o1 == o2
        for key in ("residency", "timer", "count", "freeze_step"):
            np.testing.assert_array_equal(s_full.ledger()[key], s_pol.ledger()[key])


# ---- the single-output functions (orc_attend_head, orc_score_token) used by the full-size sampled
#      parity test: pinned by the same special cases and closed values, then shown to agree with
#      orc_step's outputs on a random case

def test_attend_head_special_cases():
    rng = np.random.default_rng(5)
    d = 8
    q = f32(rng.normal(size=d))
    K1, V1 = f32(rng.normal(size=(1, d))), f32(rng.normal(size=(1, d)))
    assert np.array_equal(oracle.attend_head(q, K1, V1), V1[0].astype(np.float64))   # singleton softmax = 1
    K = f32(rng.normal(size=(5, d)))
    V = f32(rng.normal(size=(5, d)))
    np.testing.assert_allclose(oracle.attend_head(f32(np.zeros(d)), K, V), V.astype(np.float64).mean(0),
                               rtol=0, atol=1e-15)   # equal logits: the mean
    K2, V2 = K[:2], V[:2]
    gap = float(np.dot(q.astype(np.float64), K2[0].astype(np.float64) - K2[1].astype(np.float64))) / math.sqrt(d)
    w = 1.0 / (1.0 + math.exp(-gap))    # two tokens: the logistic of the scaled logit gap
    np.testing.assert_allclose(oracle.attend_head(q, K2, V2), w * V2[0].astype(np.float64) + (1 - w) * V2[1].astype(np.float64),
                               rtol=0, atol=1e-14)


def test_score_token_closed_values():
    # L=1, Hq=2, Hkv=1, d=2: |1*0.5 + 2*(-1)| + |-3*0.5 + 0.5*(-1)| = 1.5 + 2 = 3.5, over H = 2
    q = f32([[[1, 2], [-3, 0.5]]])
    k = f32([[[0.5, -1]]])
    assert oracle.score_token(q, k) == 1.75
    assert oracle.score_token(q, k, scaled=True) == 1.75 / math.sqrt(2)
    # GQA: heads 0, 1 read KV head 0 and heads 2, 3 KV head 1 (h // (Hq/Hkv)): (2+4+9+12)/4; the
    # interleaved map h % Hkv would give 26/4
    assert oracle.score_token(f32([[[1], [2], [3], [4]]]), f32([[[2], [3]]])) == 6.75


def test_single_outputs_agree_with_step():
    rng = np.random.default_rng(9)
    L, Hq, Hkv, d, P = 2, 4, 2, 16, 12
    cfg = oracle.OrcCfg(L=L, Hq=Hq, Hkv=Hkv, d=d, window=4, tau=0.3)
    K = f32(rng.normal(size=(P + 1, L, Hkv, d)))
    V = f32(rng.normal(size=(P + 1, L, Hkv, d)))
    q = f32(rng.normal(size=(L, Hq, d)))
    O, act, scores, _ = one_step(cfg, K, V, q, P)
    for l in range(L):
        for h in range(Hq):
            g = h // (Hq // Hkv)
            np.testing.assert_array_equal(oracle.attend_head(q[l, h], K[act, l, g], V[act, l, g]), O[l, h])
    for a, j in enumerate(act):
        assert oracle.score_token(q, K[j]) == scores[a]
