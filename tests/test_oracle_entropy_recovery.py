"""Pins for the entropy stage and the recovery ladder (Sec 3.6).

Entropy is pinned against closed forms (one-hot -> 0, uniform -> ln n,
(1/2,1/2) -> ln 2; a two-level distribution's H in closed form; temperature as logit scaling;
0 <= H <= ln V).  The detector and ladder are constructions (DESIGN.md R-det, R-ladder) pinned
against SPEC's worked examples and the paper's level definitions and order
SR -> WR -> FR -> RR.
"""
import math

import numpy as np
import pytest

import gen
import oracle


def f32(a):
    return np.ascontiguousarray(np.asarray(a, np.float32))


def test_entropy_closed_forms():
    V = 128256
    # naive fp64 summation over V terms: error bound ~ V * eps * ln V ~ 2e-10
    assert oracle.entropy(f32(np.zeros(V))) == pytest.approx(math.log(V), abs=V * 2.3e-16 * math.log(V))
    assert abs(math.log(V) - 11.761784) < 1e-6
    x = np.full(V, -1e4, np.float32)
    x[17] = 0.0
    assert oracle.entropy(f32(x)) == 0.0
    assert oracle.entropy(f32([3.0, 3.0])) == pytest.approx(math.log(2), abs=1e-15)
    # two-level: m entries at a, V-m at 0: H = ln Z - m a e^a / Z, Z = m e^a + (V - m)
    for m, a in ((1, 5.0), (10, 2.5), (1000, -1.0)):
        x = np.zeros(V, np.float32)
        x[:m] = a
        Z = m * math.exp(a) + (V - m)
        want = math.log(Z) - m * a * math.exp(a) / Z
        assert oracle.entropy(f32(x)) == pytest.approx(want, rel=1e-10)
    # temperature: H(x, T) = H(x / T, 1)
    rng = np.random.default_rng(1)
    x = f32(rng.standard_normal(5000) * 4)
    assert oracle.entropy(x, 2.0) == pytest.approx(oracle.entropy(f32(x / 2.0)), rel=1e-12)
    # bounds
    for s in range(5):
        h = oracle.entropy(f32(rng.standard_normal(1000) * (s + 1)))
        assert 0.0 <= h <= math.log(1000)


def test_bf16_logits_widen_exactly():
    p = gen.GenParams(seed=4, vocab=4096)
    row = gen.logits(p, 0, 3)
    assert oracle.entropy(row) == pytest.approx(oracle.entropy(gen.bf16_to_f32(row)), abs=0)


def _policy_seq(K=4, P=8, cap=400, **kw):
    cfg = oracle.OrcCfg(window=K, **kw)
    return oracle.OracleSeq(cfg, cap, P)


def test_detector_spec_examples():
    none = np.zeros(400, np.uint8)
    # constant series never triggers (sigma floor), a 5.0 after 64 x 1.0 triggers
    s = _policy_seq()
    for _ in range(64):
        _, out = s.step_policy(none, 1.0)
        assert out["recovery_action"] == 0
    _, out = s.step_policy(none, 5.0)
    assert out["recovery_action"] == 1
    # fewer than 2 observations never triggers
    s = _policy_seq()
    _, o1 = s.step_policy(none, 1.0)
    _, o2 = s.step_policy(none, 100.0)
    assert o1["recovery_action"] == 0 and o2["recovery_action"] == 0
    _, o3 = s.step_policy(none, 1000.0)
    assert o3["recovery_action"] == 1
    # exactly at the threshold is not a spike (strict >): mean 1, sigma floor 0.05, z 3 -> 1.15
    s = _policy_seq()
    for _ in range(10):
        s.step_policy(none, 1.0)
    _, o = s.step_policy(none, 1.0 + 3 * 0.05)
    assert o["recovery_action"] == 0
    s = _policy_seq()
    for _ in range(10):
        s.step_policy(none, 1.0)
    _, o = s.step_policy(none, 1.0 + 3 * 0.05 + 1e-9)
    assert o["recovery_action"] == 1


def test_ladder_order_with_planted_spikes():
    # generator logits: 8 evenly cycling baseline levels + spikes every 16 steps (config 4 pattern)
    V = 128256
    q0 = 70
    p = gen.GenParams(seed=42, vocab=V, spike_first=q0, spike_period=16, spike_count=4)
    s = _policy_seq(K=16, P=32, cap=300)
    below = np.ones(300, np.uint8)
    actions = []
    for i in range(140):
        H = oracle.entropy(gen.logits(p, 0, i - 1)) if i > 0 else None
        _, out = s.step_policy(below, H)
        if out["recovery_action"]:
            actions.append((i, out["recovery_action"], out["rewalk_requested"]))
    # logits_{i-1} carries the spike planted at step i-1 -> action at step i
    assert actions == [(q0 + 1, 1, 0), (q0 + 17, 2, 0), (q0 + 33, 3, 0), (q0 + 49, 4, 1)]


def test_ladder_absorb_and_reset():
    none = np.zeros(400, np.uint8)
    s = _policy_seq(cap=400)
    seq = []
    spikes = {10: 50.0, 15: 60.0, 26: 70.0, 80: 80.0}  # dt 5 (absorbed), 16 (escalate), 54 (reset)
    for i in range(100):
        _, out = s.step_policy(none, spikes.get(i, 1.0))
        if out["recovery_action"]:
            seq.append((i, out["recovery_action"]))
    assert seq == [(10, 1), (26, 2), (80, 1)]


def _run_cold(s, steps, cap):
    below = np.ones(cap, np.uint8)
    for _ in range(steps):
        s.step_policy(below)


def test_sr_restores_timers_above_one():
    # SR unfreezes tokens with d > 1 and leaves d = 1
    cap = 400
    s = _policy_seq(K=4, P=4, cap=cap)
    _run_cold(s, 120, cap)
    before = s.ledger()
    fro = before["residency"] == 0
    assert {1, 2}.issubset(set(before["timer"][fro].tolist()))
    r = s.restore("SR")
    after = s.ledger()
    moved = fro & (after["residency"] == 1)
    assert r == int(moved.sum())
    np.testing.assert_array_equal(moved, fro & (before["timer"] > 1))
    assert np.all(after["timer"][after["residency"] == 0] == 1)
    # counts are kept (R-count), restored tokens have timer 0
    np.testing.assert_array_equal(after["count"], before["count"])
    assert np.all(after["timer"][moved] == 0)


def test_wr_and_fr():
    cap = 400
    s = _policy_seq(K=4, P=4, cap=cap, wr_window=3)
    _run_cold(s, 150, cap)
    before = s.ledger()
    i = 150  # next step index
    fro = before["residency"] == 0
    s.restore("WR")
    after = s.ledger()
    moved = fro & (after["residency"] == 1)
    np.testing.assert_array_equal(moved, fro & (before["freeze_step"] >= i - 3))
    s.restore("FR")
    led = s.ledger()
    assert np.all(led["residency"] == 1) and np.all(led["timer"] == 0)
    # restores are reported in the next step's restored_this_step
    _, out = s.step_policy(np.zeros(cap, np.uint8))
    assert out["restored_this_step"] == int(fro.sum())
