"""Pins for the oracle's decision loop (Alg. 1 lines 3-15; Eq. 3; Sec 3.5).

Pinned against:
- the paper's printed active counts: Table 1 170 of 514, Table 3 119 of 269,
  reproduced by the all-cold trace at the paper's K=32, k=2 under the readings in
  DESIGN.md (R-tick R0, R-W infinite, R-win);
- a closed form for the all-cold trajectory, derived by hand from the single-token life cycle
  (not from the oracle): active_post(n) = K + P(n-K), P(E) = number of complete detection
  periods max(floor(sqrt(c)/k), 1) that fit in E eligible steps;
- the W1 (hot-set) closed form active_post(n) = K + sum_{j<n-K} [hot(j) ? 1 : r(n-K-1-j)];
- invariants: conservation, timer/residency consistency, tau <= 0 and K >= n baselines.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def complete_periods(E: int, k: int = 2) -> int:
    """Number of complete detection periods of one always-flagged token in E eligible steps."""
    cnt = e = c = 0
    while e < E:
        c += 1
        L = max(math.isqrt(c) // k, 1)
        if e + L <= E:
            cnt += 1
        e += L
    return cnt


def single_token_residency(E: int, k: int = 2) -> list[int]:
    """Post-step residency (1 = active) of one always-flagged token over its first E eligible steps:
    a period of length L ends with the token active (the detection step for L = 1, the restore step
    after L-1 absent steps otherwise)."""
    out = []
    c = 0
    while len(out) < E:
        c += 1
        L = max(math.isqrt(c) // k, 1)
        out.extend([0] * (L - 1) + [1])
    return out[:E]


def run_all_cold(K, P, steps, k=2.0, tick_skip_new=0, W=0, hot=None):
    cfg = oracle.OrcCfg(window=K, softness=k, tick_skip_new=tick_skip_new, history_window=W)
    cap = P + steps + 1
    s = oracle.OracleSeq(cfg, cap, P)
    below = np.ones(cap, np.uint8)
    if hot is not None:
        below[hot] = 0
    trace = []
    for _ in range(steps):
        act, out = s.step_policy(below)
        trace.append(out)
        led = s.ledger()
        # conservation and ledger consistency after every step
        res = led["residency"]
        assert out["active_post"] + out["frozen_post"] == out["n"]
        assert int(res.sum()) == out["active_post"]
        assert np.all(led["timer"][res == 0] >= 1)
        assert np.all(led["timer"][res == 1] == 0)
        # the K most recent positions are always attended and active
        assert np.all(res[out["n"] - min(K, out["n"]):] == 1)
        assert np.all(np.diff(act) > 0)
    return s, trace


def test_table1_and_table3_reproduced():
    g = _load("paper_tables.json")
    hp = g["hyperparameters"]
    t1, t3 = g["table1"], g["table3"]
    K, k = hp["K"], hp["k"]
    P = t1["total"] - t1["generated"]  # 14-token prompt, 500 generated tokens
    _, tr = run_all_cold(K, P, t1["generated"], k)
    by_n = {o["n"]: o["active_post"] for o in tr}
    assert by_n[t1["total"]] == t1["active"]
    assert by_n[t3["total"]] == t3["active"]
    assert round(100 * (1 - t1["active"] / t1["total"]), 2) == t1["compression_pct"]
    assert round(100 * (1 - t3["active"] / t3["total"]), 2) == t3["compression_pct"]


@pytest.mark.parametrize("P", [1, 5, 20, 33])
def test_tables_hold_for_any_short_prompt(P):
    # the all-cold dynamics depend only on age for P <= K+1 (no lockstep prompt cohort)
    _, tr = run_all_cold(32, P, 514 - P, 2.0)
    by_n = {o["n"]: o["active_post"] for o in tr}
    assert by_n[514] == 170 and by_n[269] == 119


def test_neighbouring_readings_miss_the_tables():
    # R1 (newly frozen tokens not ticked) and finite W give other counts
    d = _load("survey_derived.json")["readings_n514_n269"]
    for kw, want in (({"tick_skip_new": 1}, d["R1_skip_new"]), ({"W": 128}, d["W128"]),
                     ({"W": 256}, d["W256"])):
        _, tr = run_all_cold(32, 14, 500, 2.0, **kw)
        by_n = {o["n"]: o["active_post"] for o in tr}
        assert [by_n[514], by_n[269]] == want, kw


@pytest.mark.parametrize("K,n", [(32, 2000), (512, 3000), (16, 1500)])
def test_closed_form_all_cold(K, n):
    _, tr = run_all_cold(K, K, n - K, 2.0)
    for o in tr:
        assert o["active_post"] == K + complete_periods(o["n"] - K), o


@pytest.mark.slow
def test_closed_form_8k_k512():
    _, tr = run_all_cold(512, 512, 8192 - 512, 2.0)
    assert tr[-1]["n"] == 8192
    assert tr[-1]["active_post"] == 512 + complete_periods(8192 - 512) == 1349


def test_single_token_residency_bits():
    bits = _load("survey_derived.json")["single_token_residency_first80"]["bits"]
    assert "".join(map(str, single_token_residency(80))) == bits
    # and the oracle agrees: residency of position 0 with K=1, P=1
    s, tr = run_all_cold(1, 1, 81, 2.0)
    # position 0 becomes eligible at n=2 (0 < n-K); record its post-step residency per step
    s2 = oracle.OracleSeq(oracle.OrcCfg(window=1), 100, 1)
    below = np.ones(100, np.uint8)
    seq = []
    for _ in range(80):
        s2.step_policy(below)
        seq.append(int(s2.ledger()["residency"][0]))
    assert "".join(map(str, seq)) == bits


def test_tiny_lockstep_sequence():
    g = _load("survey_derived.json")["tiny_all_cold"]
    _, tr = run_all_cold(g["K"], g["P"], g["steps"], 2.0)
    assert [o["active_post"] for o in tr] == g["active_post"]


def test_fig1_staircase():
    g = _load("survey_derived.json")["fig1_every25"]["values"]
    _, tr = run_all_cold(32, 14, 475, 2.0)
    for kk, want in enumerate(g[1:], start=1):
        assert tr[25 * kk - 1]["active_post"] == want


def test_w1_hot_set_closed_form():
    rng = np.random.default_rng(7)
    K, P, steps = 16, 16, 700
    cap = P + steps + 1
    hot = np.flatnonzero(rng.random(cap) < 0.3)
    _, tr = run_all_cold(K, P, steps, 2.0, hot=hot)
    hotset = set(hot.tolist())
    r = single_token_residency(cap)
    for o in tr:
        n = o["n"]
        want = K + sum(1 if j in hotset else r[n - K - 1 - j] for j in range(n - K))
        assert o["active_post"] == want


def test_no_flags_baselines():
    # tau <= 0: s_j >= 0 never below tau -> nothing ever frozen
    s = oracle.OracleSeq(oracle.OrcCfg(window=4), 64, 8)
    none = np.zeros(64, np.uint8)
    for _ in range(40):
        act, out = s.step_policy(none)
        assert out["attended"] == out["n"] == out["active_post"] and out["frozen_this_step"] == 0
    # K >= n: every position protected even when flagged
    s = oracle.OracleSeq(oracle.OrcCfg(window=64), 64, 8)
    allb = np.ones(64, np.uint8)
    for _ in range(40):
        act, out = s.step_policy(allb)
        assert out["active_post"] == out["n"]


def test_counts_and_freeze_steps():
    # c_j counts only flagged (active, eligible) steps and persists across restores (R-count)
    s, tr = run_all_cold(4, 4, 60, 2.0)
    led = s.ledger()
    n = s.n
    # position 0 is eligible from the step where n = K+1 = 5; it is flagged on every step it is
    # active, so its count equals the number of complete periods + 1 for a partial one if active
    cnt0 = int(led["count"][0])
    E = n - 4
    assert cnt0 == sum(single_token_residency(E)[: E - 1]) + 1
