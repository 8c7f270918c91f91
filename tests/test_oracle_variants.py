"""Pins for the oracle's option branches (NEXT-3 variants), each against a hand-derived trace or a
closed form, never against the oracle's own rule restated:

- `fr_clear_counts` ("FR ... clears all detection logs"): after FR with clearing, an
  always-flagged token needs c = 4 detections again before Eq. 3 gives d = floor(sqrt(c)/k) >= 1
  at k = 2 (worked values c=1 -> 0, c=4 -> 1); without clearing its count runs on
  from 17 and every detection freezes it (d = floor(sqrt(17)/2) = 2).
- `pinned_prefix`: positions < p are never eligible, so the all-cold
  closed form K + P(n - K) (tests/test_oracle_policy.py) becomes K + p + P(n - K - p).
- WR ("Unfreeze all tokens in the last N steps"): a hand-built scenario in which three
  single tokens freeze at known steps 10, 12 and 14 with timers long enough to still be frozen at
  step 15; WR with N = 3 before step 15 restores exactly the two frozen at steps >= 12.
"""
import numpy as np

import oracle
from test_oracle_policy import complete_periods


def _seq(K, P, cap, **kw):
    return oracle.OracleSeq(oracle.OrcCfg(window=K, **kw), cap, P)


def _fr_trace(clear: int):
    """One eligible token (position 0, always flagged); every other position is hot.  16 steps
    give c = 16 -> d = 2 (frozen at step 15 with timer 1); FR at the boundary before step 16
    restores it; then 7 more steps.  Returns per-step (frozen_this_step, count of position 0)."""
    K, P = 4, 5
    cap = P + 40
    s = _seq(K, P, cap, softness=2.0, fr_clear_counts=clear)
    below = np.zeros(cap, np.uint8)
    below[0] = 1
    out = []
    for i in range(23):
        if i == 16:
            assert s.restore("FR") == 1
        _, o = s.step_policy(below)
        out.append((o["frozen_this_step"], int(s.ledger()["count"][0]), int(s.ledger()["residency"][0])))
    return out


def test_fr_clear_counts_hand_trace():
    # steps 0..15: c = 1..16; d = 0 for c < 4, 1 for 4 <= c < 16 (R0: frozen and restored by the
    # same tick, counted in frozen_this_step), 2 at c = 16 (timer 1: frozen after step 15)
    base = [(0, c, 1) for c in (1, 2, 3)] + [(1, c, 1) for c in range(4, 16)] + [(1, 16, 0)]
    with_clear = _fr_trace(1)
    without = _fr_trace(0)
    assert with_clear[:16] == base and without[:16] == base
    # after FR with clearing: c restarts at 1; d >= 1 first at c = 4 (three quiet steps)
    assert with_clear[16:] == [(0, 1, 1), (0, 2, 1), (0, 3, 1), (1, 4, 1), (1, 5, 1), (1, 6, 1), (1, 7, 1)]
    # without clearing: c = 17 -> d = 2 (frozen, absent at the next step, whose tick restores it),
    # then c = 18, 19, 20 -> d = 2 on every other step
    assert without[16:] == [(1, 17, 0), (0, 17, 1), (1, 18, 0), (0, 18, 1), (1, 19, 0), (0, 19, 1), (1, 20, 0)]


def test_pinned_prefix_closed_form():
    K, P, steps = 8, 8, 400
    for p in (0, 1, 5, 13):
        cap = P + steps + 1
        s = _seq(K, P, cap, softness=2.0, pinned_prefix=p)
        below = np.ones(cap, np.uint8)
        for _ in range(steps):
            _, o = s.step_policy(below)
            n = o["n"]
            E = n - K - p
            want = K + p + complete_periods(E) if E >= 0 else n
            assert o["active_post"] == want, (p, n, o["active_post"], want)
            led = s.ledger()
            assert np.all(led["residency"][:min(p, n)] == 1) and np.all(led["count"][:min(p, n)] == 0)


def test_wr_hand_built_scenario():
    K, P = 2, 8
    cap = P + 40

    def build(N):
        # k = 0.1: the first detection gives d = floor(sqrt(1) / 0.1) = 10 -> frozen with timer 9 (R0)
        s = _seq(K, P, cap, softness=0.1, wr_window=N)
        for i in range(15):
            below = np.zeros(cap, np.uint8)
            if i in (10, 12, 14):
                below[{10: 1, 12: 2, 14: 3}[i]] = 1
            s.step_policy(below)
        return s

    s = build(3)
    led = s.ledger()
    assert [j for j in range(led["residency"].size) if led["residency"][j] == 0] == [1, 2, 3]
    assert list(led["timer"][1:4]) == [5, 7, 9]       # 9 - (14 - 10), 9 - (14 - 12), 9
    assert s.restore("WR") == 2                       # frozen at steps >= 15 - 3 = 12: positions 2 and 3
    led = s.ledger()
    assert [j for j in range(led["residency"].size) if led["residency"][j] == 0] == [1]
    act, o = s.step_policy(np.zeros(cap, np.uint8))
    assert o["restored_this_step"] == 2 and 1 not in act and 2 in act and 3 in act
    s = build(5)                                      # steps >= 10: all three
    assert s.restore("WR") == 3
    s = build(1)                                      # steps >= 14: only position 3
    assert s.restore("WR") == 1 and s.ledger()["residency"][3] == 1
