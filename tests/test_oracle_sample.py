"""Pins of the NEXT-1 sampling oracle (oracle/sample.py) against definitions and worked examples."""
import numpy as np

from oracle.sample import interval, kept_set, sample


def _logits_of(p):
    return np.log(np.asarray(p, np.float64)).astype(np.float32)


def test_greedy_and_top1_pick_the_first_maximum():
    x = np.array([1.0, 3.0, -2.0, 3.0, 0.5], np.float32)
    assert sample(x, 0.0, 0, 1.0, 0.99) == 1
    assert sample(x, 0.7, 1, 1.0, 0.99) == 1


def test_top_k_ties_go_to_lower_indices():
    x = np.array([1.0, 3.0, 3.0, 2.0, 3.0], np.float32)
    keep, _ = kept_set(x, 1.0, 2, 1.0)
    assert keep.tolist() == [1, 2]
    keep, _ = kept_set(x, 1.0, 4, 1.0)
    assert keep.tolist() == [1, 2, 3, 4]


def test_top_p_worked_example():
    # p = (0.5, 0.3, 0.2): cumulative 0.5, 0.8, 1.0 -> the shortest prefix reaching P
    x = _logits_of([0.5, 0.3, 0.2])
    assert kept_set(x, 1.0, 0, 0.45)[0].tolist() == [0]
    assert kept_set(x, 1.0, 0, 0.55)[0].tolist() == [0, 1]
    assert kept_set(x, 1.0, 0, 0.85)[0].tolist() == [0, 1, 2]


def test_top_k_before_top_p():
    # p = (0.4, 0.3, 0.2, 0.1); top-k 2 leaves mass 0.7, of which P = 0.5 needs only the first token
    # (top-p first would keep two)
    x = _logits_of([0.4, 0.3, 0.2, 0.1])
    assert kept_set(x, 1.0, 2, 0.5)[0].tolist() == [0]
    assert kept_set(x, 1.0, 0, 0.5)[0].tolist() == [0, 1]


def test_temperature_is_a_logit_scale():
    rng = np.random.default_rng(3)
    x = rng.normal(size=64).astype(np.float32)
    _, p_half = kept_set(x, 0.5, 0, 1.0)
    _, p_twice = kept_set((2 * x).astype(np.float32), 1.0, 0, 1.0)
    np.testing.assert_allclose(p_half, p_twice, rtol=1e-12)


def test_stratified_draws_reproduce_the_distribution():
    # inverse-CDF draws at u = (i + 1/2) / N hit each kept token in proportion to its renormalised
    # probability, to within one draw
    rng = np.random.default_rng(5)
    x = rng.normal(scale=2.0, size=40).astype(np.float32)
    for T, k, P in [(1.0, 0, 1.0), (0.7, 10, 1.0), (1.3, 0, 0.8), (1.0, 12, 0.6)]:
        keep, p = kept_set(x, T, k, P)
        q = p[keep] / p[keep].sum()
        N = 20000
        counts = np.zeros(x.size)
        for i in range(N):
            counts[sample(x, T, k, P, (i + 0.5) / N)] += 1
        assert set(np.flatnonzero(counts)) <= set(keep.tolist())
        np.testing.assert_allclose(counts[keep] / N, q, atol=1.5 / N)


def test_interval_round_trip():
    rng = np.random.default_rng(7)
    x = rng.normal(size=300).astype(np.float32)
    for T, k, P in [(1.0, 0, 1.0), (0.8, 50, 0.9)]:
        keep, _ = kept_set(x, T, k, P)
        for tok in keep[::7]:
            lo, hi = interval(x, T, k, P, int(tok))
            assert lo < hi
            assert sample(x, T, k, P, 0.5 * (lo + hi)) == tok


def test_bf16_bits_input():
    x = np.array([0.5, 2.0, -1.0], np.float32)
    bits = (x.view(np.uint32) >> 16).astype(np.uint16)
    assert sample(bits, 1.0, 0, 1.0, 0.3) == sample(x, 1.0, 0, 1.0, 0.3)
