"""Pins for Eq. 3: d_j = floor(sqrt(c_j)/k) as computed by the oracle.

Pinned against: the paper's worked values, SPEC's examples, and the exact
integer square root from the standard library (math.isqrt), which is an independent
implementation of the closed form floor(sqrt(c)) — for integer k, floor(floor(sqrt(c))/k) =
floor(sqrt(c)/k).
"""
import json
import math
import os

import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_paper_anchor_values():
    g = _load("paper_tables.json")["eq3_anchors_k2"]
    for c, d in g["c_to_d"]:
        assert oracle.duration(c, 2.0) == d, (c, d)


def test_spec_examples():
    for c, k, d in _load("spec_examples.json")["duration"]["cases"]:
        assert oracle.duration(c, k) == d


@pytest.mark.parametrize("k", [1, 2, 3])
def test_exhaustive_against_isqrt(k):
    # exact for every c in [0, 1e6] at k in {1, 2, 3}; floor(sqrt(c)/k) = isqrt(c)//k.
    step = 1 if k != 1 else 1
    for c in range(0, 1_000_001, step):
        if oracle.duration(c, float(k)) != math.isqrt(c) // k:
            pytest.fail(f"c={c} k={k}: {oracle.duration(c, float(k))} != {math.isqrt(c) // k}")


def test_non_integer_softness():
    # floor(sqrt(c)/1.5) checked with exact rationals: m <= sqrt(c)/1.5  <=>  (3m)^2 <= 4c
    for c in range(0, 20000):
        m = 0
        while (3 * (m + 1)) ** 2 <= 4 * c:
            m += 1
        assert oracle.duration(c, 1.5) == m, c


def test_properties():
    # Sec 3.4: gentle early penalty (first detection -> 0), monotone in c,
    # non-increasing in k, sublinear: d(c) <= sqrt(c)/k.
    assert oracle.duration(1, 2.0) == 0
    prev = 0
    for c in range(0, 5000):
        d = oracle.duration(c, 2.0)
        assert d >= prev
        assert d <= math.sqrt(c) / 2.0 + 1e-12
        assert oracle.duration(c, 3.0) <= d
        prev = d
