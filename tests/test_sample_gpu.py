"""NEXT-1 parity: asr_sample (the next-token draw) against oracle/sample.py.

Draws are compared exactly where the answer is unique: u is placed in the middle of the oracle's
interval of a kept token (u +- half the interval cannot reach a neighbour's), and top-p values sit
halfway between two consecutive cumulative masses of the sorted kept set (the GPU sums fp32
probabilities, the oracle fp64).  Random u are checked for validity: the drawn token is kept and its
oracle interval contains u up to 1e-6.
"""
import numpy as np
import pytest

import gen
import oracle
from oracle.sample import interval, kept_set, sample

pytestmark = pytest.mark.gpu


def _rows(kind, B, V, seed):
    rng = np.random.default_rng(seed)
    if kind == "gen":   # the generator's logits rows (bf16 lattice normal with one peak)
        p = gen.GenParams(seed=seed, L=1, Hq=2, Hkv=2, d=16, vocab=V)
        return np.stack([gen.logits(p, b, b) for b in range(B)])
    if kind == "ties":  # few distinct values: many ties at every boundary
        x = rng.integers(-3, 4, size=(B, V)).astype(np.float32) * 0.5
        return x
    return (rng.normal(scale=2.0, size=(B, V))).astype(np.float32)


def _p_between(x, T, k):
    # a top-p value halfway between two consecutive normalised cumulative masses of the top-k set
    keep, p = kept_set(x, T, k, 1.0)
    order = np.lexsort((np.arange(x.size), -(x.astype(np.float64) if x.dtype != np.uint16 else
                                             (x.astype(np.uint32) << 16).view(np.float32))))
    kk = order if not (0 < k < x.size) else order[:k]
    c = np.cumsum(p[kk]) / p[kk].sum()
    i = min(len(c) - 2, max(0, int(np.searchsorted(c, 0.7))))
    return float(0.5 * (c[i] + c[i + 1])) if len(c) > 1 else 1.0


@pytest.mark.parametrize("kind,V,dtype", [("gen", 128256, "bf16"), ("normal", 5000, "f32"), ("ties", 3000, "f32"),
                                          ("normal", 131, "bf16")])
def test_sample_matches_oracle(kind, V, dtype):
    import torch
    from paper_2512_11221_b200 import asr_sample
    B = 6
    X = _rows(kind, B, V, 11 + V)
    if dtype == "bf16" and X.dtype != np.uint16:
        X = (X.view(np.uint32) >> 16).astype(np.uint16)   # truncate to bf16 bits
    xt = torch.from_numpy(X.view(np.int16)).view(torch.bfloat16).cuda() if X.dtype == np.uint16 else \
        torch.from_numpy(X).cuda()
    rng = np.random.default_rng(V)
    settings = [(0.0, 0, 1.0), (1.0, 1, 1.0), (1.0, 0, 1.0), (0.7, 50, 1.0), (1.0, 0, None), (0.8, 100, None),
                (1.3, 7, None),
                # k = 256, the top-k fast path's limit (on the 3000-value tie rows every element passes
                # the thread-maxima bound: more candidates than rank 0 holds -> the general path)
                (0.9, 256, None),
                # large k: the kept candidates overflow a CTA's shared-memory list (kCand) on some or all
                # CTAs, which then keep reading their slice
                (0.9, 2000, 1.0), (1.0, 20000, None)]
    for T, k, P in settings:
        Ps = [(_p_between(X[b], T, k) if P is None else P) for b in range(B)]
        # exact draws: u in the middle of a kept token's interval
        us, want = [], []
        for b in range(B):
            # a token drawn by the oracle (so it carries real mass) whose interval is wide enough for
            # fp32 u and fp32 probabilities (>= 1e-4 of the kept mass)
            for _ in range(50):
                tok = sample(X[b], T, k, Ps[b], float(rng.random()))
                lo, hi = interval(X[b], T, k, Ps[b], tok)
                if hi - lo >= 1e-4:
                    break
            us.append(0.5 * (lo + hi))
            want.append(tok)
        for b in range(B):   # one row per call when top-p differs per row
            if not interval(X[b], T, k, Ps[b], want[b])[1] - interval(X[b], T, k, Ps[b], want[b])[0] >= 1e-4:
                continue
            u = torch.tensor([us[b]], dtype=torch.float32, device="cuda")
            out = torch.empty(1, dtype=torch.int32, device="cuda")
            asr_sample(xt[b:b + 1], u, out, temperature=T, top_k=k, top_p=Ps[b])
            got = int(out.item())
            assert got == want[b], (kind, T, k, Ps[b], b, got, want[b], sample(X[b], T, k, Ps[b], us[b]))
        # random u, whole batch in one call (same top-p for all rows): validity
        if P is not None:
            u = rng.random(B).astype(np.float32)
            ut = torch.from_numpy(u).cuda()
            out = torch.empty(B, dtype=torch.int32, device="cuda")
            asr_sample(xt, ut, out, temperature=T, top_k=k, top_p=P)
            got = out.cpu().numpy()
            for b in range(B):
                lo, hi = interval(X[b], T, k, P, int(got[b]))
                assert lo == lo, (kind, T, k, b, int(got[b]), "not in the kept set")
                assert lo - 2e-6 <= float(u[b]) <= hi + 2e-6, (kind, T, k, b, lo, float(u[b]), hi)


def test_sample_deterministic():
    import torch
    from paper_2512_11221_b200 import asr_sample
    X = _rows("normal", 32, 20000, 3)
    xt = torch.from_numpy(X).cuda()
    u = torch.rand(32, device="cuda")
    a = torch.empty(32, dtype=torch.int32, device="cuda")
    b = torch.empty_like(a)
    asr_sample(xt, u, a, temperature=0.9, top_k=200, top_p=0.9)
    asr_sample(xt, u, b, temperature=0.9, top_k=200, top_p=0.9)
    assert torch.equal(a, b)


@pytest.mark.parametrize("B", [3, 16])
def test_sample_batched_rows(B):
    """Several rows per call: 16-CTA clusters (batch <= 4) and 4-CTA clusters (bf16, batch >= 8), one
    grid row per logits row; each row's u sits mid-interval of an oracle-drawn token."""
    import torch
    from paper_2512_11221_b200 import asr_sample
    V = 128256
    X = _rows("gen", B, V, 500 + B)
    xt = torch.from_numpy(X.view(np.int16)).view(torch.bfloat16).cuda()
    rng = np.random.default_rng(B)
    for T, k, P in [(0.8, 50, 0.9), (1.0, 0, 0.95), (0.7, 20000, 1.0)]:
        us, want = [], []
        for b in range(B):
            for _ in range(50):
                tok = sample(X[b], T, k, P, float(rng.random()))
                lo, hi = interval(X[b], T, k, P, tok)
                if hi - lo >= 1e-4:
                    break
            us.append(0.5 * (lo + hi) if hi - lo >= 1e-4 else float(rng.random()))
            want.append(tok if hi - lo >= 1e-4 else -1)
        out = torch.empty(B, dtype=torch.int32, device="cuda")
        asr_sample(xt, torch.tensor(us, dtype=torch.float32, device="cuda"), out, temperature=T, top_k=k, top_p=P)
        got = out.cpu().numpy()
        for b in range(B):
            if want[b] >= 0:
                assert int(got[b]) == want[b], (B, T, k, P, b, int(got[b]), want[b])
            else:
                lo, hi = interval(X[b], T, k, P, int(got[b]))
                assert lo - 2e-6 <= us[b] <= hi + 2e-6, (B, T, k, P, b, lo, us[b], hi)


def test_sample_uncached_slice():
    """A vocabulary whose per-CTA slice exceeds the shared-memory cache (fp32, V = 400000, one row:
    16 CTAs of 100 KB): every pass reads global memory; exact draws as above."""
    import torch
    from paper_2512_11221_b200 import asr_sample
    V = 400000
    x = _rows("normal", 1, V, 77)[0]
    xt = torch.from_numpy(x[None]).cuda()
    rng = np.random.default_rng(3)
    for T, k, P in [(0.8, 50, 0.9), (1.0, 0, 0.95), (0.7, 3000, 1.0)]:
        for _ in range(50):
            tok = sample(x, T, k, P, float(rng.random()))
            lo, hi = interval(x, T, k, P, tok)
            if hi - lo >= 1e-4:
                break
        if hi - lo < 1e-4:
            continue
        out = torch.empty(1, dtype=torch.int32, device="cuda")
        asr_sample(xt, torch.tensor([0.5 * (lo + hi)], dtype=torch.float32, device="cuda"), out,
                   temperature=T, top_k=k, top_p=P)
        assert int(out.item()) == tok, (T, k, P, int(out.item()), tok)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("B", [1, 5, 9])
def test_sample_entropy_one_pass(dtype, B):
    # asr_sample_entropy: the same token as asr_sample, and H of softmax(x / T_ent) within 1e-4 nats of the
    # oracle (fp32 accumulation over 128256 terms), for greedy and filtered draws, T_ent 1 and 0.7
    import torch
    from paper_2512_11221_b200 import asr_sample, asr_sample_entropy
    V = 128256
    g = gen.GenParams(seed=31, vocab=V, spike_first=2, spike_period=3, spike_count=9)
    rows = np.stack([gen.logits(g, b, b % 4, "bf16" if dtype == "bf16" else "f32") for b in range(B)])
    xt = torch.from_numpy(rows.view(np.int16) if dtype == "bf16" else rows).cuda()
    xt = xt.view(torch.bfloat16) if dtype == "bf16" else xt
    u = torch.rand(B, device="cuda")
    for (T, k, P) in ((0.0, 0, 1.0), (0.8, 50, 0.9), (1.0, 0, 0.95)):
        for te in (1.0, 0.7):
            t1 = torch.empty(B, dtype=torch.int32, device="cuda")
            t2 = torch.empty(B, dtype=torch.int32, device="cuda")
            h = torch.empty(B, dtype=torch.float32, device="cuda")
            asr_sample(xt, u, t1, temperature=T, top_k=k, top_p=P)
            asr_sample_entropy(xt, u, t2, h, temperature=T, top_k=k, top_p=P, entropy_temperature=te)
            assert torch.equal(t1, t2)
            for b in range(B):
                want = oracle.entropy(rows[b], te)
                assert abs(float(h[b]) - want) <= 1e-4, (T, k, P, te, b, float(h[b]), want)


@pytest.mark.parametrize("B", [1, 3, 16])
def test_sample_fast_paths_tied_peaks(B):
    """The top-k / pure top-p fast paths (candidates above the thread-maxima bound, finished by one
    CTA) where the decisions hinge on ties: a low bulk (N(0,1) - 6) under two tied peak groups (7
    tokens at 6.0, 9 at 5.5, bf16-exact), top-p between two consecutive cumulative masses inside a
    tie group (the boundary takes the lowest indices first), top-k cutting a tie group; u mid-interval
    of an oracle-drawn token (exact), then random u (validity).  Clusters of 16 / 8 / 4 CTAs."""
    import torch
    from paper_2512_11221_b200 import asr_sample
    V = 128256
    rng = np.random.default_rng(900 + B)
    X = np.empty((B, V), np.uint16)
    for b in range(B):
        x = (rng.normal(size=V) - 6.0).astype(np.float32)
        idx = rng.choice(V, 16, replace=False)
        x[idx[:7]] = 6.0
        x[idx[7:]] = 5.5
        X[b] = (x.view(np.uint32) >> 16).astype(np.uint16)   # bf16 bits (6.0 and 5.5 are exact)
    xt = torch.from_numpy(X.view(np.int16)).view(torch.bfloat16).cuda()
    for T, k in [(1.0, 0), (1.0, 10), (0.9, 12), (1.0, 200)]:
        for b in range(B):
            P = _p_between(X[b], T, k)
            tok = lo = hi = None
            for _ in range(50):
                tok = sample(X[b], T, k, P, float(rng.random()))
                lo, hi = interval(X[b], T, k, P, tok)
                if hi - lo >= 1e-4:
                    break
            if hi - lo < 1e-4:
                continue
            u = torch.tensor([0.5 * (lo + hi)], dtype=torch.float32, device="cuda")
            out = torch.empty(1, dtype=torch.int32, device="cuda")
            asr_sample(xt[b:b + 1], u, out, temperature=T, top_k=k, top_p=P)
            assert int(out.item()) == tok, (B, T, k, P, b, int(out.item()), tok)
        # the whole batch in one call, random u: the drawn token is kept and its interval holds u
        P = 0.6
        u = rng.random(B).astype(np.float32)
        out = torch.empty(B, dtype=torch.int32, device="cuda")
        asr_sample(xt, torch.from_numpy(u).cuda(), out, temperature=T, top_k=k, top_p=P)
        got = out.cpu().numpy()
        for b in range(B):
            lo, hi = interval(X[b], T, k, P, int(got[b]))
            assert lo == lo, (B, T, k, b, int(got[b]), "not in the kept set")
            assert lo - 2e-6 <= float(u[b]) <= hi + 2e-6, (B, T, k, b, lo, float(u[b]), hi)
