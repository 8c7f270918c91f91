"""Generator (gen/) properties on the host build: the LAT family's construction guarantees that
the guard band |s_j - tau| > 1e-3 of BASELINE.json's parity bar holds by proof, not by luck."""
import numpy as np

import gen


def test_determinism_and_seed_sensitivity():
    p = gen.GenParams(seed=3, L=2, Hq=4, Hkv=2, d=32)
    k1, v1 = gen.kv(p, 1, 5, 7)
    k2, v2 = gen.kv(p, 1, 5, 7)
    np.testing.assert_array_equal(k1, k2)
    np.testing.assert_array_equal(v1, v2)
    p2 = gen.GenParams(seed=4, L=2, Hq=4, Hkv=2, d=32)
    assert not np.array_equal(gen.kv(p2, 1, 5, 7)[1], v1)
    # slicing positions is consistent
    ka, _ = gen.kv(p, 1, 0, 12)
    np.testing.assert_array_equal(ka[5:12], k1)


def test_bf16_and_f32_agree_exactly():
    p = gen.GenParams(seed=8, L=2, Hq=4, Hkv=2, d=64, hot_permille=300, vocab=1000)
    kb, vb = gen.kv(p, 0, 0, 20, "bf16")
    kf, vf = gen.kv(p, 0, 0, 20, "f32")
    np.testing.assert_array_equal(gen.bf16_to_f32(kb), kf)
    np.testing.assert_array_equal(gen.bf16_to_f32(vb), vf)
    np.testing.assert_array_equal(gen.bf16_to_f32(gen.q(p, 0, 3)), gen.q(p, 0, 3, "f32"))
    np.testing.assert_array_equal(gen.bf16_to_f32(gen.logits(p, 0, 3)), gen.logits(p, 0, 3, "f32"))


def test_lat_construction_bounds():
    for d in (16, 128):
        p = gen.GenParams(seed=21, L=3, Hq=8, Hkv=2, d=d, hot_permille=300, a_hot=4)
        k, _ = gen.kv(p, 0, 0, 300, "f32")
        m = min(16, d - 2)
        hot = np.array([gen.is_hot(p, 0, j) for j in range(300)])
        assert 0.2 < hot.mean() < 0.4
        nz = (k[..., 2:] != 0).sum(-1)
        assert np.all(nz == m)
        assert np.all(np.abs(k[..., 2:]).sum(-1) <= 1.0)
        np.testing.assert_array_equal(k[..., 0][hot], 4.0)
        np.testing.assert_array_equal(k[..., 0][~hot], 0.0)
        q = gen.q(p, 0, 0, "f32")
        assert np.all(q[..., 0] == 7 / 16) and np.all(q[..., 1] == 0)
        assert np.abs(q).max() <= 7 / 16
        # per-(l, head) cold dot product bound |q.k| <= 7/16
        dots = np.einsum("lhd,tlgd->tlhg", q, k[:, :, :, :])
        assert np.abs(dots[~hot]).max() <= 7 / 16


def test_gauss_family_stats():
    p = gen.GenParams(seed=1, family=gen.GAUSS, L=1, Hq=1, Hkv=1, d=128)
    _, v = gen.kv(p, 0, 0, 400, "f32")
    assert abs(v.mean()) < 0.05 and 1.05 < v.std() < 1.25
    k, _ = gen.kv(p, 0, 0, 400, "f32")
    assert 1.05 < k.std() < 1.25


def test_needle_and_query_steps():
    p = gen.GenParams(seed=2, L=1, Hq=2, Hkv=1, d=16, needle_pos=5, query_first=10, query_count=3)
    k, _ = gen.kv(p, 0, 0, 8, "f32")
    assert np.all(k[5, ..., 1] == 128) and np.all(k[np.arange(8) != 5, ..., 1] == 0)
    assert gen.q(p, 0, 10, "f32")[0, 0, 1] == 7 / 16 and gen.q(p, 0, 13, "f32")[0, 0, 1] == 0
