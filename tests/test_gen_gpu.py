"""The device build of the generator (bench inputs in HBM) is bit-identical to the host build
(oracle inputs): same header, integer-only arithmetic."""
import numpy as np
import pytest

import gen

pytestmark = pytest.mark.gpu


def test_device_generator_matches_host():
    import torch
    p = gen.GenParams(seed=123, L=3, Hq=8, Hkv=2, d=128, hot_permille=300, a_hot=64, vocab=50000, needle_pos=7,
                      query_first=2, query_count=1, spike_first=4, spike_period=3, spike_count=2)
    B, P = 2, 20
    k = torch.empty((B, P, 3, 2, 128), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    gen.dev_kv(p, B, 5, P, k, v)
    q = torch.empty((B, 3, 8, 128), dtype=torch.bfloat16, device="cuda")
    lg = torch.empty((B, 50000), dtype=torch.bfloat16, device="cuda")
    for step in (0, 2, 4, 7):
        gen.dev_q(p, B, step, q)
        gen.dev_logits(p, B, step, lg)
        qh = q.cpu().view(torch.int16).numpy().view(np.uint16)
        lh = lg.cpu().view(torch.int16).numpy().view(np.uint16)
        for b in range(B):
            np.testing.assert_array_equal(qh[b], gen.q(p, b, step))
            np.testing.assert_array_equal(lh[b], gen.logits(p, b, step))
    kh = k.cpu().view(torch.int16).numpy().view(np.uint16)
    vh = v.cpu().view(torch.int16).numpy().view(np.uint16)
    for b in range(B):
        kk, vv = gen.kv(p, b, 5, P)
        np.testing.assert_array_equal(kh[b], kk)
        np.testing.assert_array_equal(vh[b], vv)
