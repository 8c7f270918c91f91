"""Pins of oracle/quant.py (NEXT-4, R-quant in DESIGN.md §2; PAPER.md P:207 names the quantised frozen
tier as future work).  Each test checks the oracle against something other than its own formula:
exact lattices, the rounding bound, brute-force nearest codes, special cases and torch's bf16 rounding."""
import numpy as np
import pytest
import torch

from oracle import quant


def _bits(x_f32: np.ndarray) -> np.ndarray:
    """fp32 values that are exact in bf16 -> bf16 bit patterns (truncation is exact for them)."""
    return (np.ascontiguousarray(x_f32, np.float32).view(np.uint32) >> 16).astype(np.uint16)


@pytest.mark.parametrize("bits", [8, 4])
def test_lattice_rows_are_exact(bits):
    """x = m * 2^-e with integer m, max |m| = qmax: scale = 2^-e, codes = m, dequantised x == x."""
    rng = np.random.default_rng(11)
    qm = quant.qmax_of(bits)
    rows, n = 64, 128
    m = rng.integers(-qm, qm + 1, size=(rows, n))
    m[np.arange(rows), rng.integers(0, n, rows)] = qm * rng.choice([-1, 1], rows)
    e = rng.integers(-12, 4, size=rows)
    x = (m * np.ldexp(1.0, e)[:, None]).astype(np.float32)
    codes, scales = quant.quantize(_bits(x), bits)
    assert np.array_equal(scales, np.ldexp(1.0, e).astype(np.float32))
    assert np.array_equal(codes.astype(np.int64), m)
    assert np.array_equal(quant.dequantize(codes, scales), _bits(x))


@pytest.mark.parametrize("bits", [8, 4])
def test_rounding_bound_and_brute_force(bits):
    """|code * scale - x| <= scale / 2 (round to nearest), and each code is the integer in
    [-qmax, qmax] nearest to x / scale found by exhaustive search in fp64 (except near-ties)."""
    rng = np.random.default_rng(12)
    qm = quant.qmax_of(bits)
    x = (rng.standard_normal((40, 64)) * rng.uniform(0.01, 8.0, (40, 1))).astype(np.float32)
    xb = (x.view(np.uint32) >> 16).astype(np.uint16)   # truncated to bf16
    xe = quant.bf16_bits_to_f32(xb).astype(np.float64)
    codes, scales = quant.quantize(xb, bits)
    s = scales.astype(np.float64)[:, None]
    # bound: 1/2 code step, plus the fp32 rounding of x / scale (|x / scale| <= qmax, 2^-24 relative)
    # and of scale itself — together under qmax * 2^-23 code steps
    assert np.all(np.abs(codes * s - xe) <= (0.5 + qm * 2.0 ** -23) * s)
    cand = np.arange(-qm, qm + 1, dtype=np.float64)
    dist = np.abs(cand[None, None, :] * s[:, :, None] - xe[:, :, None])
    best = cand[np.argmin(dist, axis=2)]
    srt = np.sort(dist, axis=2)
    clear = (srt[:, :, 1] - srt[:, :, 0]) > 1e-5 * s
    assert clear.mean() > 0.99
    assert np.array_equal(codes[clear], best[clear].astype(np.int8))


@pytest.mark.parametrize("bits", [8, 4])
def test_special_rows(bits):
    qm = quant.qmax_of(bits)
    z = np.zeros((2, 32), np.uint16)
    z[1, 5] = 0x8000   # -0.0
    codes, scales = quant.quantize(z, bits)
    assert np.all(scales == 0) and np.all(codes == 0)
    assert np.all(quant.dequantize(codes, scales) == 0)
    # the absmax element maps to +-qmax; negating the row negates the codes (rint is symmetric)
    rng = np.random.default_rng(13)
    x = rng.standard_normal((16, 32)).astype(np.float32)
    xb = (x.view(np.uint32) >> 16).astype(np.uint16)
    c, s = quant.quantize(xb, bits)
    cn, sn = quant.quantize(xb ^ np.uint16(0x8000), bits)
    assert np.array_equal(sn, s) and np.array_equal(cn, -c)
    xe = quant.bf16_bits_to_f32(xb)
    am = np.argmax(np.abs(xe), axis=1)
    assert np.array_equal(c[np.arange(16), am], (np.sign(xe[np.arange(16), am]) * qm).astype(np.int8))
    # one spike: the other elements collapse to 0 when below scale / 2
    sp = np.zeros((1, 16), np.float32)
    sp[0, 3] = 1024.0
    sp[0, 7] = 1.0
    c1, s1 = quant.quantize(_bits(sp), bits)
    assert c1[0, 3] == qm and c1[0, 7] == 0 and s1[0] == np.float32(1024.0 / qm)


def test_bf16_rounding_matches_torch():
    rng = np.random.default_rng(14)
    x = (rng.standard_normal(100000) * np.exp(rng.uniform(-20, 20, 100000))).astype(np.float32)
    x[:4] = [1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8, -(1.0 + 2.0 ** -8), 0.0]   # exact ties: to even
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(quant.f32_to_bf16_bits(x), ref)


def test_pack4_layout():
    c = np.array([[1, -1, 7, -7, 0, -8 + 1]], np.int8)
    p = quant.pack4(c)
    assert p.tolist() == [[0xF1, 0x97, 0x90]]
    rng = np.random.default_rng(15)
    r = rng.integers(-7, 8, size=(9, 64)).astype(np.int8)
    assert np.array_equal(quant.unpack4(quant.pack4(r)), r)
