"""NEXT-4 parity: asr_kv_quantize / asr_kv_dequantize through the C ABI
against oracle/quant.py (R-quant).  The codes are integers decided in fp32 on both sides,
so codes, scales and dequantised bf16 values must be bit-exact."""
import numpy as np
import pytest
import torch

import gen
from oracle import quant
from paper_2512_11221_b200 import asr_kv_dequantize, asr_kv_quantize

pytestmark = pytest.mark.gpu


def _special_rows(n: int) -> np.ndarray:
    """Edge rows: zeros, -0, one spike, a negative absmax, values near the fp32 subnormal range, exact
    ties of x / scale at .5 (lattice of half steps), bf16 max."""
    r = np.zeros((7, n), np.float32)
    r[1, :] = -0.0
    r[2, n // 3] = 1024.0
    r[2, n // 2] = 3.0
    r[3, :] = np.linspace(-2.0, 1.0, n)
    r[3, 0] = -4.0
    r[4, :] = np.linspace(-1.0, 1.0, n) * 2.0 ** -120
    r[5, :] = (np.arange(n) % 16 - 7.5) * 0.25            # many x / scale near half-integers
    r[5, 0] = 127 * 0.25
    r[6, :] = 3.3895313892515355e38 * np.where(np.arange(n) % 2, 1.0, -0.5)
    bits = (r.view(np.uint32) >> 16).astype(np.uint16)
    return bits


def _inputs(n: int, rows: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal((rows, n)) * np.exp(rng.uniform(-6, 4, (rows, 1)))).astype(np.float32)
    bits = (x.view(np.uint32) >> 16).astype(np.uint16)
    sp = _special_rows(n)
    k = min(rows, sp.shape[0])
    bits[:k] = sp[:k]
    return bits


def _run(xb: np.ndarray, bits: int):
    rows, n = xb.shape
    kv = torch.from_numpy(xb.view(np.int16)).cuda().view(torch.bfloat16)
    codes = torch.empty((rows, n if bits == 8 else n // 2), dtype=torch.int8 if bits == 8 else torch.uint8,
                        device="cuda")
    scales = torch.empty(rows, dtype=torch.float32, device="cuda")
    asr_kv_quantize(kv, codes, scales, bits=bits)
    back = torch.empty_like(kv)
    asr_kv_dequantize(codes, scales, back, bits=bits)
    torch.cuda.synchronize()
    return codes.cpu().numpy(), scales.cpu().numpy(), back.view(torch.int16).cpu().numpy().view(np.uint16)


def _check(xb, bits, got):
    codes, scales, back = got
    oc, osc = quant.quantize(xb, bits)
    assert np.array_equal(scales.view(np.uint32), osc.view(np.uint32))
    want_codes = oc if bits == 8 else quant.pack4(oc)
    assert np.array_equal(codes.view(np.uint8), want_codes.view(np.uint8))
    assert np.array_equal(back, quant.dequantize(oc, osc))


@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("n", [8, 16, 32, 64, 128, 256])
@pytest.mark.parametrize("rows", [1, 7, 37, 4099])
def test_quant_parity_small(n, bits, rows):
    xb = _inputs(n, rows, seed=100 * n + rows + bits)
    _check(xb, bits, _run(xb, bits))


@pytest.mark.parametrize("bits", [8, 4])
def test_quant_parity_llama_kv(bits):
    """Rows of the seeded LLaMA-3-8B-shaped K/V (the generator's distribution), layout [token][L][2][Hkv][d]."""
    g = gen.GenParams(seed=31, L=32, Hq=32, Hkv=8, d=128)
    k, v = gen.kv(g, 0, 100, 40)                      # [40][32][8][128] bf16 bits each
    tier = np.stack([k, v], axis=2).reshape(-1, 128)   # [token][L][2][Hkv] rows of d
    _check(tier, bits, _run(tier, bits))


@pytest.mark.parametrize("bits", [8, 4])
def test_quant_parity_fullsize_sampled(bits):
    """The frozen tier of the bench's configs[1] point (≈6900 frozen tokens at 8K, 512 rows each:
    3.53M rows of 128, 904 MB of bf16) in one launch, as bench.py's quant point times it; every row is
    independent, so sampled rows (plus the first and last) are checked against the oracle row by row."""
    rows, n = 6900 * 512, 128
    gk = torch.Generator(device="cuda").manual_seed(5)
    kv = (torch.randn((rows, n), device="cuda", generator=gk) *
          torch.exp(torch.empty((rows, 1), device="cuda").uniform_(-4, 3, generator=gk))).to(torch.bfloat16)
    codes = torch.empty((rows, n if bits == 8 else n // 2), dtype=torch.int8 if bits == 8 else torch.uint8,
                        device="cuda")
    scales = torch.empty(rows, dtype=torch.float32, device="cuda")
    asr_kv_quantize(kv, codes, scales, bits=bits)
    back = torch.empty_like(kv)
    asr_kv_dequantize(codes, scales, back, bits=bits)
    torch.cuda.synchronize()
    rng = np.random.default_rng(6)
    idx = torch.from_numpy(np.unique(np.concatenate([[0, rows - 1], rng.integers(0, rows, 2000)]))).cuda()
    xb = kv[idx].view(torch.int16).cpu().numpy().view(np.uint16)
    got = (codes[idx].cpu().numpy(), scales[idx].cpu().numpy(), back[idx].view(torch.int16).cpu().numpy().view(np.uint16))
    _check(xb, bits, got)
