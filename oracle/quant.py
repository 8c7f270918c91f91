"""Oracle of NEXT-4: the frozen tier stored quantised — "hybrid compression combining
ASR-KF-EGR with quantization methods" (§Future Work).

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): plain numpy, no blocking or reordering beyond the
definitions below; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline may call it.

The paper names quantisation of the frozen tier as future work and fixes no scheme; the reading
(R-quant):

* a row is one head vector of the KV cache: (token, layer, K|V, KV head) -> head_dim values, as in the
  frozen tier's layout [token][L][2][Hkv][d] (bf16);
* symmetric per-row absmax quantisation to `bits` in {8, 4}: qmax = 2^(bits-1) - 1 (127 or 7),
  amax = max_e |x_e| (exact), scale = amax / qmax, code_e = clip(rint(x_e / scale), -qmax, qmax)
  (rint: round half to even); a row of zeros has scale 0 and codes 0;
* the floating point that decides the integer codes is fp32 (the kernel's precision, as the paper
  fixes none): the division amax / qmax and x_e / scale are IEEE fp32 divisions, rounded to nearest;
* dequantisation: x'_e = bf16_rn(fp32(code_e) * scale) (one fp32 product, rounded to nearest even
  bf16);
* storage: bits = 8 -> one int8 per value; bits = 4 -> two values per byte, element 2i in the low
  nibble and 2i+1 in the high nibble, each a 4-bit two's complement code.
"""
from __future__ import annotations

import numpy as np


def bf16_bits_to_f32(a: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) -> their exact fp32 values."""
    return (np.ascontiguousarray(a).astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit patterns, round to nearest even (finite inputs): add 0x7FFF plus the lowest
    kept bit to the fp32 bit pattern, keep the upper 16 bits."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def qmax_of(bits: int) -> int:
    assert bits in (8, 4), bits
    return (1 << (bits - 1)) - 1


def quantize(x_bits: np.ndarray, bits: int = 8):
    """R-quant, per row.  x_bits: [rows][n] bf16 bit patterns (uint16).
    Returns (codes [rows][n] int8, scales [rows] float32) — codes unpacked (see pack4)."""
    x = bf16_bits_to_f32(x_bits).reshape(x_bits.shape)
    q = np.float32(qmax_of(bits))
    rows, n = x.shape
    codes = np.zeros((rows, n), np.int8)
    scales = np.zeros(rows, np.float32)
    for r in range(rows):
        amax = np.float32(np.max(np.abs(x[r]))) if n else np.float32(0)
        scale = np.float32(amax / q)                      # fp32 / fp32, rounded to nearest
        scales[r] = scale
        if scale == 0:
            continue
        y = (x[r] / scale).astype(np.float32)             # element-wise fp32 division
        codes[r] = np.clip(np.rint(y), -q, q).astype(np.int8)
    return codes, scales


def pack4(codes: np.ndarray) -> np.ndarray:
    """[rows][n] int8 codes in [-7, 7] -> [rows][n/2] uint8: element 2i low nibble, 2i+1 high nibble."""
    c = codes.astype(np.int16) & 0xF
    return (c[:, 0::2] | (c[:, 1::2] << 4)).astype(np.uint8)


def unpack4(packed: np.ndarray) -> np.ndarray:
    """Inverse of pack4 (4-bit two's complement nibbles -> int8)."""
    lo = (packed & 0xF).astype(np.int16)
    hi = (packed >> 4).astype(np.int16)
    lo = np.where(lo >= 8, lo - 16, lo)
    hi = np.where(hi >= 8, hi - 16, hi)
    out = np.empty((packed.shape[0], packed.shape[1] * 2), np.int8)
    out[:, 0::2] = lo
    out[:, 1::2] = hi
    return out


def dequantize(codes: np.ndarray, scales: np.ndarray) -> np.ndarray:
    """R-quant dequantisation: [rows][n] int8 codes, [rows] fp32 scales -> [rows][n] bf16 bits."""
    y = (codes.astype(np.float32) * scales.astype(np.float32)[:, None]).astype(np.float32)
    return f32_to_bf16_bits(y)
