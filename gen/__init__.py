"""Seeded synthetic inputs (LAT / GAUSS families) — test and bench infrastructure.

This module holds none of the method's arithmetic (see gen/asrgen.h for the spec).  The host
functions return numpy arrays (used by the oracle side of tests); the device functions fill
torch CUDA tensors (used by bench.py and GPU tests).  Both are compiled from the same
integer-only header and are bit-identical.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LAT, GAUSS = 0, 1


class _Params(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("family", ctypes.c_int32), ("L", ctypes.c_int32),
                ("Hq", ctypes.c_int32), ("Hkv", ctypes.c_int32), ("d", ctypes.c_int32),
                ("hot_permille", ctypes.c_int32), ("a_hot", ctypes.c_int32),
                ("needle_pos", ctypes.c_int32), ("needle_b", ctypes.c_int32),
                ("query_first", ctypes.c_int32), ("query_count", ctypes.c_int32),
                ("vocab", ctypes.c_int32), ("spike_first", ctypes.c_int32),
                ("spike_period", ctypes.c_int32), ("spike_count", ctypes.c_int32),
                ("peak_base16", ctypes.c_int32), ("peak_step16", ctypes.c_int32)]


@dataclasses.dataclass
class GenParams:
    seed: int = 1
    family: int = LAT
    L: int = 1
    Hq: int = 2
    Hkv: int = 2
    d: int = 16
    hot_permille: int = 0      # W0 = 0 (all-cold), W1 = 300
    a_hot: int = 4
    needle_pos: int = -1
    needle_b: int = -1
    query_first: int = -1
    query_count: int = 0
    vocab: int = 0
    spike_first: int = -1
    spike_period: int = 0
    spike_count: int = 0
    peak_base16: int = 224     # baseline peak logit 14.0 ...
    peak_step16: int = 8       # ... stepping by 0.5 over 8 levels

    def c(self) -> _Params:
        return _Params(*(getattr(self, f[0]) for f in _Params._fields_))


_host = None
_dev = None
_lock = threading.Lock()


def host_lib() -> ctypes.CDLL:
    """Thread-safe loader: configured on a local, published last (under a lock)."""
    global _host
    if _host is not None:
        return _host
    with _lock:
        if _host is not None:
            return _host
        path = os.path.join(_HERE, "libasrgen_host.so")
        import sys
        if os.path.dirname(_HERE) not in sys.path:
            sys.path.insert(0, os.path.dirname(_HERE))
        from tools.build import build_gen_host
        build_gen_host()
        L = ctypes.CDLL(path)
        P = ctypes.POINTER(_Params)
        vp, ci = ctypes.c_void_p, ctypes.c_int
        L.asrgen_host_kv.argtypes = [P, ci, ci, ci, vp, vp, ci]
        L.asrgen_host_q.argtypes = [P, ci, ci, vp, ci]
        L.asrgen_host_logits.argtypes = [P, ci, ci, vp, ci]
        for f in ("asrgen_host_is_hot", "asrgen_host_is_needle", "asrgen_host_peak_index"):
            getattr(L, f).argtypes = [P, ci, ci]
            getattr(L, f).restype = ci
        for f in ("asrgen_host_is_query_step", "asrgen_host_is_spike_step"):
            getattr(L, f).argtypes = [P, ci]
            getattr(L, f).restype = ci
        L.asrgen_host_mix.argtypes = [ctypes.c_uint64]
        L.asrgen_host_mix.restype = ctypes.c_uint64
        _host = L
    return _host


def _np_dtype(dtype: str):
    return {"bf16": (np.uint16, 0), "f32": (np.float32, 1)}[dtype]


def kv(p: GenParams, b: int, pos0: int, npos: int, dtype: str = "bf16"):
    """K, V for sequence b, positions [pos0, pos0+npos): arrays [npos][L][Hkv][d] (bf16 bits or f32)."""
    nd, code = _np_dtype(dtype)
    k = np.empty((npos, p.L, p.Hkv, p.d), nd)
    v = np.empty_like(k)
    pc = p.c()
    host_lib().asrgen_host_kv(ctypes.byref(pc), b, pos0, npos, k.ctypes.data, v.ctypes.data, code)
    return k, v


def q(p: GenParams, b: int, step: int, dtype: str = "bf16"):
    """Query of sequence b at decode step `step`: [L][Hq][d]."""
    nd, code = _np_dtype(dtype)
    out = np.empty((p.L, p.Hq, p.d), nd)
    pc = p.c()
    host_lib().asrgen_host_q(ctypes.byref(pc), b, step, out.ctypes.data, code)
    return out


def logits(p: GenParams, b: int, step: int, dtype: str = "bf16"):
    """Logits row of sequence b produced at decode step `step`: [vocab]."""
    nd, code = _np_dtype(dtype)
    out = np.empty((p.vocab,), nd)
    pc = p.c()
    host_lib().asrgen_host_logits(ctypes.byref(pc), b, step, out.ctypes.data, code)
    return out


def is_hot(p: GenParams, b: int, pos: int) -> bool:
    pc = p.c()
    return bool(host_lib().asrgen_host_is_hot(ctypes.byref(pc), b, pos))


def is_needle(p: GenParams, b: int, pos: int) -> bool:
    pc = p.c()
    return bool(host_lib().asrgen_host_is_needle(ctypes.byref(pc), b, pos))


def is_query_step(p: GenParams, step: int) -> bool:
    pc = p.c()
    return bool(host_lib().asrgen_host_is_query_step(ctypes.byref(pc), step))


def is_spike_step(p: GenParams, step: int) -> bool:
    pc = p.c()
    return bool(host_lib().asrgen_host_is_spike_step(ctypes.byref(pc), step))


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns (uint16) to float32."""
    return (a.astype(np.uint32) << 16).view(np.float32)


# ---------------------------------------------------------------- device side (torch tensors)

def dev_lib() -> ctypes.CDLL:
    global _dev
    if _dev is not None:
        return _dev
    with _lock:
        if _dev is not None:
            return _dev
        path = os.path.join(_HERE, "libasrgen_dev.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `python tools/build.py` (needs nvcc)")
        L = ctypes.CDLL(path)
        P = ctypes.POINTER(_Params)
        vp, ci = ctypes.c_void_p, ctypes.c_int
        L.asrgen_dev_kv.argtypes = [P, ci, vp, ci, ci, vp, vp, ci, vp]
        L.asrgen_dev_q.argtypes = [P, ci, ci, vp, ci, vp]
        L.asrgen_dev_logits.argtypes = [P, ci, ci, vp, ci, vp]
        for f in ("asrgen_dev_kv", "asrgen_dev_q", "asrgen_dev_logits"):
            getattr(L, f).restype = ci
        _dev = L
    return _dev


def _code(t) -> int:
    import torch
    if t.dtype == torch.bfloat16:
        return 0
    if t.dtype == torch.float32:
        return 1
    raise TypeError(t.dtype)


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def dev_kv(p: GenParams, B: int, pos0: int, npos: int, k_out, v_out, pos0_dev=None) -> None:
    """Fill k_out/v_out [B][npos][L][Hkv][d] (torch CUDA tensors) for positions pos0(+pos0_dev[b])+t."""
    pc = p.c()
    rc = dev_lib().asrgen_dev_kv(ctypes.byref(pc), B, None if pos0_dev is None else pos0_dev.data_ptr(),
                                 pos0, npos, k_out.data_ptr() if k_out is not None else None,
                                 v_out.data_ptr() if v_out is not None else None,
                                 _code(k_out if k_out is not None else v_out), _stream())
    if rc:
        raise RuntimeError(f"asrgen_dev_kv failed: {rc}")


def dev_q(p: GenParams, B: int, step: int, out) -> None:
    pc = p.c()
    rc = dev_lib().asrgen_dev_q(ctypes.byref(pc), B, step, out.data_ptr(), _code(out), _stream())
    if rc:
        raise RuntimeError(f"asrgen_dev_q failed: {rc}")


def dev_logits(p: GenParams, B: int, step: int, out) -> None:
    pc = p.c()
    rc = dev_lib().asrgen_dev_logits(ctypes.byref(pc), B, step, out.data_ptr(), _code(out), _stream())
    if rc:
        raise RuntimeError(f"asrgen_dev_logits failed: {rc}")


# ---------------------------------------------------------------- policy-replay score traces (NEXT-2)

def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = x + np.uint64(0x9E3779B97F4A7C15)
    z = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def score_trace(kind: str, batch: int, n: int, seed: int = 1, p: GenParams | None = None) -> np.ndarray:
    """Per-position relevance scores s_j, constant over the steps, fp32 [batch][n] — the input of a
    policy replay (asr_step_policy / OracleSeq.step_policy).  kind: "w0" every token 0.25 (all-cold
    under tau in (0.25, 1.5]); "w1" 1.5 for the LAT hot set of `p` (30 % with hot_permille=300), else
    0.25; "uniform" u_j in [0, 1) from a counter hash of (seed, b, j) with 2^-24 resolution (so
    `s < tau` is decided identically in fp32 and fp64 for tau on that lattice)."""
    if kind == "w0":
        return np.full((batch, n), 0.25, np.float32)
    if kind == "w1":
        assert p is not None
        out = np.full((batch, n), 0.25, np.float32)
        for b in range(batch):
            for j in range(n):
                if is_hot(p, b, j):
                    out[b, j] = 1.5
        return out
    if kind == "uniform":
        with np.errstate(over="ignore"):
            idx = (np.uint64(seed) << np.uint64(40)) + (np.arange(batch, dtype=np.uint64)[:, None] << np.uint64(24)) \
                + np.arange(n, dtype=np.uint64)[None, :]
            h = _splitmix64(idx)
        return ((h >> np.uint64(40)).astype(np.float64) * 2.0 ** -24).astype(np.float32)
    raise ValueError(kind)
