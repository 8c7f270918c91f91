"""fp64 CPU oracle of the ASR-KF-EGR generation step (arXiv 2512.11221) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this package.  The product path (paper_2512_11221_b200/) never imports it and shares no
code with it.  The arithmetic lives in oracle/orc.c (plain C, fp64); this file only marshals
numpy arrays through ctypes.  See orc.h for the passage each function follows.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LEVELS = {"SR": 1, "WR": 2, "FR": 3}


class _Cfg(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int), ("Hq", ctypes.c_int), ("Hkv", ctypes.c_int), ("d", ctypes.c_int),
                ("window", ctypes.c_int), ("tau", ctypes.c_double), ("softness", ctypes.c_double),
                ("history_window", ctypes.c_int), ("pinned_prefix", ctypes.c_int),
                ("score_scaled", ctypes.c_int), ("tick_skip_new", ctypes.c_int), ("vocab", ctypes.c_int),
                ("ent_temp", ctypes.c_double), ("det_enable", ctypes.c_int), ("det_baseline", ctypes.c_int),
                ("det_cooldown", ctypes.c_int), ("wr_window", ctypes.c_int), ("det_z", ctypes.c_double),
                ("det_sigma_floor", ctypes.c_double), ("fr_clear_counts", ctypes.c_int)]


class _Out(ctypes.Structure):
    _fields_ = [("step", ctypes.c_int), ("n", ctypes.c_int), ("attended", ctypes.c_int),
                ("active_post", ctypes.c_int), ("frozen_post", ctypes.c_int),
                ("frozen_this_step", ctypes.c_int), ("restored_this_step", ctypes.c_int),
                ("recovery_action", ctypes.c_int), ("rewalk_requested", ctypes.c_int),
                ("entropy_valid", ctypes.c_int), ("entropy", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {f[0]: getattr(self, f[0]) for f in self._fields_}


@dataclasses.dataclass
class OrcCfg:
    L: int = 1
    Hq: int = 2
    Hkv: int = 2
    d: int = 16
    window: int = 16
    tau: float = 0.5
    softness: float = 2.0
    history_window: int = 0          # 0 = infinite (R-W)
    pinned_prefix: int = 0
    score_scaled: int = 0
    tick_skip_new: int = 0           # 0 = R0 (literal Alg. 1 order)
    vocab: int = 0
    ent_temp: float = 1.0
    det_enable: int = 1
    det_baseline: int = 64
    det_cooldown: int = 16
    wr_window: int | None = None     # default: the sliding window K
    det_z: float = 3.0
    det_sigma_floor: float = 0.05
    fr_clear_counts: int = 0

    def c(self) -> _Cfg:
        vals = dataclasses.asdict(self)
        if vals["wr_window"] is None:
            vals["wr_window"] = self.window
        return _Cfg(**vals)


_lib = None
_lib_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Load (building first if stale) liborc.so.  Thread-safe: the CDLL is fully configured on a
    local and published last, under a lock, so no caller ever sees it without its argtypes."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        path = os.path.join(_HERE, "liborc.so")
        import sys
        if os.path.dirname(_HERE) not in sys.path:
            sys.path.insert(0, os.path.dirname(_HERE))
        from tools.build import build_oracle
        build_oracle()
        L = ctypes.CDLL(path)
        vp, ci = ctypes.c_void_p, ctypes.c_int
        C, O = ctypes.POINTER(_Cfg), ctypes.POINTER(_Out)
        L.orc_seq_new.argtypes = [C, ci, ci]
        L.orc_seq_new.restype = vp
        L.orc_seq_free.argtypes = [vp]
        L.orc_step.argtypes = [vp, vp, ci, vp, vp, ci, vp, ci, vp, vp, vp, O]
        L.orc_step.restype = ci
        L.orc_step_policy.argtypes = [vp, vp, ctypes.c_double, ci, vp, O]
        L.orc_step_policy.restype = ci
        L.orc_restore.argtypes = [vp, ci]
        L.orc_restore.restype = ci
        L.orc_n.argtypes = [vp]
        L.orc_n.restype = ci
        L.orc_ledger.argtypes = [vp, vp, vp, vp, vp]
        L.orc_duration.argtypes = [ctypes.c_uint32, ctypes.c_double]
        L.orc_duration.restype = ci
        L.orc_entropy.argtypes = [vp, ci, ci, ctypes.c_double]
        L.orc_entropy.restype = ctypes.c_double
        L.orc_attend_head.argtypes = [vp, ci, vp, vp, ci, ci, ci, vp]
        L.orc_score_token.argtypes = [vp, ci, vp, ci, ci, ci, ci, ci, ci]
        L.orc_score_token.restype = ctypes.c_double
        _lib = L
    return _lib


def _code(a: np.ndarray) -> int:
    if a.dtype == np.uint16:
        return 0
    if a.dtype == np.float32:
        return 1
    raise TypeError(f"oracle inputs are bf16 bits (uint16) or float32, got {a.dtype}")


def duration(c: int, k: float) -> int:
    """Eq. 3: floor(sqrt(c)/k)."""
    return lib().orc_duration(c, k)


def entropy(logits: np.ndarray, temp: float = 1.0) -> float:
    a = np.ascontiguousarray(logits)
    return lib().orc_entropy(a.ctypes.data, _code(a), a.size, temp)


def attend_head(q: np.ndarray, K: np.ndarray, V: np.ndarray) -> np.ndarray:
    """Eq. 1 for one (layer, head): q [d], K, V [n][d] (bf16 bits or f32) -> out [d] fp64."""
    q, K, V = (np.ascontiguousarray(x) for x in (q, K, V))
    n, d = K.shape
    assert q.shape == (d,) and V.shape == (n, d) and K.dtype == V.dtype
    out = np.empty(d, np.float64)
    lib().orc_attend_head(q.ctypes.data, _code(q), K.ctypes.data, V.ctypes.data, _code(K), n, d, out.ctypes.data)
    return out


def score_token(q: np.ndarray, k: np.ndarray, scaled: bool = False) -> float:
    """Eq. 2 for one token: q [L][Hq][d], k [L][Hkv][d]."""
    q, k = np.ascontiguousarray(q), np.ascontiguousarray(k)
    L, Hq, d = q.shape
    assert k.shape[0] == L and k.shape[2] == d
    return lib().orc_score_token(q.ctypes.data, _code(q), k.ctypes.data, _code(k), L, Hq, k.shape[1], d, int(scaled))


class OracleSeq:
    """One sequence's ledger + the step of Alg. 1."""

    def __init__(self, cfg: OrcCfg, capacity: int, prompt_len: int):
        self.cfg = cfg
        self.capacity = capacity
        self._c = cfg.c()
        self._h = lib().orc_seq_new(ctypes.byref(self._c), capacity, prompt_len)
        if not self._h:
            raise ValueError("orc_seq_new: bad capacity / prompt length")
        self._act = np.empty(capacity, np.int32)
        self._scores = np.empty(capacity, np.float64)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().orc_seq_free(h)
            self._h = None

    @property
    def n(self) -> int:
        return lib().orc_n(self._h)

    def step(self, q: np.ndarray, K: np.ndarray, V: np.ndarray, logits_prev: np.ndarray | None = None):
        """q [L][Hq][d]; K, V [capacity][L][Hkv][d] with positions < n+1 filled.
        Returns (O [L][Hq][d] fp64, attended positions, scores per attended, stats dict)."""
        c = self.cfg
        assert K.shape[0] >= self.capacity and K.shape[1:] == (c.L, c.Hkv, c.d), K.shape
        q = np.ascontiguousarray(q)
        K, V = np.ascontiguousarray(K), np.ascontiguousarray(V)   # the C side reads dense rows
        O = np.empty((c.L, c.Hq, c.d), np.float64)
        out = _Out()
        lp = None if logits_prev is None else np.ascontiguousarray(logits_prev)
        rc = lib().orc_step(self._h, q.ctypes.data, _code(q), K.ctypes.data, V.ctypes.data, _code(K),
                            None if lp is None else lp.ctypes.data, 0 if lp is None else _code(lp),
                            O.ctypes.data, self._act.ctypes.data, self._scores.ctypes.data,
                            ctypes.byref(out))
        if rc:
            raise ValueError("orc_step: capacity exceeded")
        A = out.attended
        return O, self._act[:A].copy(), self._scores[:A].copy(), out.as_dict()

    def step_policy(self, below: np.ndarray, H: float | None = None):
        """Policy-only step: below[pos] = 1 if position pos scores < tau this step."""
        b = np.ascontiguousarray(below, dtype=np.uint8)
        assert b.size >= self.n + 1
        out = _Out()
        rc = lib().orc_step_policy(self._h, b.ctypes.data, 0.0 if H is None else float(H),
                                   0 if H is None else 1, self._act.ctypes.data, ctypes.byref(out))
        if rc:
            raise ValueError("orc_step_policy: capacity exceeded")
        return self._act[:out.attended].copy(), out.as_dict()

    def restore(self, level: str | int) -> int:
        lv = LEVELS[level] if isinstance(level, str) else int(level)
        return lib().orc_restore(self._h, lv)

    def ledger(self) -> dict:
        n = self.n
        res = np.empty(n, np.uint8)
        timer = np.empty(n, np.int32)
        count = np.empty(n, np.uint32)
        fstep = np.empty(n, np.int32)
        lib().orc_ledger(self._h, res.ctypes.data, timer.ctypes.data, count.ctypes.data, fstep.ctypes.data)
        return {"residency": res, "timer": timer, "count": count, "freeze_step": fstep}
