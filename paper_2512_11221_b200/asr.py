"""Thin ctypes binding of libasr.so (include/asr.h) — argument marshalling only.

Every step of the ASR-KF-EGR hot path runs in the library's sm_100a kernels; this module
only converts torch tensors / numpy arrays into pointers.  There is no CPU fallback: if
libasr.so is missing or no CUDA device is present, the calls raise.

The function names are the C ABI's (asr_create, asr_step, asr_restore, asr_stats, asr_read_kv,
asr_stage_times, asr_destroy); `Context` is a small convenience wrapper over them.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ASR_LIB_PATH") or os.path.join(_HERE, "libasr.so")   # override: A/B of two builds

ASR_OK, ASR_E_INVALID, ASR_E_INVARIANT, ASR_E_CUDA, ASR_E_OOM, ASR_E_CAPACITY, ASR_E_NCCL, ASR_E_STATE = 0, 1, 2, 3, 4, 5, 6, 7
KV_BF16, KV_F32 = 0, 1
ENTROPY_GIVEN = 2   # asr_step_io.logits_dtype: logits_prev holds fp32 H[batch] (asr_sample_entropy)
MEM_DEVICE, MEM_HOST = 0, 1
SR, WR, FR = 1, 2, 3
EVICT_BELADY, EVICT_AT_FREEZE = 0, 1
STAGES = ("entropy_append_recover_compact", "attention_score", "combine_decide_tick", "step_total")


class AsrError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"asr status {code}: {msg}")
        self.code = code


class asr_config(ctypes.Structure):
    _fields_ = [("n_layers", ctypes.c_int32), ("n_q_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("batch", ctypes.c_int32), ("max_context", ctypes.c_int32),
                ("kv_dtype", ctypes.c_int32), ("window", ctypes.c_int32), ("tau", ctypes.c_float),
                ("softness", ctypes.c_float), ("history_window", ctypes.c_int32),
                ("pinned_prefix", ctypes.c_int32), ("score_mode", ctypes.c_int32), ("tick_order", ctypes.c_int32),
                ("vocab", ctypes.c_int32), ("entropy_temperature", ctypes.c_float), ("det_enable", ctypes.c_int32),
                ("det_baseline", ctypes.c_int32), ("det_cooldown", ctypes.c_int32), ("wr_window", ctypes.c_int32),
                ("det_z", ctypes.c_float), ("det_sigma_floor", ctypes.c_float), ("fr_clear_counts", ctypes.c_int32),
                ("host_mirror", ctypes.c_int32), ("profile_stages", ctypes.c_int32), ("device", ctypes.c_int32),
                ("evict_min_absence", ctypes.c_int32), ("pool_reserve", ctypes.c_int32), ("pool_tokens", ctypes.c_int64),
                ("score_heads", ctypes.c_int32), ("evict_policy", ctypes.c_int32), ("mirror_bits", ctypes.c_int32),
                ("per_layer_ledgers", ctypes.c_int32)]


class asr_step_io(ctypes.Structure):
    _fields_ = [("q", ctypes.c_void_p), ("k_new", ctypes.c_void_p), ("v_new", ctypes.c_void_p),
                ("logits_prev", ctypes.c_void_p), ("logits_dtype", ctypes.c_int32), ("memory", ctypes.c_int32),
                ("o", ctypes.c_void_p), ("entropy", ctypes.c_void_p)]


class asr_stats_t(ctypes.Structure):
    _fields_ = [("step", ctypes.c_int64), ("total", ctypes.c_int64), ("attended", ctypes.c_int64),
                ("active", ctypes.c_int64), ("frozen", ctypes.c_int64), ("frozen_this_step", ctypes.c_int64),
                ("restored_this_step", ctypes.c_int64), ("compression", ctypes.c_double),
                ("entropy", ctypes.c_float), ("entropy_valid", ctypes.c_int32),
                ("recovery_action", ctypes.c_int32), ("rewalk_requested", ctypes.c_int32),
                ("bytes_h2d", ctypes.c_int64), ("bytes_d2h", ctypes.c_int64), ("device_error", ctypes.c_uint32),
                ("resident", ctypes.c_int64), ("evicted_this_step", ctypes.c_int64),
                ("prefetched_this_step", ctypes.c_int64), ("demand_restored_this_step", ctypes.c_int64),
                ("h2d_stall_ns", ctypes.c_int64), ("free_slots", ctypes.c_int64), ("allreduce_bytes", ctypes.c_int64)]


class asr_ledger_view(ctypes.Structure):
    _fields_ = [("residency", ctypes.c_void_p), ("timer", ctypes.c_void_p), ("count", ctypes.c_void_p),
                ("freeze_step", ctypes.c_void_p), ("active_list", ctypes.c_void_p),
                ("active_len", ctypes.c_void_p), ("scores", ctypes.c_void_p), ("capacity", ctypes.c_int32),
                ("dequantized", ctypes.c_void_p)]


EXPORTS = ("asr_config_defaults", "asr_create", "asr_step", "asr_restore", "asr_stats", "asr_read_kv",
           "asr_stage_times", "asr_set_profile", "asr_timeline", "asr_flush", "asr_destroy", "asr_last_error",
           "asr_step_attend", "asr_step_decide", "asr_score_partials", "asr_nccl_unique_id", "asr_attach_nccl",
           "asr_time_attention", "asr_sample", "asr_sample_entropy", "asr_step_policy", "asr_kv_quantize",
           "asr_kv_dequantize")

_lib = None
_lib_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Load libasr.so (raises if it was not built: there is no fallback).  Thread-safe: configured on
    a local, published last."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python tools/build.py` (needs nvcc, sm_100a)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32 = ctypes.c_void_p, ctypes.c_int32
        L.asr_config_defaults.argtypes = [ctypes.POINTER(asr_config)]
        L.asr_config_defaults.restype = None
        L.asr_create.argtypes = [ctypes.POINTER(asr_config), vp, vp, vp, i32, i32, vp, ctypes.POINTER(vp)]
        L.asr_step.argtypes = [vp, ctypes.POINTER(asr_step_io), vp]
        L.asr_restore.argtypes = [vp, i32, i32, vp]
        L.asr_stats.argtypes = [vp, i32, ctypes.POINTER(asr_stats_t), ctypes.POINTER(asr_ledger_view)]
        L.asr_read_kv.argtypes = [vp, i32, i32, i32, vp, vp]
        L.asr_stage_times.argtypes = [vp, ctypes.POINTER(ctypes.c_double), i32, ctypes.POINTER(ctypes.c_int64)]
        L.asr_destroy.argtypes = [vp]
        L.asr_set_profile.argtypes = [vp, i32]
        L.asr_timeline.argtypes = [vp, ctypes.POINTER(ctypes.c_double), i32]
        L.asr_flush.argtypes = [vp, vp]
        L.asr_step_attend.argtypes = [vp, ctypes.POINTER(asr_step_io), vp]
        L.asr_step_decide.argtypes = [vp, vp]
        L.asr_score_partials.argtypes = [vp, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int64)]
        L.asr_nccl_unique_id.argtypes = [vp, i32]
        L.asr_attach_nccl.argtypes = [vp, vp, i32, i32]
        L.asr_time_attention.argtypes = [vp, i32, vp]
        L.asr_sample.argtypes = [vp, i32, i32, i32, ctypes.c_float, i32, ctypes.c_float, vp, vp, vp]
        L.asr_sample_entropy.argtypes = [vp, i32, i32, i32, ctypes.c_float, i32, ctypes.c_float, vp, vp,
                                         ctypes.c_float, vp, vp]
        L.asr_step_policy.argtypes = [vp, vp, vp, i32, vp, vp]
        L.asr_kv_quantize.argtypes = [vp, ctypes.c_int64, i32, i32, vp, vp, vp]
        L.asr_kv_dequantize.argtypes = [vp, vp, ctypes.c_int64, i32, i32, vp, vp]
        for f in ("asr_create", "asr_step", "asr_restore", "asr_stats", "asr_read_kv", "asr_stage_times",
                  "asr_set_profile", "asr_timeline", "asr_flush", "asr_destroy", "asr_step_attend",
                  "asr_step_decide", "asr_score_partials", "asr_nccl_unique_id", "asr_attach_nccl",
                  "asr_time_attention", "asr_sample", "asr_sample_entropy", "asr_step_policy", "asr_kv_quantize",
                  "asr_kv_dequantize"):
            getattr(L, f).restype = ctypes.c_int
        L.asr_last_error.argtypes = []
        L.asr_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != ASR_OK:
        raise AsrError(rc, lib().asr_last_error().decode())


@dataclasses.dataclass
class Config:
    """Mirror of asr_config; defaults = the paper's K=32, tau=0.5, k=2 at LLaMA-3-8B shape."""
    n_layers: int = 32
    n_q_heads: int = 32
    n_kv_heads: int = 8
    head_dim: int = 128
    batch: int = 1
    max_context: int = 8192
    kv_dtype: int = KV_BF16
    window: int = 32
    tau: float = 0.5
    softness: float = 2.0
    history_window: int = 0
    pinned_prefix: int = 0
    score_mode: int = 0
    tick_order: int = 0
    vocab: int = 128256
    entropy_temperature: float = 1.0
    det_enable: int = 1
    det_baseline: int = 64
    det_cooldown: int = 16
    wr_window: int | None = None   # default: window
    det_z: float = 3.0
    det_sigma_floor: float = 0.05
    fr_clear_counts: int = 0
    host_mirror: int = 1
    profile_stages: int = 0
    device: int = 0
    evict_min_absence: int = 2       # pressure mode: never evict tokens returning in fewer steps
    pool_reserve: int = 0            # pressure mode: free slots kept for demand restores (0 = batch)
    pool_tokens: int = 0             # 0 = full residency; > 0 = pressure mode (device slot pool)
    score_heads: int = 0             # head-sharded mode: H of Eq. 2 over all shards (0 = n_q_heads)
    evict_policy: int = 0            # pressure mode: EVICT_BELADY (capacity-driven) or EVICT_AT_FREEZE
    mirror_bits: int = 0             # pressure mode: 0 bf16 host mirror, 8 the INT8 frozen tier (R-quant)
    per_layer_ledgers: int = 0       # NEXT-3: one ledger per (sequence, layer); per-sequence calls take
                                     # seq = b * n_layers + l

    def c(self) -> asr_config:
        v = dataclasses.asdict(self)
        if v["wr_window"] is None:
            v["wr_window"] = self.window
        return asr_config(**v)


def _ptr(x) -> int | None:
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays must be C-contiguous")
        return x.ctypes.data
    if not x.is_contiguous():
        raise ValueError("tensors must be contiguous")
    return x.data_ptr()


_KIND = {"bf16": ("bfloat16", (np.uint16,)), "f32": ("float32", (np.float32,)), "i32": ("int32", (np.int32,)),
         "i8": ("int8", (np.int8, np.uint8)), "u8": ("uint8", (np.uint8, np.int8))}


def _arg(name: str, x, kinds, shape=None, host: bool | None = None, device: int | None = None):
    """Validate one caller buffer before its pointer crosses the C ABI (no asserts: survives -O).
    kinds: allowed element kinds (keys of _KIND); shape: exact shape, or a leading-dims prefix given as
    (..., n) tuples of ints where None matches anything; host: None = either memory kind."""
    if x is None:
        raise ValueError(f"{name}: missing")
    if isinstance(x, np.ndarray):
        ok = any(x.dtype == np.dtype(t) for k in kinds for t in _KIND[k][1])
        is_host = True
    else:
        import torch
        ok = any(x.dtype == getattr(torch, _KIND[k][0]) for k in kinds)
        is_host = not x.is_cuda
        if not is_host and device is not None and x.device.index != device:
            raise ValueError(f"{name}: on cuda:{x.device.index}, the context is on cuda:{device}")
    if not ok:
        raise ValueError(f"{name}: dtype {x.dtype} not in {kinds}")
    if host is not None and is_host != host:
        raise ValueError(f"{name}: expected {'host' if host else 'device'} memory")
    if shape is not None:
        xs = tuple(x.shape)
        if len(xs) != len(shape) or any(w is not None and w != h for w, h in zip(shape, xs)):
            raise ValueError(f"{name}: shape {xs}, expected {tuple('*' if w is None else w for w in shape)}")
    _ptr(x)
    return x


def _is_host(x) -> bool:
    return isinstance(x, np.ndarray) or not x.is_cuda


def _dtype_code(x) -> int:
    if isinstance(x, np.ndarray):
        return KV_BF16 if x.dtype == np.uint16 else KV_F32
    import torch
    return KV_BF16 if x.dtype == torch.bfloat16 else KV_F32


def _stream(stream) -> int:
    if stream is not None:
        return int(stream)
    import torch
    return torch.cuda.current_stream().cuda_stream


def asr_create(cfg: Config, prompt_k, prompt_v, prompt_len, stream=None) -> ctypes.c_void_p:
    """prompt_k/v: [B][P_max][L][Hkv][d] (torch CUDA, torch CPU or numpy); prompt_len: ints [B]."""
    c = cfg.c()
    pl = np.ascontiguousarray(np.asarray(prompt_len, np.int32))
    stride = int(prompt_k.shape[1]) if prompt_k is not None and prompt_k.ndim >= 2 else 0
    mem = MEM_HOST if prompt_k is None or _is_host(prompt_k) else MEM_DEVICE
    out = ctypes.c_void_p()
    _check(lib().asr_create(ctypes.byref(c), _ptr(prompt_k), _ptr(prompt_v), pl.ctypes.data, stride, mem,
                            _stream(stream), ctypes.byref(out)))
    _CFGS[out.value] = cfg
    return out


_CFGS: dict = {}   # ctx handle value -> Config (for argument validation)


def _io(ctx, q, k_new, v_new, o, logits_prev, entropy, entropy_given=False):
    cfg = _CFGS.get(ctx.value if isinstance(ctx, ctypes.c_void_p) else ctx)
    host = _is_host(q)
    if cfg is not None:
        B, L, Hq, Hkv, d = cfg.batch, cfg.n_layers, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim
        kv = ["bf16"] if cfg.kv_dtype == KV_BF16 else ["f32"]
        dev = None if host else cfg.device
        _arg("q", q, kv, (B, L, Hq, d), host, dev)
        _arg("k_new", k_new, kv, (B, L, Hkv, d), host, dev)
        _arg("v_new", v_new, kv, (B, L, Hkv, d), host, dev)
        _arg("o", o, ["f32"], (B, L, Hq, d), host, dev)
        if logits_prev is not None and entropy_given:
            _arg("entropy (given)", logits_prev, ["f32"], (B,), host, dev)
        elif logits_prev is not None:
            _arg("logits_prev", logits_prev, ["bf16", "f32"], (B, cfg.vocab), host, dev)
        if entropy is not None:
            _arg("entropy", entropy, ["f32"], (B,), host, dev)
    code = ENTROPY_GIVEN if entropy_given else (_dtype_code(logits_prev) if logits_prev is not None else 0)
    return asr_step_io(_ptr(q), _ptr(k_new), _ptr(v_new), _ptr(logits_prev), code,
                       MEM_HOST if host else MEM_DEVICE, _ptr(o), _ptr(entropy))


def asr_step(ctx, q, k_new, v_new, o, logits_prev=None, entropy=None, stream=None, entropy_given=False) -> None:
    """entropy_given: logits_prev is fp32 H[batch] from asr_sample_entropy instead of the logits rows."""
    io = _io(ctx, q, k_new, v_new, o, logits_prev, entropy, entropy_given)
    _check(lib().asr_step(ctx, ctypes.byref(io), _stream(stream)))


def asr_step_attend(ctx, q, k_new, v_new, o, logits_prev=None, entropy=None, stream=None) -> None:
    io = _io(ctx, q, k_new, v_new, o, logits_prev, entropy)
    _check(lib().asr_step_attend(ctx, ctypes.byref(io), _stream(stream)))


def asr_step_decide(ctx, stream=None) -> None:
    _check(lib().asr_step_decide(ctx, _stream(stream)))


def asr_score_partials(ctx):
    """(device pointer, element count) of the packed per-token partial score sums of a head shard
    (count = sum over sequences of |A_b|; synchronises)."""
    p, n = ctypes.c_void_p(), ctypes.c_int64()
    _check(lib().asr_score_partials(ctx, ctypes.byref(p), ctypes.byref(n)))
    return p.value, n.value


def asr_nccl_unique_id() -> bytes:
    buf = (ctypes.c_char * 128)()
    _check(lib().asr_nccl_unique_id(buf, 128))
    return bytes(buf)


def asr_attach_nccl(ctx, unique_id: bytes, nranks: int, rank: int) -> None:
    buf = (ctypes.c_char * 128).from_buffer_copy(unique_id)
    _check(lib().asr_attach_nccl(ctx, buf, nranks, rank))


def asr_restore(ctx, seq: int, level: int, stream=None) -> None:
    _check(lib().asr_restore(ctx, seq, level, _stream(stream)))


def asr_stats(ctx, seq: int, capacity: int = 0, detail: bool = False) -> dict:
    st = asr_stats_t()
    view = None
    arrays = {}
    if detail:
        arrays = {"residency": np.zeros(capacity, np.uint8), "timer": np.zeros(capacity, np.int32),
                  "count": np.zeros(capacity, np.uint32), "freeze_step": np.zeros(capacity, np.int32),
                  "active_list": np.zeros(capacity, np.int32), "active_len": np.zeros(1, np.int32),
                  "scores": np.zeros(capacity, np.float32), "dequantized": np.zeros(capacity, np.uint8)}
        view = asr_ledger_view(*(arrays[k].ctypes.data for k in ("residency", "timer", "count", "freeze_step",
                                                                 "active_list", "active_len", "scores")),
                               capacity, arrays["dequantized"].ctypes.data)
    _check(lib().asr_stats(ctx, seq, ctypes.byref(st), ctypes.byref(view) if view is not None else None))
    out = {f[0]: getattr(st, f[0]) for f in asr_stats_t._fields_}
    if detail:
        n, A = int(st.total), int(arrays["active_len"][0])
        out["ledger"] = {k: arrays[k][:n] for k in ("residency", "timer", "count", "freeze_step")}
        out["dequantized"] = arrays["dequantized"][:n]
        out["active_list"] = arrays["active_list"][:A]
        out["scores"] = arrays["scores"][:A]
    return out


def asr_read_kv(ctx, cfg: Config, seq: int, pos: int, from_mirror: bool = False):
    dt = np.uint16 if cfg.kv_dtype == KV_BF16 else np.float32
    k = np.zeros((1 if cfg.per_layer_ledgers else cfg.n_layers, cfg.n_kv_heads, cfg.head_dim), dt)
    v = np.zeros_like(k)
    _check(lib().asr_read_kv(ctx, seq, pos, int(from_mirror), k.ctypes.data, v.ctypes.data))
    return k, v


def asr_stage_times(ctx):
    ms = (ctypes.c_double * len(STAGES))()
    n = ctypes.c_int64()
    _check(lib().asr_stage_times(ctx, ms, len(STAGES), ctypes.byref(n)))
    return list(ms), int(n.value)


def asr_tail_trace(ctx, n_slots: int = 26):
    """Diagnostics (ASR_TIMELINE=1): per-warp stamps of the fused tail of the last step, us relative
    to the step start, -1 = not stamped: array [148 * 32][8] (row = CTA * 32 + slot)."""
    rows, cols = 148 * 32, 8
    total = n_slots + rows * cols
    us = (ctypes.c_double * total)()
    _check(lib().asr_timeline(ctx, us, total))
    return np.frombuffer(us, dtype=np.float64)[n_slots:].reshape(rows, cols).copy()


def asr_timeline(ctx) -> list:
    """[pre start, end, attention start, end, post start, end, decide end, next-A end, combine end,
    entropy units end, append units end, phase B start, phase B end, first attention CTA end,
    post released, fused tail: barrier arrival, barrier release, tile warps' decide / tick / count /
    look-back / write ends, first tile warp done, CTA past the attention, past the phase-B wait] (us)."""
    us = (ctypes.c_double * 26)()
    _check(lib().asr_timeline(ctx, us, 26))
    return list(us)


def asr_flush(ctx, stream=None) -> None:
    _check(lib().asr_flush(ctx, _stream(stream)))


def asr_set_profile(ctx, on: bool) -> None:
    _check(lib().asr_set_profile(ctx, int(bool(on))))


def asr_sample(logits, uniforms, token_out, temperature: float = 1.0, top_k: int = 0, top_p: float = 1.0,
               stream=None) -> None:
    """NEXT-1 next-token draw (include/asr.h asr_sample): logits [B][V] bf16/fp32, uniforms [B] fp32,
    token_out [B] int32 — CUDA tensors (torch) of the caller."""
    import torch
    _arg("logits", logits, ["bf16", "f32"], (None, None), False)
    B, V = logits.shape
    _arg("uniforms", uniforms, ["f32"], (B,), False, logits.device.index)
    _arg("token_out", token_out, ["i32"], (B,), False, logits.device.index)
    dt = KV_BF16 if logits.dtype == torch.bfloat16 else KV_F32
    _check(lib().asr_sample(ctypes.c_void_p(logits.data_ptr()), dt, B, V, float(temperature), int(top_k),
                            float(top_p), ctypes.c_void_p(uniforms.data_ptr()), ctypes.c_void_p(token_out.data_ptr()),
                            _stream(stream)))


def asr_sample_entropy(logits, uniforms, token_out, entropy_out, temperature: float = 1.0, top_k: int = 0,
                       top_p: float = 1.0, entropy_temperature: float = 1.0, stream=None) -> None:
    """NEXT-1 + (a6) in one pass over each row (include/asr.h asr_sample_entropy): the draw of asr_sample
    and entropy_out[b] = H(softmax(logits[b] / entropy_temperature)) — pass entropy_out to the next
    asr_step as logits_prev with entropy_given=True."""
    import torch
    _arg("logits", logits, ["bf16", "f32"], (None, None), False)
    B, V = logits.shape
    _arg("uniforms", uniforms, ["f32"], (B,), False, logits.device.index)
    _arg("token_out", token_out, ["i32"], (B,), False, logits.device.index)
    _arg("entropy_out", entropy_out, ["f32"], (B,), False, logits.device.index)
    dt = KV_BF16 if logits.dtype == torch.bfloat16 else KV_F32
    _check(lib().asr_sample_entropy(_vp(logits), dt, B, V, float(temperature), int(top_k), float(top_p), _vp(uniforms),
                                    _vp(token_out), float(entropy_temperature), _vp(entropy_out), _stream(stream)))


def asr_kv_quantize(kv, codes, scales, bits: int = 8, stream=None) -> None:
    """NEXT-4 frozen-tier quantisation (include/asr.h asr_kv_quantize): kv [..., n] bf16 (rows = all
    leading dims), codes [rows][n] int8 (bits 8) or [rows][n/2] uint8 (bits 4), scales [rows] fp32 —
    CUDA tensors (torch) of the caller."""
    n = kv.shape[-1]
    rows = kv.numel() // n if n else 0
    _arg("kv", kv, ["bf16"], None, False)
    _arg("codes", codes, ["i8", "u8"], (rows, n if bits == 8 else n // 2), False, kv.device.index)
    _arg("scales", scales, ["f32"], (rows,), False, kv.device.index)
    _check(lib().asr_kv_quantize(_vp(kv), rows, n, int(bits), _vp(codes), _vp(scales), _stream(stream)))


def asr_kv_dequantize(codes, scales, kv, bits: int = 8, stream=None) -> None:
    """NEXT-4 inverse map (include/asr.h asr_kv_dequantize): codes + scales -> kv [..., n] bf16."""
    n = kv.shape[-1]
    rows = kv.numel() // n if n else 0
    _arg("kv", kv, ["bf16"], None, False)
    _arg("codes", codes, ["i8", "u8"], (rows, n if bits == 8 else n // 2), False, kv.device.index)
    _arg("scales", scales, ["f32"], (rows,), False, kv.device.index)
    _check(lib().asr_kv_dequantize(_vp(codes), _vp(scales), rows, n, int(bits), _vp(kv), _stream(stream)))


def _vp(x) -> ctypes.c_void_p:
    return ctypes.c_void_p(_ptr(x))


def asr_time_attention(ctx, reps: int, stream=None) -> None:
    _check(lib().asr_time_attention(ctx, int(reps), _stream(stream)))


def asr_destroy(ctx) -> None:
    _CFGS.pop(ctx.value if isinstance(ctx, ctypes.c_void_p) else ctx, None)
    _check(lib().asr_destroy(ctx))


class Context:
    """Convenience owner of one asr_ctx."""

    def __init__(self, cfg: Config, prompt_k, prompt_v, prompt_len, stream=None):
        self.cfg = cfg
        self._h = asr_create(cfg, prompt_k, prompt_v, prompt_len, stream)

    def step(self, q, k_new, v_new, o, logits_prev=None, entropy=None, stream=None, entropy_given=False):
        asr_step(self._h, q, k_new, v_new, o, logits_prev, entropy, stream, entropy_given)

    def attend(self, q, k_new, v_new, o, logits_prev=None, entropy=None, stream=None):
        asr_step_attend(self._h, q, k_new, v_new, o, logits_prev, entropy, stream)

    def decide(self, stream=None):
        asr_step_decide(self._h, stream)

    def score_partials(self):
        return asr_score_partials(self._h)

    def attach_nccl(self, unique_id: bytes, nranks: int, rank: int):
        asr_attach_nccl(self._h, unique_id, nranks, rank)

    def restore(self, seq: int, level: int, stream=None):
        asr_restore(self._h, seq, level, stream)

    @property
    def n_seq(self) -> int:
        """Sequences of the context's per-sequence calls (batch, or batch * n_layers with per-layer ledgers)."""
        return self.cfg.batch * (self.cfg.n_layers if self.cfg.per_layer_ledgers else 1)

    def stats(self, seq: int, detail: bool = False) -> dict:
        return asr_stats(self._h, seq, self.cfg.max_context, detail)

    def read_kv(self, seq: int, pos: int, from_mirror: bool = False):
        return asr_read_kv(self._h, self.cfg, seq, pos, from_mirror)

    def stage_times(self):
        return asr_stage_times(self._h)

    def timeline(self):
        return asr_timeline(self._h)

    def flush(self, stream=None):
        asr_flush(self._h, stream)

    def set_profile(self, on: bool):
        asr_set_profile(self._h, on)

    def step_policy(self, scores, logits_prev=None, entropy=None, stream=None):
        """NEXT-2 policy replay step: scores [B][max_context] fp32 (CUDA tensor) instead of attention."""
        import torch
        c = self.cfg
        _arg("scores", scores, ["f32"], (self.n_seq, c.max_context), False, c.device)
        lg = None if logits_prev is None else _arg("logits_prev", logits_prev, ["bf16", "f32"],
                                                   (c.batch, c.vocab), False, c.device)
        if entropy is not None:
            _arg("entropy", entropy, ["f32"], (c.batch,), False, c.device)
        dt = 0 if lg is None or lg.dtype == torch.bfloat16 else 1
        _check(lib().asr_step_policy(self._h, ctypes.c_void_p(scores.data_ptr()),
                                     None if lg is None else ctypes.c_void_p(lg.data_ptr()), dt,
                                     None if entropy is None else ctypes.c_void_p(entropy.data_ptr()),
                                     _stream(stream)))

    def time_attention(self, reps: int, stream=None):
        asr_time_attention(self._h, reps, stream)

    def close(self):
        if self._h:
            asr_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
