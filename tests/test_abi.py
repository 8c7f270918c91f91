"""CPU checks of the C-ABI boundary (no compute calls: there is no GPU here).

- libasr.so loads and exports every function include/asr.h declares;
- the ctypes structs match the C layout (sizes and offsets, from a gcc-compiled probe);
- configuration errors are reported synchronously as ASR_E_INVALID with a message;
- the oracle and the product path share no code (no cross includes / imports).
"""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2512_11221_b200 import asr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "asr.h")


def declared_functions():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(asr_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol():
    names = declared_functions()
    assert set(names) == set(asr.EXPORTS), names
    out = subprocess.run(["nm", "-D", "--defined-only", asr.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (asr_\w+)", out))
    missing = set(names) - exported
    assert not missing, missing
    L = asr.lib()
    for n in names:
        assert hasattr(L, n)


def test_struct_layout_matches_header(tmp_path):
    probe = tmp_path / "probe.c"
    structs = {"asr_config": asr.asr_config, "asr_step_io": asr.asr_step_io, "asr_stats_t": asr.asr_stats_t,
               "asr_ledger_view": asr.asr_ledger_view}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "asr.h"', "int main(void){"]
    for s, cls in structs.items():
        lines.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{s}.{f} %zu\\n", offsetof({s}, {f}));')
    lines.append("return 0;}")
    probe.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(probe), "-o", str(exe)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for s, cls in structs.items():
        assert int(got[s]) == ctypes.sizeof(cls), s
        for f, _ in cls._fields_:
            assert int(got[f"{s}.{f}"]) == getattr(cls, f).offset, (s, f)


def test_defaults_are_the_papers():
    c = asr.asr_config()
    asr.lib().asr_config_defaults(ctypes.byref(c))
    assert (c.window, c.tau, c.softness) == (32, 0.5, 2.0)
    assert (c.n_layers, c.n_q_heads, c.n_kv_heads, c.head_dim, c.vocab) == (32, 32, 8, 128, 128256)


@pytest.mark.parametrize("bad", [dict(n_layers=0), dict(n_q_heads=6, n_kv_heads=4), dict(head_dim=48),
                                 dict(window=0), dict(softness=0.0), dict(history_window=129), dict(history_window=-1),
                                 dict(kv_dtype=7), dict(batch=0), dict(det_baseline=1000)])
def test_invalid_config_is_rejected_synchronously(bad):
    cfg = asr.Config(**bad)
    with pytest.raises(asr.AsrError) as e:
        asr.asr_create(cfg, None, None, [0] * max(cfg.batch, 1), stream=0)
    assert e.value.code == asr.ASR_E_INVALID
    assert asr.lib().asr_last_error()


def test_bad_prompt_length_rejected():
    with pytest.raises(asr.AsrError) as e:
        asr.asr_create(asr.Config(max_context=16), None, None, [20], stream=0)
    assert e.value.code == asr.ASR_E_INVALID


def test_oracle_and_product_share_no_code():
    csrc = os.path.join(ROOT, "paper_2512_11221_b200")
    for dirpath, _, files in os.walk(csrc):
        for f in files:
            if f.endswith((".cu", ".cpp", ".h", ".cuh", ".py")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"(?:#include|import|from)\s+[\"<]?(\w+)", txt), f
                assert "orc.h" not in txt and "asrgen" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".c", ".h", ".py")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            deps = re.findall(r"(?:#include\s+[\"<]([\w./]+)|^\s*(?:import|from)\s+([\w.]+))", txt, flags=re.M)
            deps = {a or b for a, b in deps}
            assert not any("asr" in x or "paper_2512" in x or "gen" == x.split(".")[0] for x in deps), (f, deps)


@pytest.mark.parametrize("args", [
    dict(logits=None), dict(dtype=5), dict(batch=0), dict(batch=65536), dict(vocab=0), dict(vocab=1 << 24),
    dict(temperature=float("nan")), dict(top_p=float("inf")), dict(uniforms=None), dict(token_out=None)])
def test_sample_invalid_arguments_rejected(args):
    """asr_sample validates before touching the device (include/asr.h): ASR_E_INVALID, no launch."""
    p = ctypes.c_void_p(16)   # never dereferenced: validation fails first
    a = dict(logits=p, dtype=asr.KV_BF16, batch=1, vocab=128256, temperature=1.0, top_k=0, top_p=1.0,
             uniforms=p, token_out=p)
    a.update(args)
    rc = asr.lib().asr_sample(a["logits"], a["dtype"], a["batch"], a["vocab"], a["temperature"], a["top_k"],
                              a["top_p"], a["uniforms"], a["token_out"], None)
    assert rc == asr.ASR_E_INVALID
    assert asr.lib().asr_last_error()


@pytest.mark.parametrize("fn,args", [
    (f, a) for f in ("asr_kv_quantize", "asr_kv_dequantize") for a in (
        dict(kv=None), dict(codes=None), dict(scales=None), dict(rows=-1), dict(rows=(1 << 40) + 1), dict(n=0),
        dict(n=48), dict(n=512), dict(bits=2), dict(bits=16), dict(kv=ctypes.c_void_p(24)),
        dict(codes=ctypes.c_void_p(20)), dict(bits=4, codes=ctypes.c_void_p(18)), dict(scales=ctypes.c_void_p(18)))])
def test_kv_quant_invalid_arguments_rejected(fn, args):
    """asr_kv_quantize / asr_kv_dequantize (NEXT-4) validate before touching the device: ASR_E_INVALID."""
    p = ctypes.c_void_p(256)   # never dereferenced: validation fails first
    a = dict(kv=p, rows=1024, n=128, bits=8, codes=p, scales=p)
    a.update(args)
    if fn == "asr_kv_quantize":
        rc = asr.lib().asr_kv_quantize(a["kv"], a["rows"], a["n"], a["bits"], a["codes"], a["scales"], None)
    else:
        rc = asr.lib().asr_kv_dequantize(a["codes"], a["scales"], a["rows"], a["n"], a["bits"], a["kv"], None)
    assert rc == asr.ASR_E_INVALID
    assert asr.lib().asr_last_error()


def test_kv_quant_zero_rows_is_a_noop():
    p = ctypes.c_void_p(256)
    assert asr.lib().asr_kv_quantize(p, 0, 128, 8, p, p, None) == 0
    assert asr.lib().asr_kv_dequantize(p, p, 0, 128, 4, p, None) == 0


def test_binding_has_no_shadowed_definitions():
    """Every top-level name of the ctypes binding is defined once (a second helper of the same name once
    silently replaced the first and broke numpy host-memory I/O)."""
    import ast
    tree = ast.parse(open(asr.__file__).read())
    names = [n.name for n in tree.body if isinstance(n, (ast.FunctionDef, ast.ClassDef))]
    assert len(names) == len(set(names)), sorted({n for n in names if names.count(n) > 1})


def test_binding_validates_buffers_before_the_abi():
    """The binding rejects wrong dtypes / shapes / memory kinds with ValueError (not assert: it must
    survive python -O) before any pointer reaches the library (an fp16 logits row or a
    bf16 `o` would otherwise be read / written out of bounds)."""
    import numpy as np
    import torch
    cfg = asr.Config(n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=16, batch=3, max_context=64, vocab=100)
    h = ctypes.c_void_p(0xDEAD0)
    asr._CFGS[h.value] = cfg
    try:
        bf, f32 = torch.bfloat16, torch.float32
        q = torch.zeros(3, 2, 4, 16, dtype=bf)
        kn = torch.zeros(3, 2, 2, 16, dtype=bf)
        o = torch.zeros(3, 2, 4, 16, dtype=f32)
        lg = torch.zeros(3, 100, dtype=bf)
        ent = torch.zeros(3, dtype=f32)
        io = asr._io(h, q, kn, kn, o, lg, ent)          # all valid (host memory)
        assert io.memory == asr.MEM_HOST and io.logits_dtype == asr.KV_BF16
        bad = [
            dict(q=q.to(torch.float16)),                  # wrong KV dtype
            dict(o=o.to(bf)),                             # bf16 o would be written as fp32
            dict(o=torch.zeros(3, 2, 4, 8, dtype=f32)),   # undersized o
            dict(logits_prev=lg.to(torch.float16)),       # fp16 logits read as fp32
            dict(logits_prev=torch.zeros(3, 99, dtype=bf)),
            dict(entropy=torch.zeros(2, dtype=f32)),
            dict(k_new=torch.zeros(3, 2, 4, 16, dtype=bf)),   # Hq heads instead of Hkv
            dict(q=torch.zeros(3, 2, 16, 4, dtype=bf).transpose(2, 3)),   # non-contiguous
        ]
        for kw in bad:
            a = dict(q=q, k_new=kn, v_new=kn, o=o, logits_prev=lg, entropy=ent)
            a.update(kw)
            with pytest.raises(ValueError):
                asr._io(h, **a)
        # numpy host buffers: bf16 as uint16 bits
        qn = np.zeros((3, 2, 4, 16), np.uint16)
        asr._io(h, qn, np.zeros((3, 2, 2, 16), np.uint16), np.zeros((3, 2, 2, 16), np.uint16),
                np.zeros((3, 2, 4, 16), np.float32), None, None)
        with pytest.raises(ValueError):
            asr._io(h, qn, np.zeros((3, 2, 2, 16), np.uint16), np.zeros((3, 2, 2, 16), np.uint16),
                    np.zeros((3, 2, 4, 16), np.float64), None, None)
    finally:
        asr._CFGS.pop(h.value, None)
