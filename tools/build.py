"""Build every native library of the repo in-tree.

- gen/libasrgen_host.so     gcc     seeded input generator, host build (test/bench infrastructure)
- gen/libasrgen_dev.so      nvcc    seeded input generator, sm_100a build (test/bench infrastructure)
- oracle/liborc.so          gcc     fp64 CPU oracle (test infrastructure)
- paper_2512_11221_b200/libasr.so   nvcc   the product: C-ABI library + sm_100a kernels

Each target is rebuilt only when one of its sources is newer than the .so.
"""
from __future__ import annotations

import contextlib
import fcntl
import glob
import os
import subprocess
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


_TLOCK = threading.Lock()


@contextlib.contextmanager
def _locked():
    """Serialise builds across threads (pytest workers) and processes (torchrun ranks)."""
    with _TLOCK:
        os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
        with open(os.path.join(ROOT, "build", ".lock"), "w") as f:
            fcntl.flock(f, fcntl.LOCK_EX)
            try:
                yield
            finally:
                fcntl.flock(f, fcntl.LOCK_UN)


def _tmp(out: str) -> str:
    """Every target is linked to a private temp path and os.replace()d into place, so a concurrent
    dlopen never sees a half-written file."""
    return f"{out}.tmp.{os.getpid()}.{threading.get_ident()}"


def _stale(out: str, srcs: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[0]} -> exit {r.returncode}")


def build_gen_host(force: bool = False) -> str:
    out = os.path.join(ROOT, "gen", "libasrgen_host.so")
    srcs = [os.path.join(ROOT, "gen", f) for f in ("asrgen.h", "asrgen_host.c")]
    with _locked():
        if force or _stale(out, srcs):
            _run(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _tmp(out), srcs[1]])
            os.replace(_tmp(out), out)
    return out


def build_oracle(force: bool = False) -> str:
    out = os.path.join(ROOT, "oracle", "liborc.so")
    srcs = [os.path.join(ROOT, "oracle", f) for f in ("orc.h", "orc.c")]
    with _locked():
        if force or _stale(out, srcs):
            _run(["gcc", "-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off", "-shared", "-fPIC",
                  "-o", _tmp(out), srcs[1], "-lm"])
            os.replace(_tmp(out), out)
    return out


def build_gen_dev(force: bool = False) -> str:
    out = os.path.join(ROOT, "gen", "libasrgen_dev.so")
    srcs = [os.path.join(ROOT, "gen", f) for f in ("asrgen.h", "asrgen_dev.cu")]
    with _locked():
        if force or _stale(out, srcs):
            _run([NVCC, *ARCH, "-O3", "-lineinfo", "-shared", "-cudart", "shared", "-Xcompiler", "-fPIC",
                  "-o", _tmp(out), srcs[1]])
            os.replace(_tmp(out), out)
    return out


def _nccl_include() -> str:
    """nccl.h of the NCCL that torch ships (headers only: libasr.so dlopens libnccl.so.2)."""
    try:
        import nvidia.nccl
        base = list(nvidia.nccl.__path__)[0]
    except Exception:
        import site
        base = os.path.join(site.getsitepackages()[0], "nvidia", "nccl")
    return os.path.join(base, "include")


def build_asr(force: bool = False, out: str | None = None) -> str:
    with _locked():
        return _build_asr(force, out)


def _build_asr(force: bool, out_path: str | None = None) -> str:
    pkg = os.path.join(ROOT, "paper_2512_11221_b200")
    out = out_path or os.path.join(pkg, "libasr.so")
    csrc = os.path.join(pkg, "csrc")
    cu = sorted(glob.glob(os.path.join(csrc, "*.cu")))
    cpp = sorted(glob.glob(os.path.join(csrc, "*.cpp")))
    hdr = sorted(glob.glob(os.path.join(csrc, "*.cuh")) + glob.glob(os.path.join(csrc, "*.h"))
                 + glob.glob(os.path.join(ROOT, "include", "*.h")))
    if not (force or _stale(out, cu + cpp + hdr)):
        return out
    objdir = os.path.join(ROOT, "build", "asr" if out_path is None else "asr_" + os.path.basename(out_path))
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    objs = []
    common = ["-I", os.path.join(ROOT, "include"), "-I", csrc]
    if os.environ.get("ASR_TAIL_TRACE") == "1":   # diagnostic build: per-warp stamps of the fused tail
        common.append("-DASR_TAIL_TRACE")
    if os.environ.get("ASR_CHECKS") == "1":       # diagnostic build: device-side bounds checks (kErrCheck)
        common.append("-DASR_CHECKS")
    common += os.environ.get("ASR_NVCC_DEFS", "").split()   # A/B experiments (e.g. -DASR_KPF=2)
    for s in cu:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xptxas", "-warn-spills", *common, "-c", s, "-o", o])
        objs.append(o)
    nccl_inc = _nccl_include()
    for s in cpp:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        _run([NVCC, "-O2", "-std=c++17", "-Xcompiler", "-fPIC,-Wall", *common, "-I", nccl_inc, "-c", s, "-o", o])
        objs.append(o)
    _run([NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", _tmp(out), *objs, "-ldl"])
    os.replace(_tmp(out), out)
    return out


def build_all(force: bool = False, cuda: bool = True) -> None:
    build_gen_host(force)
    build_oracle(force)
    if cuda:
        build_gen_dev(force)
        build_asr(force)


if __name__ == "__main__":
    if "--checks" in sys.argv:   # the bounds-checked diagnostic library, beside the product one
        os.environ["ASR_CHECKS"] = "1"
        print(build_asr(force=True, out=os.path.join(ROOT, "build", "libasr_checks.so")))
        sys.exit(0)
    if "--variant" in sys.argv:   # an experiment library: --variant NAME (flags from ASR_NVCC_DEFS)
        name = sys.argv[sys.argv.index("--variant") + 1]
        print(build_asr(force=True, out=os.path.join(ROOT, "build", "ab", f"libasr_{name}.so")))
        sys.exit(0)
    build_all(force="--force" in sys.argv, cuda="--no-cuda" not in sys.argv)
    print("built")
