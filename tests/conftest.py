"""Test configuration: registers the `gpu` marker and puts the repo root on sys.path.

`-m "not gpu"` tests run on a CPU-only box (oracle pins, generator, host logic, C-ABI exports);
`-m gpu` tests need a B200 and call the CUDA path through the C ABI.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    # Build every native library once, here, in the main process (atomic writes, file-locked), so no
    # test ever triggers a build from a worker thread.  The CUDA targets need nvcc (present in this
    # image on CPU and GPU boxes); without it only the host targets are built.
    import shutil
    from tools.build import NVCC, build_all
    build_all(cuda=bool(shutil.which("nvcc") or os.path.exists(NVCC)))
