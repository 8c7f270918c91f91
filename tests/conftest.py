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
