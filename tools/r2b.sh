timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pytest_parity.log 2>&1; tail -5 gpurun_out/pytest_parity.log
