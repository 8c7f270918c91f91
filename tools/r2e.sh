timeout 1200 python -m pytest tests/test_sample_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/pytest_se.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest_se.log
