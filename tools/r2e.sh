timeout 2400 python -m pytest tests/test_fullsize_gpu.py tests/test_needle_gpu.py -x -q > gpurun_out/pytest_full.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest_full.log
