timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_abi.py -x -q -k "int8 or pressure or abi" > gpurun_out/pytest_int8.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest_int8.log
