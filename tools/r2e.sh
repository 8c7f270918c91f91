timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -k "per_layer or tiny_w0 or entropy_given" > gpurun_out/pytest_pl.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest_pl.log
