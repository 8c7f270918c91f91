timeout 1500 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo bench_rc=$?
tail -c 600 gpurun_out/bench_default.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
