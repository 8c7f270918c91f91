timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo bench_rc=$?
bash tools/gpu_profile.sh r2_b1 > gpurun_out/prof_b1.log 2>&1; tail -1 gpurun_out/prof_b1.log
bash tools/gpu_profile.sh r2_32k --context 32768 --no-mirror > gpurun_out/prof_32k.log 2>&1; tail -1 gpurun_out/prof_32k.log
