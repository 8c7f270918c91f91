set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2a.log 2>&1; echo rc=$? >> gpurun_out/pytest_r2a.log
timeout 300 python bench.py --points= --no-cpu-baseline > gpurun_out/bench_fused.log 2>&1
ASR_FUSE_TAIL=0 timeout 300 python bench.py --points= --no-cpu-baseline > gpurun_out/bench_nofuse.log 2>&1
timeout 300 python bench.py --points= --no-cpu-baseline --no-e2e --timeline > gpurun_out/bench_fused_tl.log 2>&1
timeout 300 python bench.py --points= --no-cpu-baseline --no-e2e --batch 64 --steps 16 --warmup 4 > gpurun_out/bench_fused_b64.log 2>&1
ASR_FUSE_TAIL=0 timeout 300 python bench.py --points= --no-cpu-baseline --no-e2e --batch 64 --steps 16 --warmup 4 > gpurun_out/bench_nofuse_b64.log 2>&1
tail -3 gpurun_out/pytest_r2a.log
