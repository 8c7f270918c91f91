#!/bin/bash
# Profiling recipe for the bench workload (run under gpurun from the repo root).
#   1. plain run of the exact command line (must exit 0 before ncu touches it)
#   2. per-launch device times of the library's kernels (cold-cache, serialised) -> launches_<tag>.csv
#   3. one `--set full` capture of the attention kernel (the dominant kernel) -> attn_<tag>.ncu-rep
# The ncu runs only profile inside the NVTX range "timed" that bench.py opens around its timed steps
# (--nvtx), so the thousands of growth-phase launches are not replayed.
# Usage: tools/gpu_profile.sh <tag> [extra bench args...]
TAG=${1:-r1}; shift || true
ARGS="--steps 5 --warmup 3 --no-cpu-baseline --no-e2e --points= --nvtx $*"
timeout 600 python bench.py $ARGS > gpurun_out/plain_${TAG}.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" \
    -k regex:"attn|phase|copy_kernel|combine" --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py $ARGS > gpurun_out/ncu_launch_${TAG}.log 2>&1 || echo "ncu launch list failed"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
    -k regex:"attn|phase|combine" -c 4 -o gpurun_out/attn_${TAG} \
    python bench.py $ARGS > gpurun_out/ncu_full_${TAG}.log 2>&1 || echo "ncu full failed"
echo profile-done
