# phase-D block size (co-residency beside the batch-1 attention CTA under PDL): 512 (default) / 256 / 128
export PYTHONUNBUFFERED=1
python tools/build.py > /dev/null 2>&1
ASR_LIB_PATH=build/ab/libasr_pd128.so timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -1
for r in 1 2; do
for v in "" build/ab/libasr_pd256.so build/ab/libasr_pd128.so; do
ASR_LIB_PATH=$v timeout 600 python bench.py --points=ctx32k --no-cpu-baseline --no-e2e > gpurun_out/l.log 2>&1
python - "lib=${v:-default}" <<'PY'
import json,sys
d=[json.loads(l) for l in open('gpurun_out/l.log') if l.startswith('{')][0]
print(sys.argv[1], 'b1 8k', round(d['ms_per_step']*1000,2), 'phaseD', round(d['detail']['stage_ms_per_step_profiled']['combine_decide_tick']*1000,2), '32k', round(d['points']['ctx32k']['ms_per_step']*1000,2))
PY
done; done
ASR_LIB_PATH=build/ab/libasr_pd128.so timeout 600 python bench.py --points= --no-cpu-baseline --no-e2e --timeline > gpurun_out/l.log 2>&1
python - <<'PY'
import json
d=[json.loads(l) for l in open('gpurun_out/l.log') if l.startswith('{')][0]
print('pd128 timeline', json.dumps(d['detail']['timeline'])[:400])
PY
