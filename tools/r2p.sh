# batch-64 attention-alone after keeping the flat append out of the attention kernel; batch 1; parity
export PYTHONUNBUFFERED=1
python tools/build.py > /dev/null 2>&1
for r in 1 2; do
for v in "" build/ab/libasr_9b39c64.so; do
ASR_LIB_PATH=$v timeout 600 python bench.py --batch 64 --steps 8 --warmup 3 --points= --no-cpu-baseline --no-e2e > gpurun_out/p.log 2>&1
python - "lib=${v:-HEAD}" <<'PY'
import json,sys
d=[json.loads(l) for l in open('gpurun_out/p.log') if l.startswith('{')][0]
print(sys.argv[1], 'b64', round(d['ms_per_step']*1000,1), 'attn alone frac', round(d['roofline']['frac'],3), 'phaseA', round(d['detail']['stage_ms_per_step_profiled']['entropy_append_recover_compact']*1000,1))
PY
done; done
timeout 600 python bench.py --points=ctx32k --no-cpu-baseline --no-e2e > gpurun_out/p.log 2>&1
python - <<'PY'
import json
d=[json.loads(l) for l in open('gpurun_out/p.log') if l.startswith('{')][0]
print('HEAD b1 8k', round(d['ms_per_step']*1000,2), '32k', round(d['points']['ctx32k']['ms_per_step']*1000,2))
PY
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -x -q -k "not 32768" 2>&1 | tail -1
