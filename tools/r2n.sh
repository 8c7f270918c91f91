# configs[2] (batch 64): HEAD vs e6a5664 on one box
export PYTHONUNBUFFERED=1
python tools/build.py > /dev/null 2>&1
for r in 1 2; do
for v in "" build/ab/libasr_e6a5664.so; do
ASR_LIB_PATH=$v timeout 600 python bench.py --batch 64 --steps 16 --warmup 4 --points= --no-cpu-baseline --no-e2e > gpurun_out/n.log 2>&1
python - "lib=${v:-HEAD}" <<'PY'
import json,sys
d=[json.loads(l) for l in open('gpurun_out/n.log') if l.startswith('{')][0]
print(sys.argv[1], round(d['ms_per_step']*1000,1), 'attn alone frac', round(d['roofline']['frac'],3), {k: round(v*1000,1) for k,v in d['detail']['stage_ms_per_step_profiled'].items()})
PY
done; done
