# rate-balanced cut: EWMA weight of a new rate measurement
export PYTHONUNBUFFERED=1
python tools/build.py > /dev/null 2>&1
for r in 1 2; do
for v in 0.5 0.25 0.75 1.0; do
ASR_SK_EWMA=$v timeout 600 python bench.py --points=ctx32k --no-cpu-baseline --no-e2e > gpurun_out/q.log 2>&1
python - "ewma=$v" <<'PY'
import json,sys
d=[json.loads(l) for l in open('gpurun_out/q.log') if l.startswith('{')][0]
print(sys.argv[1], 'b1 8k', round(d['ms_per_step']*1000,2), '32k', round(d['points']['ctx32k']['ms_per_step']*1000,2))
PY
done; done
