# batch-1 cut variants: uniform, rate-balanced (default), cost model with item-boundary cost gamma
export PYTHONUNBUFFERED=1
python tools/build.py > /dev/null 2>&1
for r in 1 2; do
for v in "ASR_SK_BALANCE=0" "ASR_SK_BALANCE=1" "ASR_SK_BALANCE=2 ASR_SK_GAMMA=0" "ASR_SK_BALANCE=2 ASR_SK_GAMMA=1" "ASR_SK_BALANCE=2 ASR_SK_GAMMA=2" "ASR_SK_BALANCE=2 ASR_SK_GAMMA=4"; do
env $v timeout 600 python bench.py --points=ctx32k --no-cpu-baseline --no-e2e > gpurun_out/j.log 2>&1
python - "$v" <<'PY'
import json,sys
for l in open('gpurun_out/j.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['points']
        print(sys.argv[1], 'b1 8k', round(d['ms_per_step']*1000,2), 'attn', round(d['roofline']['achieved']), '32k', round(p['ctx32k']['ms_per_step']*1000,2))
PY
done; done
