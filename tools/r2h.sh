# stage breakdown of the rate-balanced split at batch 8 / 64 (ASR_SK_DYN=0)
export PYTHONUNBUFFERED=1
python tools/build.py > /dev/null 2>&1
for v in 0 1; do
for b in 8 64; do
ASR_SK_DYN=0 ASR_SK_BALANCE=$v timeout 600 python bench.py --batch $b --steps 16 --points= --no-cpu-baseline --no-e2e --timeline > gpurun_out/h.log 2>&1
python - "bal=$v b=$b" <<'PY'
import json,sys
for l in open('gpurun_out/h.log'):
    if l.startswith('{'):
        d=json.loads(l); det=d['detail']
        print(sys.argv[1], round(d['ms_per_step']*1000,2), 'attn GB/s', round(d['roofline'].get('achieved')), det.get('stage_ms_per_step_profiled'))
        print('   ', json.dumps(det.get('timeline'))[:600])
PY
done; done
