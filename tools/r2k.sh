# batch-64 phase A: entropy splits per unit (block count vs per-warp work)
export PYTHONUNBUFFERED=1
python tools/build.py > /dev/null 2>&1
for v in 8 16 32 64 8; do
ASR_ENT_PER_UNIT=$v timeout 600 python bench.py --batch 64 --steps 16 --points= --no-cpu-baseline --no-e2e --timeline > gpurun_out/k.log 2>&1
python - "epu=$v" <<'PY'
import json,sys
d=[json.loads(l) for l in open('gpurun_out/k.log') if l.startswith('{')][0]
t=d['detail']['timeline']
print(sys.argv[1], round(d['ms_per_step']*1000,1), 'phaseA stage', round(d['detail']['stage_ms_per_step_profiled']['entropy_append_recover_compact']*1000,1), 'tl pre', t['pre_start_end_attn_start_end_post_start_end_us'][:2], t['pre_entropy_end_append_end_phaseB_start_end_us'])
PY
done
