for r in 1 2; do
for v in "ASR_DECIDE_POSITIONS=256" "ASR_DECIDE_POSITIONS=384" "ASR_DECIDE_POSITIONS=512" "ASR_DECIDE_POSITIONS=1024"; do
env $v timeout 600 python bench.py --points=ctx32k --no-cpu-baseline --no-e2e > gpurun_out/sk.log 2>&1
python - "$v" <<'PY'
import json,sys
for l in open('gpurun_out/sk.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['points']
        print(sys.argv[1], '8k', round(d['ms_per_step']*1000,2), round(d['detail']['stage_ms_per_step_profiled']['combine_decide_tick']*1000,2), '32k', round(p['ctx32k']['ms_per_step']*1000,2))
PY
done; done
