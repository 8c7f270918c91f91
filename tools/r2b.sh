timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pytest_parity.log 2>&1; tail -1 gpurun_out/pytest_parity.log
for r in 1 2; do
for v in "ASR_NO_LEAN=0" "ASR_NO_LEAN=1"; do
env $v timeout 600 python bench.py --points=ctx32k,c2 --no-cpu-baseline --no-e2e > gpurun_out/sk.log 2>&1
python - "$v" <<'PY'
import json,sys
for l in open('gpurun_out/sk.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['points']
        print(sys.argv[1], '8k', round(d['ms_per_step']*1000,2), round(d['detail']['stage_ms_per_step_profiled']['combine_decide_tick']*1000,2), '32k', round(p['ctx32k']['ms_per_step']*1000,2), 'b64', round(p['c2']['ms_per_step']*1000,1))
PY
done; done
