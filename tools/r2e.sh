timeout 1200 python -m pytest tests/test_sweep.py -x -q > gpurun_out/pytest_sweep.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest_sweep.log
timeout 600 python bench.py --points=sweep,sample --no-cpu-baseline --no-e2e > gpurun_out/bench_sweep.log 2>&1; echo rc=$?
python -c "
import json
for l in open('gpurun_out/bench_sweep.log'):
    if l.startswith('{'):
        d=json.loads(l); sw=d['detail']['sensitivity_sweep']; print(sw['workload'], round(sw['seconds'],2), round(sw['cell_steps_per_s'])); print(sw['table'][:3]); print(json.dumps(d['detail']['next_token_draw']))
"
