# batch-1 step: where the non-attention time goes (L2 flush on/off, graph on/off), timelines
export PYTHONUNBUFFERED=1
python tools/build.py > /dev/null 2>&1
for v in "X=0" "ASR_BENCH_NO_FLUSH=1" "ASR_NO_GRAPH=1" "ASR_NO_PDL=1"; do
env $v timeout 600 python bench.py --points= --no-cpu-baseline --no-e2e > gpurun_out/i.log 2>&1
env $v timeout 600 python bench.py --points= --no-cpu-baseline --no-e2e --timeline > gpurun_out/it.log 2>&1
python - "$v" <<'PY'
import json,sys
d=[json.loads(l) for l in open('gpurun_out/i.log') if l.startswith('{')][0]
t=[json.loads(l) for l in open('gpurun_out/it.log') if l.startswith('{')][0]
det=t['detail']
print(sys.argv[1], 'step', round(d['ms_per_step']*1000,2), 'stages', {k: round(v*1000,2) for k,v in d['detail']['stage_ms_per_step_profiled'].items()})
print('   tl step', round(t['ms_per_step']*1000,2), json.dumps(det.get('timeline'))[:420])
PY
done
python tools/graph_overhead.py 2>&1 | tail -5
