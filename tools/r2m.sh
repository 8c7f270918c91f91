# phase D on a programmatic (PDL) edge after the attention, 512- vs 128-thread blocks (co-resident)
export PYTHONUNBUFFERED=1
python tools/build.py > /dev/null 2>&1
for r in 1 2; do
for v in "X=0" "ASR_PD_PROG=1" "ASR_PD_PROG=1 ASR_LIB_PATH=build/ab/libasr_pd128.so"; do
env $v timeout 600 python bench.py --points=ctx32k --no-cpu-baseline --no-e2e > gpurun_out/m.log 2>&1
python - "$v" <<'PY'
import json,sys
d=[json.loads(l) for l in open('gpurun_out/m.log') if l.startswith('{')][0]
print(sys.argv[1], 'b1 8k', round(d['ms_per_step']*1000,2), '32k', round(d['points']['ctx32k']['ms_per_step']*1000,2))
PY
done; done
