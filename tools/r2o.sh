# bisect the batch-64 attention-alone regression (asr_time_attention GB/s)
export PYTHONUNBUFFERED=1
python tools/build.py > /dev/null 2>&1
for r in 1 2; do
for v in "" build/ab/libasr_e6a5664.so build/ab/libasr_9b39c64.so build/ab/libasr_60692ef.so build/ab/libasr_8a67efb.so; do
ASR_LIB_PATH=$v timeout 600 python bench.py --batch 64 --steps 8 --warmup 3 --points= --no-cpu-baseline --no-e2e > gpurun_out/o.log 2>&1
python - "lib=${v:-HEAD}" <<'PY'
import json,sys
d=[json.loads(l) for l in open('gpurun_out/o.log') if l.startswith('{')][0]
print(sys.argv[1], round(d['ms_per_step']*1000,1), 'attn alone frac', round(d['roofline']['frac'],3))
PY
done; done
