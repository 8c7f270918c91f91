for r in 1 2; do
for v in "ASR_TAIL_EXP=0" "ASR_TAIL_EXP=2" "ASR_FUSE_TAIL=0"; do
env $v timeout 300 python bench.py --points= --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.$r.log 2>&1
python -c "
import json
for l in open('gpurun_out/ab_$v.$r.log'):
  if l.startswith('{'):
    d=json.loads(l); print('$v', round(d['ms_per_step']*1000,2), round(d['detail']['step_ms_median']*1000,2), round(d['roofline']['ms_per_launch']*1000,2))
"
done; done
