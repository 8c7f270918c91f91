# A/B of the rate-balanced static split (ASR_SK_BALANCE): batch 1 at 8K / 32K, batch 4 and 8 at 8K
export PYTHONUNBUFFERED=1
python tools/build.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/parity_bal.log 2>&1; echo parity=$?
for r in 1 2; do
for v in 0 1; do
ASR_SK_BALANCE=$v timeout 600 python bench.py --points=ctx32k --no-cpu-baseline --no-e2e > gpurun_out/sk.log 2>&1
python - "bal=$v" <<'PY'
import json,sys
for l in open('gpurun_out/sk.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['points']
        print(sys.argv[1], 'b1 8k', round(d['ms_per_step']*1000,2), 'attn', d['roofline'].get('achieved'), '32k', round(p['ctx32k']['ms_per_step']*1000,2))
PY
for b in 4 8; do
ASR_SK_BALANCE=$v timeout 600 python bench.py --batch $b --points= --no-cpu-baseline --no-e2e > gpurun_out/skb.log 2>&1
python - "bal=$v b=$b" <<'PY'
import json,sys
for l in open('gpurun_out/skb.log'):
    if l.startswith('{'):
        d=json.loads(l)
        print(sys.argv[1], round(d['ms_per_step']*1000,2), 'attn GB/s', d['roofline'].get('achieved'))
PY
done
done; done
for v in "ASR_SK_DYN=8" "ASR_SK_DYN=0 ASR_SK_BALANCE=1" "ASR_SK_DYN=0 ASR_SK_BALANCE=0"; do
env $v timeout 600 python bench.py --batch 64 --steps 16 --points= --no-cpu-baseline --no-e2e > gpurun_out/skb.log 2>&1
python - "$v b=64" <<'PY'
import json,sys
for l in open('gpurun_out/skb.log'):
    if l.startswith('{'):
        d=json.loads(l)
        print(sys.argv[1], round(d['ms_per_step']*1000,2), 'attn GB/s', d['roofline'].get('achieved'))
PY
done
ASR_SK_BALANCE=1 timeout 600 python bench.py --points= --no-cpu-baseline --no-e2e --timeline > gpurun_out/tl_bal.log 2>&1
ASR_SK_BALANCE=0 timeout 600 python bench.py --points= --no-cpu-baseline --no-e2e --timeline > gpurun_out/tl_nobal.log 2>&1
echo done
