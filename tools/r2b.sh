timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pytest_parity.log 2>&1; tail -2 gpurun_out/pytest_parity.log
for r in 1 2; do
for lib in build/ab/libasr_b9f59eb.so paper_2512_11221_b200/libasr.so; do
ASR_LIB_PATH=$PWD/$lib timeout 600 python bench.py --points=ctx32k,c2 --no-cpu-baseline --no-e2e > gpurun_out/sk.log 2>&1
python - "$lib" <<'PY'
import json,sys
for l in open('gpurun_out/sk.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['points']
        print(sys.argv[1][-20:], '8k', round(d['ms_per_step']*1000,2), round(d['roofline']['frac'],3), '32k', round(p['ctx32k']['ms_per_step']*1000,2), round(p['ctx32k']['roofline']['frac'],3), 'b64', round(p['c2']['ms_per_step']*1000,1), round(p['c2']['roofline']['frac'],3))
PY
done; done
