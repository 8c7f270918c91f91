for r in 1 2; do
for lib in build/ab/libasr_HEAD.so paper_2512_11221_b200/libasr.so; do
ASR_LIB_PATH=$PWD/$lib timeout 600 python bench.py --points=ctx32k --no-cpu-baseline --no-e2e > gpurun_out/sk.log 2>&1
python - "$lib" <<'PY'
import json,sys
for l in open('gpurun_out/sk.log'):
    if l.startswith('{'):
        d=json.loads(l); p=d['points']
        print(sys.argv[1][-22:], '8k', round(d['ms_per_step']*1000,2), round(d['detail']['stage_ms_per_step_profiled']['combine_decide_tick']*1000,2), '32k', round(p['ctx32k']['ms_per_step']*1000,2))
PY
done; done
timeout 300 python bench.py --points= --no-cpu-baseline --no-e2e --timeline > gpurun_out/bench_tl.log 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/bench_tl.log'):
    if l.startswith('{'):
        d=json.loads(l); t=d['detail']['timeline']; print(round(d['ms_per_step']*1000,2), t['pre_start_end_attn_start_end_post_start_end_us'], t['post_decide_end_next_list_end_combine_end_us'], t['cta_past_attention_past_phaseB_wait_us'])
PY
