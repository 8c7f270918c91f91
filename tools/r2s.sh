export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/san
for tool in memcheck synccheck racecheck; do
for c in batch1_redo decide_lookback pressure fused_tail sampler_quant; do
timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize.py $c > gpurun_out/san/${tool}_$c.log 2>&1
echo "$tool $c rc=$?" | tee -a gpurun_out/san/summary.txt
done; done
