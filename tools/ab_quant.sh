# A/B of the NEXT-4 quantize kernel across libasr builds (ASR_LIB_PATH); run under gpurun from the repo root.
for v in libasr.so libasr_rg1.so libasr_rg4.so; do
  ASR_LIB_PATH=$PWD/paper_2512_11221_b200/$v timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench, json
d=bench.quant_point(0)
print('$v', json.dumps({b:{k:d[b][k] for k in ('quantize_us','quantize_frac','dequantize_us')} for b in ('int8','int4')}))
" 2>&1 | tail -1
done
