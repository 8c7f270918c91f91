"""One INT8 and one INT4 quantize + dequantize of the bench's frozen tier (3.53M rows of 128 bf16), for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_11221_b200 import asr_kv_dequantize, asr_kv_quantize  # noqa: E402

rows, n = 6900 * 512, 128
kv = torch.randn((rows, n), device="cuda").to(torch.bfloat16)
back = torch.empty_like(kv)
scales = torch.empty(rows, dtype=torch.float32, device="cuda")
for bits in (8, 4):
    codes = torch.empty((rows, n if bits == 8 else n // 2), dtype=torch.int8, device="cuda")
    asr_kv_quantize(kv, codes, scales, bits=bits)
    asr_kv_dequantize(codes, scales, back, bits=bits)
torch.cuda.synchronize()
print("quant probe ok")
