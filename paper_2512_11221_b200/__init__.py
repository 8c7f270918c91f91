"""B200-native ASR-KF-EGR per-decode-step KV-management hot path (arXiv 2512.11221).

The product is libasr.so (C ABI: include/asr.h, sm_100a kernels in csrc/); this package only
holds its ctypes binding.  See DESIGN.md.
"""
from .asr import (Config, Context, AsrError, asr_create, asr_step, asr_restore, asr_stats, asr_read_kv,  # noqa: F401
                  asr_sample, asr_sample_entropy, asr_kv_quantize, asr_kv_dequantize, asr_stage_times,
                  asr_set_profile, asr_flush, asr_destroy, asr_step_attend, asr_step_decide, asr_score_partials,
                  asr_nccl_unique_id, asr_attach_nccl, lib, KV_BF16, KV_F32, ENTROPY_GIVEN, EVICT_BELADY,
                  EVICT_AT_FREEZE, SR, WR, FR, STAGES)
