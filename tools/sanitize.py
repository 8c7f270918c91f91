"""Small cases for compute-sanitizer (measurement tool, run under gpurun):

  compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize.py [case ...]

Each case drives the CUDA path through the C ABI on tiny shapes and checks it against the oracle
(tests/harness.py), covering: batch 1 with phase A/B inside the attention kernel and the grid-barrier
redo pass (planted entropy spikes), the multi-block decide with its tagged look-back, pressure mode
(Belady and at-freeze eviction: free-stack pushes / pops, prefetch and demand copies), the fused tail,
the sampler's thread-block clusters and the quantised tier kernels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def case_batch1_redo():
    from harness import Case, run
    run(Case(L=1, Hq=4, Hkv=1, d=128, B=1, prompt=(40,), steps=70, window=8, vocab=4096, seed=91,
             spike_first=20, spike_period=16, spike_count=3, hot_permille=300, a_hot=64, restore_at={30: (0, 1)}))


def case_decide_lookback():
    from harness import Case, run
    os.environ["ASR_DECIDE_POSITIONS"] = "128"   # several decide blocks per sequence (read at create)
    run(Case(L=1, Hq=4, Hkv=1, d=128, B=2, prompt=(600, 450), steps=12, window=8, seed=92))
    del os.environ["ASR_DECIDE_POSITIONS"]


def case_pressure():
    from harness import Case, run
    run(Case(prompt=(64,), steps=120, window=8, seed=62, pool_tokens=176, pool_reserve=2))   # needs <= 165 at once
    run(Case(B=2, prompt=(30, 12), steps=60, window=4, seed=81, pool_tokens=200, evict_min=1, evict_policy=1,
             restore_at={40: (-1, 3), 55: (0, 1)}))


def case_fused_tail():
    from harness import Case, run
    os.environ["ASR_FUSE_TAIL"] = "1"
    run(Case(L=1, Hq=4, Hkv=1, d=128, B=2, prompt=(90, 33), steps=20, window=8, vocab=4096, seed=93,
             spike_first=10, spike_period=16, spike_count=1, hot_permille=300, a_hot=64))
    del os.environ["ASR_FUSE_TAIL"]


def case_sampler_quant():
    import numpy as np
    import torch

    import gen
    from oracle import quant
    from oracle.sample import interval, sample
    from paper_2512_11221_b200 import asr_kv_dequantize, asr_kv_quantize, asr_sample
    g = gen.GenParams(seed=7, vocab=50000)
    for B, (T, k, P) in ((1, (0.8, 64, 0.9)), (3, (1.0, 0, 0.95)), (9, (0.0, 0, 1.0))):
        rows = np.stack([gen.logits(g, b, 3) for b in range(B)])
        toks = [sample(rows[b], T, k, P, 0.37) for b in range(B)]
        us = [0.5 * sum(interval(rows[b], T, k, P, toks[b])) for b in range(B)]
        xt = torch.from_numpy(rows.view(np.int16)).view(torch.bfloat16).cuda()
        out = torch.empty(B, dtype=torch.int32, device="cuda")
        asr_sample(xt, torch.tensor(us, dtype=torch.float32, device="cuda"), out, temperature=T, top_k=k, top_p=P)
        assert out.cpu().tolist() == toks
    k_, v_ = gen.kv(gen.GenParams(seed=9, L=1, Hq=8, Hkv=8, d=128), 0, 0, 5)
    rows = np.stack([k_, v_], axis=2).reshape(-1, 128)
    kv = torch.from_numpy(rows.view(np.int16)).cuda().view(torch.bfloat16)
    for bits in (8, 4):
        codes = torch.empty((rows.shape[0], 128 if bits == 8 else 64), dtype=torch.int8 if bits == 8 else torch.uint8,
                            device="cuda")
        scales = torch.empty(rows.shape[0], dtype=torch.float32, device="cuda")
        back = torch.empty_like(kv)
        asr_kv_quantize(kv, codes, scales, bits=bits)
        asr_kv_dequantize(codes, scales, back, bits=bits)
        oc, osc = quant.quantize(rows, bits)
        assert np.array_equal(scales.cpu().numpy(), osc)


CASES = {n[5:]: f for n, f in dict(globals()).items() if n.startswith("case_")}

if __name__ == "__main__":
    import torch
    torch.cuda.init()
    for name in (sys.argv[1:] or list(CASES)):
        CASES[name]()
        print("case", name, "ok", flush=True)
