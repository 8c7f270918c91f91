"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle, element by element.

Sizes are chosen so the oracle finishes in seconds yet the work spans several tiles, several
split-KV chunks and ragged tails; edge cases cover ragged prompts (including an empty one),
GQA, fp32 KV, tau <= 0 (full attention), K >= n, the R1 tick, pinned prefixes, explicit
restores, planted entropy spikes (SR -> WR -> FR -> RR) and host-memory I/O.
"""
import numpy as np
import pytest

import gen
from harness import Case, run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(1001, 1017))
def test_tiny_w0(seed):
    # BASELINE.json configs[0]: 1 layer, 2 heads, d=16, K=16, 32 steps, batch 1 (SURVEY A.3 sequence)
    s = run(Case(seed=seed))
    if seed == 1001:
        want = [33, 34, 35, 36, 37, 38, 39, 40, 41, 42, 43, 44, 45, 46, 47, 31, 48, 32, 49, 33, 50, 34, 51, 35, 52,
                36, 53, 37, 54, 38, 55, 39]
        assert s["final"][0]["active"] == want[-1]


@pytest.mark.parametrize("seed", [1001, 1002, 1003])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_tiny_w1_and_gqa(seed, dtype):
    run(Case(seed=seed, hot_permille=300, dtype=dtype))
    run(Case(seed=seed, Hq=2, Hkv=1, hot_permille=300, a_hot=64, dtype=dtype))


def test_ragged_multitile_batch():
    # several 32-token tiles and split chunks per (b, l), ragged |A_b|, peaked attention (a_hot=64)
    c = Case(L=2, Hq=8, Hkv=2, d=64, B=3, prompt=(1, 150, 67), steps=120, window=8, hot_permille=300,
             a_hot=64, seed=77)
    s = run(c)
    assert s["frozen"] > 0 and s["restored"] > 0


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_llama_head_layout_moderate_context(dtype):
    # LLaMA-3-8B head layout (Hq=32, Hkv=8, d=128) on 2 layers, 600+ tokens, chunks > 1
    c = Case(L=2, Hq=32, Hkv=8, d=128, B=2, prompt=(600, 333), steps=12, window=64, hot_permille=300,
             a_hot=64, seed=2001, dtype=dtype)
    run(c)


def test_empty_prompt_and_tiny_window():
    run(Case(B=2, prompt=(0, 5), steps=40, window=1, seed=5))


def test_tau_nonpositive_is_full_attention_gauss():
    # GAUSS family: realistic logits std ~1.3, tau = 0 -> nothing frozen; O vs fp64 full attention
    for dtype in ("bf16", "f32"):
        s = run(Case(L=2, Hq=8, Hkv=2, d=128, B=2, prompt=(300, 200), steps=6, window=4, tau=0.0,
                     family=gen.GAUSS, seed=9, dtype=dtype))
        assert s["frozen"] == 0


def test_window_covers_context():
    s = run(Case(prompt=(10,), steps=20, window=64, seed=3))
    assert s["frozen"] == 0


def test_r1_tick_pinned_prefix_scaled_score():
    run(Case(prompt=(40,), steps=60, window=8, tick_order=1, seed=21))
    run(Case(prompt=(40,), steps=60, window=8, pinned_prefix=5, seed=22))
    # scaled mode: s/sqrt(16) with tau 0.05 keeps the guard band (cold <= 7/64 ... 0.109; hot >= 0.328)
    run(Case(prompt=(40,), steps=40, window=8, score_mode=1, tau=0.2, hot_permille=300, seed=23))


def test_explicit_restores():
    c = Case(prompt=(40, 23), steps=80, window=4, seed=31, B=2,
             restore_at={30: (-1, 1), 45: (1, 2), 60: (0, 3)})
    s = run(c)
    assert s["restored"] > 0


def test_entropy_spikes_ladder():
    c = Case(L=1, Hq=4, Hkv=2, d=32, B=2, prompt=(20, 33), steps=140, window=8, vocab=128256, seed=41,
             spike_first=60, spike_period=16, spike_count=4)
    run(c)


def test_host_memory_io():
    run(Case(L=2, Hq=8, Hkv=2, d=64, B=2, prompt=(50, 64), steps=30, window=8, hot_permille=300,
             vocab=3000, host_io=True, seed=51))


# ------------------------------------------------------------------ (a5) pressure mode: real offload
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_pressure_mode_tiny(dtype):
    # evict every freeze (evict_min=1): frozen tokens leave the device and are prefetched back one step
    # before they return (early on the sublinear schedule gives 1-2 step absences, so the pool still
    # needs ~n slots here); results identical to the oracle, bytes restored exactly
    s = run(Case(prompt=(32,), steps=64, window=8, seed=61, dtype=dtype, pool_tokens=100, evict_min=1, evict_policy=1))
    assert s["evicted"] > 0 and s["prefetched"] > 0


def test_pressure_mode_llama_heads_and_recovery():
    # MMA attention path with slot indirection; planted entropy spikes force demand copies (SR/WR/FR)
    c = Case(L=2, Hq=32, Hkv=8, d=128, B=2, prompt=(40, 25), steps=110, window=8, vocab=128256, seed=71,
             spike_first=50, spike_period=16, spike_count=4, pool_tokens=300, hot_permille=300, a_hot=64,
             evict_policy=1)
    s = run(c)
    assert s["evicted"] > 0 and s["prefetched"] > 0 and s["demand"] > 0


def test_pressure_mode_explicit_restore_and_evict_threshold():
    s = run(Case(B=2, prompt=(30, 12), steps=70, window=4, seed=81, pool_tokens=200, evict_min=1, evict_policy=1,
                 restore_at={40: (-1, 3), 55: (0, 1)}))
    assert s["evicted"] > 0 and s["demand"] > 0


@pytest.mark.parametrize("hq,hkv", [(28, 4), (16, 2), (8, 1), (16, 4), (32, 8)])
def test_mma_path_gqa_layouts(hq, hkv):
    # the tensor-core attention kernel covers 1/2/4/8 KV heads and up to 8 (4 for 8 KV heads) query
    # heads per KV head: Qwen2-7B-like (28 q / 4 KV), head shards of LLaMA-3-8B (16/4, 8/2 ...), G = 8
    run(Case(L=2, Hq=hq, Hkv=hkv, d=128, B=2, prompt=(90, 37), steps=20, window=16, hot_permille=300, a_hot=64,
             seed=3000 + hq + hkv, vocab=2048))


@pytest.mark.parametrize("logits_dtype", ["bf16", "f32"])
def test_batch1_phase_a_inside_attention_with_recovery(logits_dtype):
    # batch 1 on the tensor-core path runs phase A/B on an extra warp of the attention kernel while
    # the attention already streams A_i as the previous step compacted it; planted entropy spikes make
    # recovery recompact A_i mid-kernel, which forces the in-kernel second pass (grid barrier + redo);
    # explicit restores between steps recompact the precomputed A_i in place
    c = Case(L=2, Hq=32, Hkv=8, d=128, B=1, prompt=(60,), steps=150, window=8, vocab=128256, seed=91,
             spike_first=50, spike_period=16, spike_count=4, hot_permille=300, a_hot=64,
             restore_at={30: (0, 1), 120: (0, 3)}, logits_dtype=logits_dtype)
    s = run(c)
    assert s["restored"] > 0 and s["recoveries"] >= 3   # SR, WR, FR fired (each forced a redo pass)


def test_large_batch_grouped_phase_a_units():
    # batch > 1 on the tensor-core path with phase A as its own kernel (units grouped per warp / layer
    # range) and the combine as a separate kernel (batch * L * Hq > 64 warps per SM)
    run(Case(L=4, Hq=32, Hkv=8, d=128, B=80, prompt=tuple(20 + (7 * b) % 50 for b in range(80)), steps=12,
             window=8, vocab=1024, seed=93, hot_permille=300, a_hot=64))


@pytest.mark.parametrize("W", [8, 64, 100, 128])
def test_finite_history_window(W):
    # NEXT-3: Eq. 3's count c_j over the last W steps only — a per-token 128-bit detection
    # history on the device; ledgers (counts within the window), lists and O bitwise against the
    # oracle's detection log.  W < run length makes counts fall back and durations shrink.
    s = run(Case(prompt=(40,), steps=160, window=8, seed=300 + W, history_window=W))
    assert s["frozen"] > 0
    run(Case(L=2, Hq=32, Hkv=8, d=128, B=1, prompt=(60,), steps=90, window=8, hot_permille=300, a_hot=64,
             vocab=4096, seed=400 + W, history_window=W))


def test_time_attention_leaves_no_trace():
    # bench.py times the attention kernel alone between steps (asr_time_attention); the steps after it
    # must stay bitwise on the oracle (batch 1: phase A/B inside the attention kernel; batch 3: not)
    run(Case(L=2, Hq=32, Hkv=8, d=128, B=1, prompt=(70,), steps=30, window=8, hot_permille=300, a_hot=64,
             vocab=4096, seed=501, time_attention_at=(5, 6, 17)))
    run(Case(L=2, Hq=32, Hkv=8, d=128, B=3, prompt=(70, 20, 45), steps=30, window=8, hot_permille=300,
             a_hot=64, vocab=4096, seed=502, time_attention_at=(5, 17)))


@pytest.mark.parametrize("B", [1, 2])
def test_fr_clear_counts(B):
    # NEXT-3 option: FR also clears the detection counts (oracle pinned in test_oracle_variants.py);
    # planted spikes drive the ladder through SR, WR, FR, RR; counts compared bitwise every step
    c = Case(L=2, Hq=32, Hkv=8, d=128, B=B, prompt=(60, 41)[:B], steps=150, window=8, vocab=128256, seed=95,
             spike_first=50, spike_period=16, spike_count=4, fr_clear_counts=1)
    s = run(c)
    assert s["recoveries"] >= 3 * B


@pytest.fixture
def sk_balance(monkeypatch):
    monkeypatch.setenv("ASR_SK_BALANCE", "1")   # read at asr_create (default: batch 1 only)


@pytest.mark.parametrize("B", [1, 2])
def test_rate_balanced_split(sk_balance, B):
    # the rate-balanced cut of the attention's static split (asr_internal.h, sk_weighted) engages at
    # T >= 8 x grid tiles once step i - 4's rates exist: 32 layers over ~1000 attended tokens, 14
    # steps; ledgers bitwise, O within the bf16 bar at every step (only the combine's order moves)
    import torch
    s = run(Case(L=32, Hq=32, Hkv=8, d=128, B=B, prompt=(2000, 1900)[:B], steps=14, window=16, hot_permille=500,
                 a_hot=64, vocab=4096, seed=720 + B))
    grid = torch.cuda.get_device_properties(0).multi_processor_count   # the attention's persistent grid
    assert min(s["tiles"][4:]) >= 8 * grid, s["tiles"]


@pytest.fixture
def fused_tail(monkeypatch):
    monkeypatch.setenv("ASR_FUSE_TAIL", "1")   # read at asr_create


@pytest.mark.parametrize("B", [1, 3])
def test_fused_tail_mode(fused_tail, B):
    # opt-in one-kernel step (DevState::fuse_tail): decide + tick + A_{i+1} (segment look-back) +
    # combine inside the attention kernel after a grid barrier; bitwise the same ledgers and lists
    run(Case(L=2, Hq=32, Hkv=8, d=128, B=B, prompt=(300, 129, 77)[:B], steps=40, window=16, hot_permille=300,
             a_hot=64, vocab=4096, seed=700 + B))
    # finite W, planted entropy spikes (recovery recompacts A_i mid-kernel at batch 1: redo pass)
    run(Case(L=2, Hq=32, Hkv=8, d=128, B=B, prompt=(60, 41, 33)[:B], steps=150, window=8, vocab=128256,
             seed=710 + B, spike_first=50, spike_period=16, spike_count=4, history_window=64))


# ------------------------------------------------------------------ (a5) capacity-driven Belady eviction
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_pressure_belady_tight_pool(dtype):
    # a pool smaller than the context: nothing is evicted until the free stack runs short; then the
    # resident frozen tokens returning last go first.  All-cold prompt of 64 + 200 steps, K = 8:
    # 264 tokens on a 220-slot pool (the trace needs >= 207 at once: A_{i+1} + the tokens returning
    # at step i+1's tick + the spare; a smaller pool is infeasible for any policy).  Results bitwise
    # the oracle's; bytes restored exactly.
    s = run(Case(prompt=(64,), steps=200, window=8, seed=62, dtype=dtype, pool_tokens=220))
    assert s["evicted"] > 0 and s["prefetched"] > 0


def test_pressure_belady_llama_batch_with_recovery():
    # MMA path, 2 sequences (410 tokens) sharing one 390-slot pool (the all-cold lockstep cohorts need
    # up to 360 slots at once near the end), a planted spike (SR); the per-step cut keeps the free
    # stack above the next step's appends + prefetches + pool_reserve
    c = Case(L=2, Hq=32, Hkv=8, d=128, B=2, prompt=(80, 50), steps=140, window=8, vocab=128256, seed=72,
             spike_first=60, spike_period=16, spike_count=1, pool_tokens=390, pool_reserve=24)
    s = run(c)
    assert s["evicted"] > 0 and s["prefetched"] > 0


@pytest.mark.parametrize("B", [1, 2])
def test_entropy_given_by_the_sampler(B):
    # NEXT-1 fused with the entropy stage: asr_sample_entropy draws the next token and takes H in the
    # same read of each row; the step consumes H (ASR_ENTROPY_GIVEN) instead of re-reading the row.
    # Planted spikes drive the ladder; ledgers, lists and H bitwise / within 1e-4 of the oracle.
    c = Case(L=2, Hq=32, Hkv=8, d=128, B=B, prompt=(60, 41)[:B], steps=120, window=8, vocab=128256, seed=97,
             spike_first=50, spike_period=16, spike_count=3, entropy_given=True)
    s = run(c)
    assert s["recoveries"] >= 3 * B


@pytest.mark.parametrize("policy", [0, 1])
def test_pressure_int8_frozen_tier(policy):
    # NEXT-4 wired into the host link: the mirror holds R-quant INT8 rows; restored tokens come back
    # dequantised.  Decisions, lists and scores bitwise, O within the bf16 bar, against the oracle fed
    # the dequantised rows for exactly the tokens the device holds dequantised; the mirror's bytes equal
    # oracle/quant.py's codes and scales, the device slots the appended or dequantised rows.
    c = Case(L=2, Hq=32, Hkv=8, d=128, B=2, prompt=(70, 40), steps=120, window=8, vocab=4096, seed=99,
             hot_permille=300, a_hot=64, spike_first=60, spike_period=16, spike_count=1, mirror_bits=8,
             evict_policy=policy, evict_min=1 if policy else 2, pool_tokens=340 if policy else 330, pool_reserve=48)
    s = run(c)
    assert s["evicted"] > 0 and s["prefetched"] > 0


@pytest.mark.parametrize("shape", [(3, 8, 2, 64), (2, 32, 8, 128)])
def test_per_layer_ledgers(shape):
    # NEXT-3: one ledger per (sequence, layer) — layer l freezes on s_j^(l) = (1/Hq) sum_h |q.k| of its
    # own heads and attends its own list.  Oracle: one single-layer OracleSeq per (b, l) fed that
    # layer's q / K / V and the sequence's logits; ledgers, lists, scores bitwise, O within 2e-3, every
    # step, generic (d = 64) and tensor-core (LLaMA layout) attention; planted spikes drive recovery
    import torch
    from harness import o_rel_err
    from paper_2512_11221_b200 import Config, Context
    import oracle
    L, Hq, Hkv, d = shape
    B, P, steps, K, V = 2, (50, 31), 90, 8, 4096
    p = gen.GenParams(seed=321 + d, L=L, Hq=Hq, Hkv=Hkv, d=d, hot_permille=300, a_hot=64, vocab=V,
                      spike_first=40, spike_period=16, spike_count=2)
    cap = max(P) + steps + 1
    # tau between the LAT cold scores: per-layer scores are multiples of u = 2^-8 / Hq (exact in fp32), so
    # tau at a half-lattice point decides identically in fp32 and fp64, and cold tokens score above or
    # below it depending on the layer's q — the layers' ledgers diverge
    u = 2.0 ** -8 / Hq
    tau = (np.floor(0.055 / u) + 0.5) * u   # near the median cold per-layer score
    KV = [gen.kv(p, b, 0, cap) for b in range(B)]
    pk = np.zeros((B, max(P), L, Hkv, d), np.uint16)
    pv = np.zeros_like(pk)
    for b in range(B):
        pk[b, :P[b]], pv[b, :P[b]] = KV[b][0][:P[b]], KV[b][1][:P[b]]
    to_t = lambda a: torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda()
    cfg = Config(n_layers=L, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, batch=B, max_context=cap, window=K, vocab=V,
                 tau=float(tau), per_layer_ledgers=1)
    ctx = Context(cfg, to_t(pk), to_t(pv), list(P))
    assert ctx.n_seq == B * L
    ocfg = oracle.OrcCfg(L=1, Hq=Hq, Hkv=Hkv, d=d, window=K, vocab=V, tau=float(tau))
    orc = [[oracle.OracleSeq(ocfg, cap, P[b]) for _ in range(L)] for b in range(B)]
    differ = False
    for i in range(steps):
        q = np.stack([gen.q(p, b, i) for b in range(B)])
        kn = np.stack([KV[b][0][P[b] + i] for b in range(B)])
        vn = np.stack([KV[b][1][P[b] + i] for b in range(B)])
        lg = np.stack([gen.logits(p, b, i - 1) for b in range(B)]) if i > 0 else None
        o = torch.zeros((B, L, Hq, d), dtype=torch.float32, device="cuda")
        ctx.step(to_t(q), to_t(kn), to_t(vn), o, logits_prev=None if lg is None else to_t(lg))
        O = o.cpu().numpy()
        for b in range(B):
            acts = []
            for l in range(L):
                Ob, act, scores, out = orc[b][l].step(q[b][l:l + 1], KV[b][0][:, l:l + 1], KV[b][1][:, l:l + 1],
                                                       None if lg is None else lg[b])
                g = ctx.stats(b * L + l, detail=True)
                where = f"step {i} seq {b} layer {l}"
                np.testing.assert_array_equal(g["active_list"], act, err_msg=where)
                assert np.array_equal(g["scores"], scores.astype(np.float32)), where
                led = orc[b][l].ledger()
                for key in ("residency", "timer", "count", "freeze_step"):
                    np.testing.assert_array_equal(g["ledger"][key], led[key], err_msg=f"{where} {key}")
                assert g["recovery_action"] == out["recovery_action"] and g["device_error"] == 0, where
                assert o_rel_err(O[b, l:l + 1], Ob) <= 2e-3, where
                acts.append(tuple(act))
            differ |= len(set(acts)) > 1
    assert differ   # the layers' ledgers do diverge (per-layer scores differ)
    ctx.close()
