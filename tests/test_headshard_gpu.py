"""Head-sharded mode (north_star "optional head-sharded mode whose per-token partial
score sums are all-reduced"): every shard holds a slice of the KV heads (and their query heads) of all
sequences; the per-token partial Eq. 2 sums are summed across shards between asr_step_attend and
asr_step_decide, after which every shard takes the same decisions as an unsharded context.

One GPU cannot host an NCCL communicator with two ranks, so the two-shard case is emulated with two
contexts on the same device whose partial-score buffers are summed with a device add (the math NCCL's
all-reduce performs); the NCCL path itself is exercised with a one-rank communicator.
"""
import numpy as np
import pytest

import gen
import oracle
from harness import o_rel_err

pytestmark = pytest.mark.gpu


class _CAI:   # wrap a raw device pointer for torch (CUDA array interface)
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3}


def _t(a):
    import torch
    return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda()


@pytest.mark.parametrize("shape", [(1, 4, 2, 16), (2, 32, 8, 128)])
def test_two_shards_match_unsharded_oracle(shape):
    import torch
    from paper_2512_11221_b200 import Config, Context
    L, Hq, Hkv, d = shape
    B, P, steps, K = 2, 40, 40, 8
    S = 2
    hq, hk = Hq // S, Hkv // S
    p = gen.GenParams(seed=91, L=L, Hq=Hq, Hkv=Hkv, d=d, hot_permille=300, a_hot=64, vocab=4096)
    cap = P + steps + 1
    KV = [gen.kv(p, b, 0, cap) for b in range(B)]
    pk = np.stack([KV[b][0][:P] for b in range(B)])
    pv = np.stack([KV[b][1][:P] for b in range(B)])
    shards = []
    for r in range(S):
        cfg = Config(n_layers=L, n_q_heads=hq, n_kv_heads=hk, head_dim=d, batch=B, max_context=cap, window=K,
                     vocab=4096, score_heads=Hq)
        shards.append(Context(cfg, _t(np.ascontiguousarray(pk[:, :, :, r * hk:(r + 1) * hk])),
                              _t(np.ascontiguousarray(pv[:, :, :, r * hk:(r + 1) * hk])), [P] * B))
    orc = [oracle.OracleSeq(oracle.OrcCfg(L=L, Hq=Hq, Hkv=Hkv, d=d, window=K, vocab=4096), cap, P) for _ in range(B)]
    for i in range(steps):
        q = np.stack([gen.q(p, b, i) for b in range(B)])
        kn = np.stack([KV[b][0][P + i] for b in range(B)])
        vn = np.stack([KV[b][1][P + i] for b in range(B)])
        lg = np.stack([gen.logits(p, b, i - 1) for b in range(B)]) if i > 0 else None
        outs = []
        for r, ctx in enumerate(shards):
            o = torch.zeros((B, L, hq, d), dtype=torch.float32, device="cuda")
            ctx.attend(_t(np.ascontiguousarray(q[:, :, r * hq:(r + 1) * hq])),
                       _t(np.ascontiguousarray(kn[:, :, r * hk:(r + 1) * hk])),
                       _t(np.ascontiguousarray(vn[:, :, r * hk:(r + 1) * hk])), o,
                       logits_prev=None if lg is None else _t(lg))
            outs.append(o)
        # the all-reduce: sum of the shards' per-token partials, written back to every shard
        bufs = [torch.as_tensor(_CAI(*ctx.score_partials()), device="cuda") for ctx in shards]
        total = bufs[0] + bufs[1]
        for x in bufs:
            x.copy_(total)
        for ctx in shards:
            ctx.decide()
        for b in range(B):
            O, act, scores, out = orc[b].step(q[b], KV[b][0], KV[b][1], None if lg is None else lg[b])
            led = orc[b].ledger()
            for r, ctx in enumerate(shards):
                g = ctx.stats(b, detail=True)
                np.testing.assert_array_equal(g["active_list"], act, err_msg=f"step {i} seq {b} shard {r}")
                for key in ("residency", "timer", "count", "freeze_step"):
                    np.testing.assert_array_equal(g["ledger"][key], led[key])
                assert np.array_equal(g["scores"], scores.astype(np.float32))
                assert g["recovery_action"] == out["recovery_action"]
                err = o_rel_err(outs[r][b].cpu().numpy(), O[:, r * hq:(r + 1) * hq])
                assert err <= 2e-3, (i, b, r, err)
    for ctx in shards:
        ctx.close()


def test_nccl_single_rank_step():
    import torch
    from harness import Case, run
    from paper_2512_11221_b200 import asr_nccl_unique_id
    uid = asr_nccl_unique_id()
    assert len(uid) == 128
    # a one-rank communicator: asr_step runs attend -> ncclAllReduce -> decide; parity with the oracle
    run(Case(L=2, Hq=8, Hkv=2, d=64, B=2, prompt=(30, 50), steps=30, window=8, hot_permille=300, seed=93,
             nccl_world1=True))


def test_nccl_allreduce_moves_exactly_the_attended_partials():
    # the head-sharded all-reduce is packed by a prefix over |A_b|: 4 bytes per attended token of the
    # batch (not the [B][max_context] buffer); a one-rank communicator, LLaMA head layout
    import torch
    from paper_2512_11221_b200 import Config, Context, asr_nccl_unique_id
    from paper_2512_11221_b200.dist import ledger_digest
    B, P, L, Hq, Hkv, d = 3, 90, 2, 32, 8, 128
    p = gen.GenParams(seed=95, L=L, Hq=Hq, Hkv=Hkv, d=d, hot_permille=300, a_hot=64)
    cap = P + 40
    KV = [gen.kv(p, b, 0, cap) for b in range(B)]
    pk = np.stack([KV[b][0][:P] for b in range(B)])
    pv = np.stack([KV[b][1][:P] for b in range(B)])
    cfg = Config(n_layers=L, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, batch=B, max_context=cap, window=8, vocab=0)
    ctx = Context(cfg, _t(pk), _t(pv), [P - 7 * b for b in range(B)])
    ctx.attach_nccl(asr_nccl_unique_id(), 1, 0)
    before = ctx.stats(0)["allreduce_bytes"]
    for i in range(30):
        q = np.stack([gen.q(p, b, i) for b in range(B)])
        kn = np.stack([KV[b][0][P - 7 * b + i] for b in range(B)])
        vn = np.stack([KV[b][1][P - 7 * b + i] for b in range(B)])
        o = torch.zeros((B, L, Hq, d), dtype=torch.float32, device="cuda")
        ctx.step(_t(q), _t(kn), _t(vn), o)
        sts = [ctx.stats(b) for b in range(B)]
        after = sts[0]["allreduce_bytes"]
        assert after - before == 4 * sum(s["attended"] for s in sts), (i, after - before)
        before = after
    assert len(ledger_digest(ctx, B)) == 64
    ctx.close()
