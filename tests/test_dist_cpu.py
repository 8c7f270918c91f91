"""Host logic of the sequence-sharded multi-GPU mode, on CPU with the gloo backend (world size 2).

The GPU hot path has no collective; what N>1 adds is the partition of the batch and the
max/sum-over-ranks reduction of timings and token counts — tested here with real processes.
The per-sequence independence that makes sharding exact is pinned on the oracle: running a batch
split across two "ranks" gives bitwise the same ledgers and outputs as running it whole.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2512_11221_b200.dist import shard


def test_shard_partition_properties():
    for total in range(0, 40):
        for world in range(1, 9):
            parts = [shard(total, r, world) for r in range(world)]
            covered = []
            for first, cnt in parts:
                covered.extend(range(first, first + cnt))
            assert covered == list(range(total))
            counts = [c for _, c in parts]
            assert max(counts) - min(counts) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_11221_b200.dist import max_over_ranks, sum_over_ranks
    # each rank "times" its shard: rank-dependent times; the job time is the max, tokens the sum
    first, cnt = shard(7, rank, world)
    t = 1.0 + rank * 0.5
    q.put((rank, max_over_ranks(t), sum_over_ranks(cnt), first, cnt))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_reductions():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [1.5, 1.5]          # max over ranks
    assert [r[2] for r in res] == [7.0, 7.0]          # every sequence counted once
    assert [(r[3], r[4]) for r in res] == [(0, 4), (4, 3)]


def _id_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2512_11221_b200.dist import head_shard, share_nccl_id
    uid = share_nccl_id(lambda: bytes(range(128)))
    q.put((rank, uid, head_shard(32, 8, rank, world)))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_head_shard_setup():
    # every rank receives rank 0's NCCL id; the KV heads (and their GQA query heads) are partitioned
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] == bytes(range(128)) for r in res)
    assert [r[2] for r in res] == [(0, 16, 0, 4), (16, 32, 4, 8)]


def test_head_shard_partition():
    from paper_2512_11221_b200.dist import head_shard
    for world in (1, 2, 4, 8):
        kv, qh = [], []
        for r in range(world):
            q0, q1, k0, k1 = head_shard(32, 8, r, world)
            kv.extend(range(k0, k1))
            qh.extend(range(q0, q1))
            assert all(h // 4 in range(k0, k1) for h in range(q0, q1))   # GQA groups stay whole
        assert kv == list(range(8)) and qh == list(range(32))
    with pytest.raises(ValueError):
        head_shard(32, 8, 0, 3)


def test_sharded_batch_equals_whole_batch_on_oracle():
    import gen
    import oracle
    p = gen.GenParams(seed=77, L=1, Hq=4, Hkv=2, d=16, hot_permille=300)
    cfg = oracle.OrcCfg(L=1, Hq=4, Hkv=2, d=16, window=4)
    B, P, steps = 5, 8, 30
    cap = P + steps + 1
    KV = [gen.kv(p, b, 0, cap) for b in range(B)]

    def run(seqs):
        out = {}
        for b in seqs:
            s = oracle.OracleSeq(cfg, cap, P)
            trace = []
            for i in range(steps):
                O, act, sc, st = s.step(gen.q(p, b, i), KV[b][0], KV[b][1])
                trace.append((O.copy(), act.copy(), st["active_post"]))
            out[b] = trace
        return out

    whole = run(range(B))
    split = {}
    for rank in range(2):
        first, cnt = shard(B, rank, 2)
        split.update(run(range(first, first + cnt)))
    for b in range(B):
        for (o1, a1, n1), (o2, a2, n2) in zip(whole[b], split[b]):
            np.testing.assert_array_equal(o1, o2)
            np.testing.assert_array_equal(a1, a2)
            assert n1 == n2


def test_bench_gpus_n_spawns_ranks_and_checks_world():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks (torch.distributed.run on
    127.0.0.1); rank 0 alone prints the line.  Exercised on CPU through the reference arm (the
    oracle), which needs no GPU; a WORLD_SIZE that contradicts --gpus is refused."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    args = [sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
            "--warmup", "0", "--context", "560", "--window", "512"]
    r = subprocess.run(args, capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["cpu_baseline"]["cores"] >= 1
    env["WORLD_SIZE"] = "1"
    r = subprocess.run(args, capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stdout
