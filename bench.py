"""bench.py — decode throughput of the ASR-KF-EGR per-step KV-management hot path on B200.

Contract (driver): `python bench.py --gpus N --steps K --warmup W [--impl asr|reference]` prints ONE
JSON line on rank 0.  A "step" = one asr_step over the context's batch: append, entropy + detector
+ recovery, compaction, split-KV attention over the active set with the fused Eq. 2 score,
combine, decide + tick, and the host-mirror copy — every stage of SURVEY.md §8(a).

Workload (BASELINE.json configs[1], the headline): LLaMA-3-8B shape (32 layers, 32 q / 8 KV heads,
d=128, vocab 128256), bf16 KV, window K=512, tau=0.5, k=2, batch 1 per GPU, 8K context reached by
decoding from a 512-token prompt ("grown" state), synthetic LAT inputs (all-cold W0 by
default, --family w1 for the 30 % hot mix).  Metric: decode tokens/s (unit tok/s, whole job = all
ranks).  Further points (--points, each with its own roofline line): configs[2] (8K, batch 64),
32K at batch 1 (the north_star's context), configs[3] (32K prefill, batch 16, needle + entropy-
triggered recovery), the 30 % hot mix, tau = 0 (full KV), pressure mode (50 % device pool, Belady),
the next-token draw, policy replay and the quantised frozen tier.  --workload c4: configs[4]'s
per-GPU share (256 sequences at 32K over --gpus ranks, no host mirror).

Timing: W untimed warm-up steps, then K steps each bracketed by CUDA events on the launching stream
with a 256 MiB L2 flush between steps (outside the events); barrier + synchronize on both sides;
the max over ranks of the summed step times.  Multi-GPU: one process per GPU, each rank owns its own
batch (sequence sharding, no collective on the hot path) -> "scaling": "weak"; `--gpus N` without a
torchrun environment re-launches itself under torch.distributed.run with N ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L, HQ, HKV, D, VOCAB = 32, 32, 8, 128, 128256
TOKEN_KV_BYTES = L * 2 * HKV * D * 2          # one token, all layers, K+V bf16 = 128 KiB


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="asr", choices=["asr", "reference"])
    ap.add_argument("--context", type=int, default=8192)
    ap.add_argument("--batch", type=int, default=1, help="sequences per GPU")
    ap.add_argument("--window", type=int, default=512)
    ap.add_argument("--family", default="w0", choices=["w0", "w1"])
    ap.add_argument("--tau", type=float, default=0.5, help="tau; <= 0 freezes nothing (the full-KV baseline)")
    ap.add_argument("--history-window", type=int, default=0, help="W of Eq. 3's count (0 = lifetime, R-W)")
    ap.add_argument("--seed", type=int, default=2001)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="budget of the cpu_baseline sample")
    ap.add_argument("--nvtx", action="store_true", help="NVTX range 'timed' around the timed steps (for ncu)")
    ap.add_argument("--timeline", action="store_true", help="device timeline of 8 extra steps (ASR_TIMELINE)")
    ap.add_argument("--pool-frac", type=float, default=0.0,
                    help="pressure mode: device slots = pool_frac * batch * context (0 = full residency)")
    ap.add_argument("--evict-min", type=int, default=2, help="pressure mode: never evict tokens returning sooner")
    ap.add_argument("--evict-policy", type=int, default=0, help="pressure mode: 0 Belady under pressure, 1 at freeze")
    ap.add_argument("--mirror-bits", type=int, default=0, help="pressure mode: 0 bf16 host mirror, 8 INT8 frozen tier")
    ap.add_argument("--points", default=parse_default_points(),
                    help="comma list of extra workloads (POINTS, or 'sample': the next-token draw) or '' for none")
    ap.add_argument("--workload", default="c1", choices=["c1", "c3", "c4"],
                    help="c1: grown state (configs[1]/[2] and the context points); c3: configs[3] (32K prefill, "
                         "needle + entropy spikes); c4: configs[4]'s per-rank share (256/N sequences at 32K)")
    ap.add_argument("--no-mirror", action="store_true", help="full residency without the pinned host mirror")
    ap.add_argument("--head-shard", action="store_true",
                    help="N>1: split the KV heads across ranks (NCCL score all-reduce) instead of the sequences")
    return ap.parse_args()


C3_Q = 55         # configs[3]: first step at which the prefill cohort (and the needle) is frozen with timer
                  # >= 2 (d = 3 from c = 36; tests/test_needle_gpu.py finds it with the oracle
                  # and asserts 55)
C3_NEEDLE = 16384


def gen_params(a, rank: int):
    import gen
    g = gen.GenParams(seed=a.seed + 7919 * rank, family=gen.LAT, L=L, Hq=HQ, Hkv=HKV, d=D,
                      hot_permille=300 if a.family == "w1" else 0, a_hot=4, vocab=VOCAB)
    if a.workload == "c3":   # needle in every sequence, retrieval queries after q, spikes -> SR at q+1, WR at q+17
        g.needle_pos, g.needle_b = C3_NEEDLE, -1
        g.query_first, g.query_count = C3_Q + 1, 8
        g.spike_first, g.spike_period, g.spike_count = C3_Q, 16, 2
    return g


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (the profiling recipe's clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.p = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(dev), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------ oracle arm

def _oracle_worker(wid: int, layers: int, context: int, window: int, family: str, seed: int, seconds: float,
                   steps, warmup: int, q) -> None:
    """One host core: the fp64 oracle (as it stands) on `layers` of the 32 layers of the workload's
    sequence, warm ledger from the oracle's own policy replay (untimed, the grown state), then full
    oracle steps (Alg. 1 lines 1-15 over the explicit A_i) timed one by one."""
    import numpy as np

    import gen
    import oracle
    g = gen.GenParams(seed=seed, family=gen.LAT, L=layers, Hq=HQ, Hkv=HKV, d=D,
                      hot_permille=300 if family == "w1" else 0, a_hot=4, vocab=VOCAB)
    P = window
    grow = context - P - 1
    total_steps = (steps if steps is not None else 100_000) + warmup
    cap = context + total_steps + 1
    cfg = oracle.OrcCfg(L=layers, Hq=HQ, Hkv=HKV, d=D, window=window, tau=0.5, softness=2.0, vocab=VOCAB)
    K, V = gen.kv(g, 0, 0, cap)
    s = oracle.OracleSeq(cfg, cap, P)
    below = np.ones(cap, np.uint8)
    if family == "w1":
        for j in range(cap):
            below[j] = 0 if gen.is_hot(g, 0, j) else 1
    for _ in range(grow):
        s.step_policy(below)
    done, t_total, i = 0, 0.0, grow
    while True:
        qv = gen.q(g, 0, i)
        lg = gen.logits(g, 0, i - 1)
        t0 = time.perf_counter()
        s.step(qv, K, V, lg)
        dt = time.perf_counter() - t0
        i += 1
        if warmup > 0:
            warmup -= 1
            continue
        done += 1
        t_total += dt
        if steps is not None and done >= steps:
            break
        if steps is None and t_total >= seconds:
            break
    q.put((wid, layers, done, t_total))


def oracle_sample(a, seconds_budget: float, steps: int | None = None, warmup: int = 0):
    """Time the fp64 oracle (as it stands) on the box's host cores over the same workload: the 32
    layers of one decode step are split over min(32, cores) processes (one C oracle each, running
    concurrently); a step is done when every process has done its layers, so tokens/s =
    min over processes of steps/s.  Layer subsets decide identically (LAT classes hold per head:
    DESIGN.md §4), so every process replays the same ledger."""
    import multiprocessing as mp
    cores = max(1, min(L, os.cpu_count() or 1))
    per = [L // cores + (1 if r < L % cores else 0) for r in range(cores)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_oracle_worker, args=(w, per[w], a.context, a.window, a.family, a.seed,
                                                      seconds_budget, steps, warmup, q)) for w in range(cores)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=3600) for _ in procs]
    for pr in procs:
        pr.join()
    rate = min(done / t for _, _, done, t in res)             # full steps (tokens) per second
    done = min(d for _, _, d, _ in res)
    return {"value": rate, "steps": done, "seconds": done / rate, "cores": cores,
            "sample": f"1 sequence x {done} decode steps at n~{a.context}, all {L} layers split over {cores} "
                      f"host processes (one fp64 C oracle each, concurrent), policy-replay warm ledger"}


def run_reference(a, rank: int, world: int):
    if rank != 0:
        return
    r = oracle_sample(a, 0, steps=a.steps, warmup=a.warmup)
    ms = 1000.0 / r["value"]
    line = {"impl": "reference", "metric": "decode tokens/sec at LLaMA-3-8B shape vs context; achieved HBM GB/s vs 8 TB/s",
            "value": r["value"], "unit": "tok/s", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"llama3-8b-shape ctx{a.context} batch1 window{a.window} {a.family}",
                       "context": a.context, "batch_per_gpu": 1, "window": a.window, "family": a.family},
            "cpu_baseline": {"value": r["value"], "unit": "tok/s", "cores": r["cores"], "kind": "oracle",
                             "sample": r["sample"]},
            "e2e": {"value": r["value"], "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------ GPU arm

def run_asr(a, rank: int, world: int, local_rank: int):
    import numpy as np
    import torch
    import torch.distributed as dist

    import gen
    from paper_2512_11221_b200 import Config, Context, KV_BF16, STAGES

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # head-sharded mode: this rank holds hkv_r of the KV heads (and their query heads) of every sequence
    # and the per-token partial scores are all-reduced over NCCL inside asr_step
    hq_r, hkv_r = (HQ // world, HKV // world) if a.head_shard else (HQ, HKV)
    if a.timeline:
        os.environ["ASR_TIMELINE"] = "1"
    B = a.batch
    W, K = a.warmup, a.steps
    if a.workload == "c3":
        # configs[3]: a 32K prompt (prefill: every token Active, R-prefill), decoded until the needle's
        # cohort is frozen (step C3_Q); the timed steps cover the spike-triggered SR at C3_Q + 1 and the
        # retrieval queries, the profiled pass the WR at C3_Q + 17
        P = a.context - 256
        grow = max(0, C3_Q - 3 - W)
    else:
        P = a.window                             # grown state: decoded from a window-sized prompt
        grow = a.context - P - 1                 # steps before the measured region starts
    e2e_steps = 0 if a.no_e2e else K
    max_ctx = P + grow + W + 2 * K + e2e_steps + 16
    g = gen_params(a, 0 if a.head_shard else rank)
    g.Hq, g.Hkv = hq_r, hkv_r
    pool = int(a.pool_frac * B * a.context) + 4 * B if a.pool_frac > 0 else 0
    cfg = Config(n_layers=L, n_q_heads=hq_r, n_kv_heads=hkv_r, head_dim=D, batch=B, max_context=max_ctx,
                 kv_dtype=KV_BF16, window=a.window, tau=a.tau, softness=2.0, vocab=VOCAB, profile_stages=0,
                 device=local_rank, pool_tokens=pool, evict_min_absence=a.evict_min, history_window=a.history_window,
                 evict_policy=a.evict_policy, host_mirror=0 if (a.no_mirror and a.pool_frac == 0) else 1,
                 mirror_bits=a.mirror_bits if pool else 0,
                 score_heads=HQ if a.head_shard else 0)
    need = B * max_ctx * TOKEN_KV_BYTES * (2 if a.workload == "c3" else 1) * 1.03 + (2 << 30)
    free_b, _ = torch.cuda.mem_get_info(dev)
    if need > free_b:
        return {"unavailable": f"{a.workload} batch {B} at {a.context} tokens needs {need / 2**30:.0f} GiB of HBM, "
                               f"{free_b / 2**30:.0f} GiB free on this GPU (run with more ranks)"}
    bf = torch.bfloat16
    pk = torch.empty((B, P, L, hkv_r, D), dtype=bf, device=dev)
    pv = torch.empty_like(pk)
    gen.dev_kv(g, B, 0, P, pk, pv)
    torch.cuda.synchronize()
    ctx = Context(cfg, pk, pv, [P] * B)
    if a.head_shard:
        from paper_2512_11221_b200 import asr_nccl_unique_id
        from paper_2512_11221_b200.dist import share_nccl_id
        uid = share_nccl_id(asr_nccl_unique_id) if world > 1 else asr_nccl_unique_id()
        # NCCL prints its version banner on stdout at init; keep stdout for the one JSON line
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            ctx.attach_nccl(uid, world, rank)
        finally:
            os.dup2(saved, 1)
            os.close(saved)
    del pk, pv
    q = torch.empty((B, L, hq_r, D), dtype=bf, device=dev)
    kn = torch.empty((B, L, hkv_r, D), dtype=bf, device=dev)
    vn = torch.empty_like(kn)
    lg = torch.empty((B, VOCAB), dtype=bf, device=dev)
    o = torch.empty((B, L, hq_r, D), dtype=torch.float32, device=dev)
    ent = torch.empty((B,), dtype=torch.float32, device=dev)
    pos_dev = torch.full((B,), P, dtype=torch.int32, device=dev)

    def inputs(i, qb, kb, vb, lb):
        gen.dev_q(g, B, i, qb)
        gen.dev_kv(g, B, 0, 1, kb, vb, pos0_dev=pos_dev + i)
        gen.dev_logits(g, B, i - 1, lb)

    clocks = Clocks(local_rank)   # samples from the growth phase (seconds of load) through the timed region
    t_grow = time.perf_counter()
    for i in range(grow):
        inputs(i, q, kn, vn, lg)
        ctx.step(q, kn, vn, o, logits_prev=lg if i > 0 else None, entropy=ent)
    torch.cuda.synchronize()
    t_grow = time.perf_counter() - t_grow
    # inputs of the measured steps (warm-up, timed, profiled), resident in HBM before timing
    n_meas = W + 2 * K
    Q = torch.empty((n_meas, B, L, hq_r, D), dtype=bf, device=dev)
    KN = torch.empty((n_meas, B, L, hkv_r, D), dtype=bf, device=dev)
    VN = torch.empty_like(KN)
    LG = torch.empty((n_meas, B, VOCAB), dtype=bf, device=dev)
    for t in range(n_meas):
        inputs(grow + t, Q[t], KN[t], VN[t], LG[t])
    # L2 flush between timed steps (outside the events): write a 256 MiB buffer (> 126 MB L2), then
    # read another 256 MiB buffer so the flush's dirty lines are written back before the step starts
    flush_w = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush_r = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush_acc = torch.empty((), dtype=torch.float32, device=dev)

    no_flush = os.environ.get("ASR_BENCH_NO_FLUSH") == "1"   # diagnostics only (never a bench value)

    class _Flush:
        @staticmethod
        def zero_():
            if no_flush:
                return
            flush_w.zero_()
            torch.sum(flush_r, dim=0, out=flush_acc)
    flush = _Flush()
    st = torch.cuda.current_stream()
    for t in range(W):
        flush.zero_()
        ctx.step(Q[t], KN[t], VN[t], o, logits_prev=LG[t], entropy=ent)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    io0 = ctx.stats(0)
    ctx.stage_times()   # resets the library's launch counter (synchronises; outside the timed region)
    if a.nvtx:
        torch.cuda.nvtx.range_push("timed")
    t_wall = time.perf_counter()
    for t in range(K):
        flush.zero_()
        ev[t][0].record(st)
        ctx.step(Q[W + t], KN[W + t], VN[W + t], o, logits_prev=LG[W + t], entropy=ent)
        ev[t][1].record(st)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    if a.nvtx:
        torch.cuda.nvtx.range_pop()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    total_ms = sum(step_ms)
    stats = [ctx.stats(b) for b in range(B)]
    rank_identical = None
    if a.head_shard:   # every shard must have taken bitwise the same decisions: all-gathered digests
        from paper_2512_11221_b200.dist import ledger_digest, ranks_agree
        rank_identical = ranks_agree(ledger_digest(ctx, B))
    allreduce_bytes_step = (stats[0]["allreduce_bytes"] - io0["allreduce_bytes"]) / K
    h2d_timed = stats[0]["bytes_h2d"] - io0["bytes_h2d"]    # context-wide counters
    d2h_timed = stats[0]["bytes_d2h"] - io0["bytes_d2h"]
    _, launches_timed = ctx.stage_times()   # library kernels launched in the timed region
    # ---- the same K-step workload again with stage events (graph event nodes between the kernels, no
    #      programmatic overlap): per-stage device times and the attention kernel's duration (roofline)
    ctx.set_profile(True)
    ctx.stage_times()
    recov = []      # configs[3]: recovery actions seen (the spike-triggered ladder), per profiled step
    att_steps = []  # sum over sequences of |A_i| of every profiled step (stage times are device events:
                    # the host reads between steps do not enter them)
    for t in range(K):
        flush.zero_()
        ctx.step(Q[W + K + t], KN[W + K + t], VN[W + K + t], o, logits_prev=LG[W + K + t], entropy=ent)
        sts = [ctx.stats(b) for b in range(B)]
        att_steps.append(sum(x["attended"] for x in sts))
        if a.workload == "c3" and sts[0]["recovery_action"]:
            recov.append({"step": int(sts[0]["step"]), "level": int(sts[0]["recovery_action"]),
                          "restored": int(sts[0]["restored_this_step"])})
    torch.cuda.synchronize()
    stage_ms, launches = ctx.stage_times()
    ctx.set_profile(False)
    stats_p = [ctx.stats(b) for b in range(B)]
    # ---- the attention kernel alone (asr_time_attention): R back-to-back launches over the A_i the
    #      next step would attend, after an L2 flush, bracketed by CUDA events on the launch stream
    R = 4
    alone = []
    for _ in range(3):
        flush.zero_()
        torch.cuda.synchronize()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(st)
        ctx.time_attention(R)   # on the current stream (st)
        eb.record(st)
        torch.cuda.synchronize()
        alone.append(ea.elapsed_time(eb) / R)
    attn_alone_ms = statistics.median(alone)
    timeline = None
    if a.timeline:
        tls = []
        from paper_2512_11221_b200.asr import asr_tail_trace
        traces = []
        for t in range(8):
            flush.zero_()
            ctx.step(Q[W + t], KN[W + t], VN[W + t], o, logits_prev=LG[W + t], entropy=ent)
            tls.append(ctx.timeline())
            traces.append(asr_tail_trace(ctx._h))
        tr = traces[-1]
        settle = tr[[c * 32 + w for c in range(148) for w in range(10)]]
        settle = settle[settle[:, 0] >= 0]
        comb = tr[[c * 32 + 16 + w for c in range(148) for w in range(10)]]
        comb = comb[comb[:, 0] >= 0]
        if len(settle):
            d = np.diff(settle, axis=1)
            print("tail trace settle warps:", len(settle), "start med/max", np.median(settle[:, 0]), settle[:, 0].max(),
                  "stage durations med", np.round(np.median(d, axis=0), 3).tolist(), "max", np.round(d.max(axis=0), 3).tolist(),
                  "end max", settle[:, 7].max(), file=sys.stderr)
        if len(comb):
            print("tail trace combine warps:", len(comb), "start med/max", np.median(comb[:, 0]), comb[:, 0].max(),
                  "dur med/max", np.median(comb[:, 7] - comb[:, 0]), (comb[:, 7] - comb[:, 0]).max(),
                  "end max", comb[:, 7].max(), file=sys.stderr)
        med = [round(statistics.median(x), 3) for x in zip(*tls)]
        timeline = {"pre_start_end_attn_start_end_post_start_end_us": med[:6],
                    "post_decide_end_next_list_end_combine_end_us": med[6:9],
                    "pre_entropy_end_append_end_phaseB_start_end_us": med[9:13],
                    "attn_first_cta_end_us": med[13:14], "post_released_us": med[14:15],
                    "tail_barrier_arrive_release_decide_tick_count_lookback_write_first_us": med[15:23],
                    "cta_past_attention_past_phaseB_wait_us": med[23:25], "tail_dry_pass_end_us": med[25:26]}
        print("timeline (us):", json.dumps(tls), file=sys.stderr)
    # attended per step: the mean over the profiled pass's steps (the K steps right after the timed
    # ones; |A_i| drifts by a few tokens per step in the grown state and cycles with the cohort in
    # configs[3]'s prefill state, so the mean over K steps stands for the timed steps)
    att_last = sum(s["attended"] for s in stats)
    att_prof = sum(att_steps) / len(att_steps)
    total_t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(total_t, op=dist.ReduceOp.MAX)
    total_max = float(total_t.item())
    # ---- e2e through the C ABI with HOST buffers (copies inside the timed region)
    e2e = None
    if e2e_steps:
        hq = [torch.empty((B, L, hq_r, D), dtype=bf).pin_memory() for _ in range(2)]
        hk = [torch.empty((B, L, hkv_r, D), dtype=bf).pin_memory() for _ in range(2)]
        hv = [torch.empty((B, L, hkv_r, D), dtype=bf).pin_memory() for _ in range(2)]
        hl = [torch.empty((B, VOCAB), dtype=bf).pin_memory() for _ in range(2)]
        ho = torch.empty((B, L, hq_r, D), dtype=torch.float32).pin_memory()
        he = torch.empty((B,), dtype=torch.float32).pin_memory()
        base = grow + n_meas
        hq_rs, HKs, HVs, HLs = [], [], [], []
        for t in range(e2e_steps):
            inputs(base + t, q, kn, vn, lg)
            hq_rs.append(q.cpu().pin_memory()); HKs.append(kn.cpu().pin_memory())
            HVs.append(vn.cpu().pin_memory()); HLs.append(lg.cpu().pin_memory())
        # one untimed host-I/O step allocates the library's staging buffers
        inputs(base + e2e_steps, q, kn, vn, lg)
        ctx.step(q.cpu().pin_memory(), kn.cpu().pin_memory(), vn.cpu().pin_memory(), ho,
                 logits_prev=lg.cpu().pin_memory(), entropy=he)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # the library's pipelined host I/O (inputs of step t+1 copied while step t computes, outputs of
        # step t copied while step t+1 computes), with the same L2 flush before every step as the
        # device-timed loop: the flushes are bracketed by their own events and their time subtracted
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(e2e_steps)]
        e0.record(st)
        for t in range(e2e_steps):
            fev[t][0].record(st)
            flush.zero_()
            fev[t][1].record(st)
            ctx.step(hq_rs[t], HKs[t], HVs[t], ho, logits_prev=HLs[t], entropy=he)
        ctx.flush()   # the stream waits for the last step's outputs to land in host memory
        e1.record(st)
        torch.cuda.synchronize()
        e2e_total = e0.elapsed_time(e1) - sum(f0.elapsed_time(f1) for f0, f1 in fev)
        e2e_ms = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        h2d = B * (L * hq_r * D * 2 + 2 * L * hkv_r * D * 2 + VOCAB * 2)
        d2h = B * (L * hq_r * D * 4 + 4)
        e2e = {"value": B * e2e_steps * (1 if a.head_shard else world) / (float(e2e_ms.item()) / 1000.0), "unit": "tok/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "note": "asr_step with pinned host q/k/v/logits in and o/entropy out, copies inside the timed region "
                       "(the library overlaps them with neighbouring steps on two copy streams); L2 flushed before "
                       "every step, the flushes' own event-timed durations subtracted"}
    # ---- roofline of the dominant kernel (attention + fused score), measured live via stage events
    attn_ms = stage_ms[1]
    # algorithmic bytes per attended token-layer: K+V rows (2*Hkv*d*2 B) + index (4 B) + score partial (4 B);
    # per (sequence, layer): q (Hq*d*2 B).  |A_i| per step ~ att_last (drifts < 0.5 % over the window).
    bytes_per_step = L * att_prof * (2 * hkv_r * D * 2 + 8) + B * L * hq_r * D * 2
    # batch 1: phase A runs inside the attention kernel (logits row read, k_new/v_new read + slot write)
    n_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    if a.pool_frac == 0 and B * (64 + L) <= n_sms:
        bytes_per_step += B * (VOCAB * 2 + 2 * (2 * L * hkv_r * D * 2))
    achieved_prof = bytes_per_step * K / (attn_ms / 1000.0) / 1e9
    # the kernel alone moves the attention's bytes only (no phase A inside); its A is the next step's:
    # the post-step Active tokens + the one the next step appends, per sequence
    att_next = sum(x["active"] + 1 for x in stats_p)
    bytes_alone = L * att_next * (2 * hkv_r * D * 2 + 8) + B * L * hq_r * D * 2
    achieved = bytes_alone / (attn_alone_ms / 1000.0) / 1e9
    peak, peak_kind = measured_peak_hbm()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "attn_traffic.json")) as f:
            for tr in json.load(f)["entries"]:
                if tr.get("context") == a.context and tr.get("family") == a.family and tr.get("batch") == B:
                    traffic = tr["dram_bytes_per_launch"]
    except Exception:
        pass
    # sequence sharding: every rank decodes its own batch; head sharding: all ranks decode one batch
    value = B * K * (1 if a.head_shard else world) / (total_max / 1000.0)
    # the whole step against the same roofline: the attention's algorithmic bytes of a mean step (the
    # profiled pass's |A_i|) / the timed step time
    step_bytes = L * att_prof * (2 * hkv_r * D * 2 + 8) + B * L * hq_r * D * 2
    step_gbs = step_bytes / (total_max / K / 1000.0) / 1e9
    stall_ns = (stats[0]["h2d_stall_ns"] - io0["h2d_stall_ns"]) / K if pool else 0.0
    link_peak = None
    if pool and rank == 0:   # pinned host -> device cudaMemcpyAsync peak on this box, same run
        hbuf = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
        dbuf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        for _ in range(2):
            dbuf.copy_(hbuf, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(5):
            dbuf.copy_(hbuf, non_blocking=True)
        e1.record(st)
        torch.cuda.synchronize()
        link_peak = 5 * (256 << 20) / (e0.elapsed_time(e1) / 1000.0) / 1e9
        del hbuf, dbuf
    ctx.close()
    del Q, KN, VN, LG, flush_w, flush_r
    torch.cuda.empty_cache()
    if rank != 0:
        return None
    cpu = None
    if not a.no_cpu_baseline and world == 1:
        r = oracle_sample(a, a.cpu_seconds)
        cpu = {"value": r["value"], "unit": "tok/s", "cores": r["cores"], "kind": "oracle", "sample": r["sample"]}
    if a.workload == "c3":
        wl = f"configs[3]: llama3-8b-shape ctx{a.context} prefill batch{B} window{a.window} needle+entropy-spikes"
        state = f"{P}-token prompt (prefill, every token Active), decoded to step {C3_Q - 3} before timing"
    elif a.workload == "c4":
        wl = f"configs[4] share: llama3-8b-shape ctx{a.context} batch{B}/rank of {B * world} window{a.window} {a.family}"
        state = "grown from a 512-token prompt"
    else:
        wl = (f"llama3-8b-shape ctx{a.context} batch{B} window{a.window} {a.family}"
              + (f" pool{a.pool_frac:g}" if pool else "") + (" int8-tier" if pool and a.mirror_bits == 8 else "") + (f" tau{a.tau:g}" if a.tau != 0.5 else "")
              + (f" W{a.history_window}" if a.history_window else ""))
        state = "grown from a 512-token prompt"
    line = {
        "metric": "decode tokens/sec at LLaMA-3-8B shape vs context; achieved HBM GB/s vs 8 TB/s",
        "value": value, "unit": "tok/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": total_max / K, "higher_is_better": True, "scaling": "strong" if a.head_shard else "weak",
        "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic",
        "config": {"workload": wl,
                   "context": a.context, "batch_per_gpu": B, "window": a.window, "tau": a.tau, "k": 2,
                   "family": a.family, "state": state,
                   "l2": "flushed between timed steps (256 MiB write + 256 MiB read, outside the events)",
                   "parallelism": (f"head-sharded x{world} (NCCL all-reduce of per-token partial scores)" if a.head_shard
                                   else f"sequence-sharded x{world} (no hot-path collective)"),
                   "head_shard": {"rank_identical_decisions": rank_identical,
                                  "allreduce_bytes_per_step": allreduce_bytes_step,
                                  "attended_bytes_per_step": 4 * att_prof} if a.head_shard else None},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "attention+score (split-KV over A_i)",
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                     "bytes_per_launch": bytes_alone, "ms_per_launch": attn_alone_ms,
                     "timing": f"CUDA events around {R} back-to-back launches of the attention kernel over the "
                               "A_i of the measured workload (asr_time_attention, after an L2 flush; median of 3)",
                     "step_level": {"achieved": step_gbs, "frac": step_gbs / peak, "bytes_per_step": step_bytes,
                                    "timing": "the attention's algorithmic bytes per step / the timed step time "
                                              "(every stage of the step in the denominator)"},
                     "profiled_pass": {"achieved": achieved_prof, "frac": achieved_prof / peak,
                                       "bytes_per_launch": bytes_per_step, "ms_per_launch": attn_ms / K,
                                       "timing": "CUDA event nodes around the kernel inside K further steps "
                                                 "(includes its launch latency and, at batch 1, phase A/B)"}},
        "e2e": e2e,
        "gpu_launches": launches_timed,
        "cpu_baseline": cpu,
        "clocks": clk,
        "offload": {"mode": "pressure" if pool else "full residency", "pool_tokens": pool,
                    "evict_min_absence": a.evict_min if pool else None,
                    "resident_tokens": sum(s_["resident"] for s_ in stats),
                    "total_tokens": sum(s_["total"] for s_ in stats),
                    "h2d_bytes_per_step": h2d_timed / K, "d2h_bytes_per_step": d2h_timed / K,
                    "host_link_gbs": (h2d_timed + d2h_timed) / (total_max / 1000.0) / 1e9,
                    "host_link_peak_gbs": link_peak,
                    "host_link_frac": ((h2d_timed / (total_max / 1000.0) / 1e9) / link_peak) if link_peak else None,
                    "evict_policy": ("belady" if a.evict_policy == 0 else "at-freeze") if pool else None,
                    "h2d_stall_us_per_step": stall_ns / 1000.0,
                    "note": "H2D = prefetch + demand copies of evicted tokens (device-driven gather over the mapped "
                            "mirror); D2H = write-once mirror of appended tokens; host_link_peak = pinned "
                            "cudaMemcpyAsync H2D of 256 MiB in the same run; stall = demand copies + prefetch copies "
                            "outlasting the attention kernel (device clock)"},
        "detail": {"attended_per_step": att_prof / B, "attended_per_step_range": [min(att_steps) / B, max(att_steps) / B],
                   "active_post": stats[0]["active"], "total": stats[0]["total"],
                   "compression": stats[0]["compression"],
                   "stage_ms_per_step_profiled": {n: v / K for n, v in zip(STAGES, stage_ms)},
                   "profiled_launches": launches,
                   "timeline": timeline,
                   "step_ms_min": min(step_ms), "step_ms_median": statistics.median(step_ms),
                   "wall_s_timed": t_wall, "grow_s": t_grow,
                   "host_link_d2h_mirror_bytes_per_step": B * TOKEN_KV_BYTES if cfg.host_mirror else 0,
                   "recovery_in_profiled_pass": recov if a.workload == "c3" else None},
    }
    return line


POINTS = {   # extra workloads measured after the headline
    "c2": dict(batch=64, steps=16, warmup=4, pool_frac=0.0),        # BASELINE.json configs[2]: 8K, batch 64
    "ctx32k": dict(context=32768, steps=32, no_mirror=True),        # the north_star's 32K context, batch 1
    "c3": dict(workload="c3", context=32768, batch=16, steps=16, warmup=3, no_mirror=True),   # configs[3]
    "w1": dict(family="w1"),                                        # 30 % hot tokens (SURVEY W1 family)
    "full": dict(tau=0.0),                                          # full-KV baseline: nothing freezes
    "pool": dict(pool_frac=0.5, steps=16, warmup=4),                # pressure mode: 50 % device pool, Belady
    "pool8": dict(pool_frac=0.5, steps=16, warmup=4, mirror_bits=8),   # + the INT8 frozen tier on the link
    "w128": dict(history_window=128),                               # NEXT-3: finite history window W
    "c4share": dict(workload="c4", context=32768, batch=32, steps=8, warmup=3, no_mirror=True),  # opt-in
}


def sample_point(local_rank: int) -> dict:
    """NEXT-1: the next-token draw (asr_sample) at the LLaMA-3 vocabulary, batch 1 and 64, timed with
    CUDA events over 20 calls (logits resident in HBM; algorithmic bytes = one read of each row):
    us_per_call back to back from Python (the host launch path included), us_per_call_device the same
    calls replayed from a CUDA graph (rows_per_s and GB/s from the device time)."""
    import torch

    import gen
    from paper_2512_11221_b200 import asr_sample, asr_sample_entropy
    dev = torch.device("cuda", local_rank)
    out = {}
    for B in (1, 64):
        g = gen.GenParams(seed=7, L=1, Hq=2, Hkv=2, d=16, vocab=VOCAB)
        lg = torch.empty((B, VOCAB), dtype=torch.bfloat16, device=dev)
        gen.dev_logits(g, B, 5, lg)
        u = torch.rand(B, device=dev)
        tok = torch.empty(B, dtype=torch.int32, device=dev)
        ent = torch.empty(B, dtype=torch.float32, device=dev)
        res = {}
        for name, (T, k, P) in {"greedy": (0.0, 0, 1.0), "T0.8_k50_p0.9": (0.8, 50, 0.9), "T1_p0.95": (1.0, 0, 0.95)}.items():
            for fused in (False, True):   # fused: + the row's entropy for the next step (asr_sample_entropy)
                def call():
                    if fused:
                        asr_sample_entropy(lg, u, tok, ent, temperature=T, top_k=k, top_p=P)
                    else:
                        asr_sample(lg, u, tok, temperature=T, top_k=k, top_p=P)
                for _ in range(3):
                    call()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(20):
                    call()
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1000 / 20
                # device time: the same 20 calls replayed from a CUDA graph (no Python launch path)
                s = torch.cuda.Stream(device=dev)
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.stream(s):
                    with torch.cuda.graph(gr, stream=s):
                        for _ in range(20):
                            call()
                torch.cuda.synchronize()
                gr.replay()
                torch.cuda.synchronize()
                e0.record()
                gr.replay()
                e1.record()
                torch.cuda.synchronize()
                ud = e0.elapsed_time(e1) * 1000 / 20
                res[name + ("+entropy" if fused else "")] = {"us_per_call": round(us, 2), "us_per_call_device": round(ud, 2),
                                                            "rows_per_s": round(B / ud * 1e6),
                                                            "gbs_one_read": round(B * VOCAB * 2 / ud / 1e3, 1)}
        out[f"batch{B}"] = res
    return out


def quant_point(local_rank: int) -> dict:
    """NEXT-4: the quantised frozen tier (asr_kv_quantize / asr_kv_dequantize).  Tier = the frozen
    KV of the configs[1] point (6900 tokens x 32 layers x K,V x 8 heads = 3.53M rows of 128 bf16, 904 MB;
    larger than L2, so every call streams HBM).  Kernel GB/s = algorithmic bytes (bf16 read + codes and
    scales written, or the reverse) / CUDA-event time over 10 calls.  Restore over the host link: the
    pressure-mode H2D volume per step at 8K (105 MB of bf16) copied from pinned memory as
    bf16, vs its INT8/INT4 codes + scales copied and dequantised on the device."""
    import torch

    from paper_2512_11221_b200 import asr_kv_dequantize, asr_kv_quantize
    dev = torch.device("cuda", local_rank)
    peak, kind = measured_peak_hbm()
    rows, n = 6900 * 512, 128
    g = torch.Generator(device=dev).manual_seed(5)
    kv = torch.randn((rows, n), device=dev, generator=g).to(torch.bfloat16)
    back = torch.empty_like(kv)
    scales = torch.empty(rows, dtype=torch.float32, device=dev)
    out = {"rows": rows, "row_elems": n, "peak_gbs": peak, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({kind})"}

    def timed(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps   # ms

    for bits in (8, 4):
        cb = n if bits == 8 else n // 2
        codes = torch.empty((rows, cb), dtype=torch.int8, device=dev)
        moved = rows * (2 * n + cb + 4)
        tq = timed(lambda: asr_kv_quantize(kv, codes, scales, bits=bits))
        td = timed(lambda: asr_kv_dequantize(codes, scales, back, bits=bits))
        # host-link restore of 105 MB of bf16 KV (the pressure-mode H2D per step at 8K): 420K rows of 256 B
        rr = 105 * 1024 * 1024 // (2 * n)
        h_bf16 = torch.empty((rr, n), dtype=torch.bfloat16, pin_memory=True)
        h_codes = torch.empty((rr, cb), dtype=torch.int8, pin_memory=True)
        h_sc = torch.empty(rr, dtype=torch.float32, pin_memory=True)
        d_codes = torch.empty((rr, cb), dtype=torch.int8, device=dev)
        d_sc = torch.empty(rr, dtype=torch.float32, device=dev)
        d_kv = torch.empty((rr, n), dtype=torch.bfloat16, device=dev)
        t_bf16 = timed(lambda: d_kv.copy_(h_bf16, non_blocking=True), reps=5)

        def q_restore():
            d_codes.copy_(h_codes, non_blocking=True)
            d_sc.copy_(h_sc, non_blocking=True)
            asr_kv_dequantize(d_codes, d_sc, d_kv, bits=bits)
        t_q = timed(q_restore, reps=5)
        out[f"int{bits}"] = {
            "quantize_us": round(tq * 1e3, 1), "quantize_gbs": round(moved / tq / 1e6, 1),
            "quantize_frac": round(moved / tq / 1e6 / peak, 3),
            "dequantize_us": round(td * 1e3, 1), "dequantize_gbs": round(moved / td / 1e6, 1),
            "dequantize_frac": round(moved / td / 1e6 / peak, 3),
            "bytes_per_row": {"bf16": 2 * n, "codes": cb, "scale": 4},
            "restore_105MB": {"bf16_h2d_us": round(t_bf16 * 1e3, 1), "quant_h2d_plus_dequant_us": round(t_q * 1e3, 1),
                              "h2d_bytes_bf16": rr * 2 * n, "h2d_bytes_quant": rr * (cb + 4),
                              "speedup": round(t_bf16 / t_q, 2)}}
        del codes, h_bf16, h_codes, h_sc, d_codes, d_sc, d_kv
    return out


def replay_point(local_rank: int) -> dict:
    """NEXT-2: policy replay (asr_step_policy) of the all-cold trace for 1024 sequences at 8K context,
    K = 512 — Alg. 1 lines 3-15 + compaction for every sequence, no attention; sequence-steps per second
    (CUDA events over 32 steps, after the sequences have grown to 8K)."""
    import torch

    from paper_2512_11221_b200 import Config, Context
    dev = torch.device("cuda", local_rank)
    B, ctxlen, P, K = 1024, 8192, 512, 32
    cfg = Config(n_layers=1, n_q_heads=2, n_kv_heads=2, head_dim=16, batch=B, max_context=ctxlen + K + 8, window=512,
                 tau=0.5, softness=2.0, vocab=0, host_mirror=0, device=local_rank)
    pk = torch.zeros((B, P, 1, 2, 16), dtype=torch.bfloat16, device=dev)
    ctx = Context(cfg, pk, pk.clone(), [P] * B)
    scores = torch.full((B, cfg.max_context), 0.25, dtype=torch.float32, device=dev)   # every token below tau
    for _ in range(ctxlen - P):
        ctx.step_policy(scores)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        ctx.step_policy(scores)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    st = ctx.stats(0)
    ctx.close()
    return {"workload": f"policy replay, all-cold trace, {B} sequences at {ctxlen} tokens, K=512",
            "ms_per_step": ms, "sequence_steps_per_s": B / (ms / 1000.0), "active_post": st["active"],
            "total": st["total"]}


def spawn_ranks(a) -> int:
    """`--gpus N` outside torchrun: re-launch this command as N ranks (one process per GPU) under
    torch.distributed.run on 127.0.0.1 and return its exit code (rank 0 prints the line)."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def sweep_point(local_rank: int) -> dict:
    """NEXT-2: the (tau, K, k, W) sensitivity sweep (SPEC run_sweep) of the policy on a uniform
    relevance trace, 4 sequences grown from a 1024-token prompt by 512 steps, 32 cells replayed on the GPU
    (paper_2512_11221_b200/sweep.py); cell-steps per second over the whole sweep (host stats included)."""
    import torch

    import gen
    from paper_2512_11221_b200.sweep import run_sweep
    B, prompt, steps = 4, 1024, 512
    sc = torch.from_numpy(gen.score_trace("uniform", B, prompt + steps + 1, seed=3)).cuda(local_rank)
    grid = {"tau": [0.2, 0.4, 0.6, 0.8], "window": [32, 512], "softness": [1.0, 2.0], "history_window": [0, 64]}
    t0 = time.perf_counter()
    rows = run_sweep(grid, sc, steps, prompt, device=local_rank)
    dt = time.perf_counter() - t0
    table = [{k: r[k] for k in ("tau", "window", "softness", "history_window", "mean_compression", "max_absence",
                                "recoveries", "final_active", "final_total")} for r in rows]
    return {"workload": f"uniform trace, batch {B}, prompt {prompt} + {steps} steps, {len(rows)} cells",
            "seconds": dt, "cell_steps_per_s": len(rows) * steps / dt, "table": table}


def main():
    a = parse()
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        sys.exit(spawn_ranks(a))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        print(json.dumps({"error": f"--gpus {a.gpus} but WORLD_SIZE={world}: launch one rank per GPU"}), flush=True)
        sys.exit(2)
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    if a.workload == "c4":
        # configs[4]: 256 sequences at 32K sharded by sequence over the ranks (weak in the per-rank share)
        a.context, a.batch, a.no_mirror = 32768, max(1, 256 // world), True
        a.points = a.points if a.points != parse_default_points() else ""
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_asr(a, rank, world, local_rank)
    if line is not None and "unavailable" in line:
        print(json.dumps({"metric": "decode tokens/sec at LLaMA-3-8B shape vs context; achieved HBM GB/s vs 8 TB/s",
                          "unavailable": line["unavailable"], "n_gpus": world}), flush=True)
        sys.exit(0)
    points = {}
    wanted = [x for x in a.points.split(",") if x]
    for name in [x for x in wanted if x not in ("sample", "replay", "quant", "sweep")]:
        b = argparse.Namespace(**vars(a))
        for k, v in POINTS[name].items():
            setattr(b, k, v)
        b.no_e2e, b.no_cpu_baseline, b.timeline = True, True, False
        r = run_asr(b, rank, world, local_rank)
        if r is None:
            continue
        if "unavailable" in r:
            points[name] = {"unavailable": r["unavailable"]}
            continue
        points[name] = {"workload": r["config"]["workload"], "value": r["value"], "unit": r["unit"],
                        "ms_per_step": r["ms_per_step"], "steps": r["steps"], "warmup": r["warmup"],
                        "roofline": {k: r["roofline"][k] for k in ("bound", "achieved", "peak", "frac", "unit",
                                                                   "bytes_per_launch", "ms_per_launch")},
                        "step_level": r["roofline"]["step_level"],
                        "offload": r["offload"], "clocks": r["clocks"], "gpu_launches": r["gpu_launches"],
                        "attended_per_step": r["detail"]["attended_per_step"],
                        "compression": r["detail"]["compression"],
                        "state": r["config"]["state"]}
        if r["detail"].get("recovery_in_profiled_pass") is not None:
            points[name]["recovery_in_profiled_pass"] = r["detail"]["recovery_in_profiled_pass"]
    if line is not None and world == 1 and "sample" in wanted:
        line["detail"]["next_token_draw"] = sample_point(local_rank)
    if line is not None and world == 1 and "replay" in wanted:
        line["detail"]["policy_replay"] = replay_point(local_rank)
    if line is not None and world == 1 and "quant" in wanted:
        line["detail"]["frozen_tier_quant"] = quant_point(local_rank)
    if line is not None and world == 1 and "sweep" in wanted:
        line["detail"]["sensitivity_sweep"] = sweep_point(local_rank)
    if line is not None:
        if points:
            line["points"] = points
            if "full" in points and points["full"].get("value", 0) > 0:   # ASR-KF-EGR vs attending the whole cache
                line["detail"]["speedup_vs_full_kv"] = line["value"] / points["full"]["value"]
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def parse_default_points() -> str:
    return "c2,ctx32k,c3,w1,full,pool,pool8,sample,replay,quant,sweep"


if __name__ == "__main__":
    main()
