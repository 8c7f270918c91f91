"""NEXT-2 sweep (paper_2512_11221_b200/sweep.py): the (tau, K, k, W) grid of policy replays on the GPU
against the oracle's policy replay of every cell (per-step active counts bit-exact), plus SPEC run_sweep's
worked properties: tau = 0 on a trace of scores >= 0 freezes nothing; k = 1 compresses at
least as much as k = 2 on the same trace; a singleton grid equals a direct run."""
import itertools

import numpy as np
import pytest

import gen
import oracle


def test_score_trace_is_deterministic_and_on_its_lattice():
    a = gen.score_trace("uniform", 3, 500, seed=4)
    b = gen.score_trace("uniform", 3, 500, seed=4)
    assert np.array_equal(a, b) and a.dtype == np.float32
    assert a.min() >= 0.0 and a.max() < 1.0
    assert np.all(a * 2.0 ** 24 == np.round(a * 2.0 ** 24))     # multiples of 2^-24: fp32 == fp64 decisions
    assert abs(float(a.mean()) - 0.5) < 0.05
    assert not np.array_equal(a, gen.score_trace("uniform", 3, 500, seed=5))
    assert np.all(gen.score_trace("w0", 2, 10) == 0.25)


def _oracle_cell(scores_row, tau, K, k, W, prompt, steps):
    cfg = oracle.OrcCfg(window=K, tau=tau, softness=k, history_window=W)
    s = oracle.OracleSeq(cfg, prompt + steps + 1, prompt)
    below = (scores_row < np.float32(tau)).astype(np.uint8)   # the kernel's precision decides (fp32 tau)
    trace = []
    for _ in range(steps):
        _, out = s.step_policy(below[:s.n + 1])
        trace.append(out["active_post"])
    return trace, int(s.ledger()["timer"].max())


@pytest.mark.gpu
def test_sweep_matches_oracle_replay_per_cell():
    import torch
    from paper_2512_11221_b200.sweep import run_sweep
    B, prompt, steps = 2, 120, 150
    sc = gen.score_trace("uniform", B, prompt + steps + 1, seed=11)
    grid = {"tau": [0.0, 0.3, 0.7], "window": [8, 32], "softness": [1.0, 2.0], "history_window": [0, 16]}
    rows = run_sweep(grid, torch.from_numpy(sc).cuda(), steps, prompt)
    assert len(rows) == 3 * 2 * 2 * 2
    by = {(r["tau"], r["window"], r["softness"], r["history_window"]): r for r in rows}
    for cell in itertools.product(*grid.values()):
        r = by[cell]
        trace, maxt = _oracle_cell(sc[0], *cell, prompt, steps)
        assert r["active_trace"] == trace, cell
        if cell[0] == 0.0:
            assert r["mean_compression"] == 0.0   # SPEC: tau = 0 on scores >= 0 freezes nothing
    for tau, K, W in itertools.product(grid["tau"], grid["window"], grid["history_window"]):
        # SPEC: k = 1 gives longer durations than k = 2 on the same trace -> at least as much compression
        assert by[(tau, K, 1.0, W)]["mean_compression"] >= by[(tau, K, 2.0, W)]["mean_compression"] - 1e-12
    one = run_sweep({"tau": [0.3], "window": [8], "softness": [2.0], "history_window": [0]},
                    torch.from_numpy(sc).cuda(), steps, prompt)
    assert one[0]["active_trace"] == by[(0.3, 8, 2.0, 0)]["active_trace"]   # singleton grid == direct run
