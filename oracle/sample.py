"""Oracle of NEXT-1: the next-token draw that closes Alg. 1 ("Generate next token",
P:102) — temperature, top-k and top-p (nucleus) filtering and one categorical draw per sequence.

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): plain numpy in fp64, no blocking or reordering
beyond the definitions below; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline may
call it.  The paper fixes none of this (it names greedy decoding for the passkey test, and
temperature/top-p as generation settings); the readings, listed in DESIGN.md §2 as R-sample:

* T <= 0 or top_k == 1: greedy, the lowest index among the maximal logits.
* p_v = softmax(x / T) over the whole row (x = the logits as given, bf16 values exact in fp64).
* top-k (k > 0): keep the k largest logits; ties at the boundary go to the lower indices.
* top-p (0 < P < 1), applied after top-k (the Hugging Face warper order): order the kept tokens by
  (logit descending, index ascending) and keep the shortest prefix whose probability mass is >= P
  times the mass of the top-k set.
* the draw: u in [0, 1) is an input (the caller's random number); the sampled token is the smallest
  vocab index j in the kept set with  sum_{i kept, i <= j} p_i  >  u * sum_{i kept} p_i  (inverse CDF in
  vocabulary order — the same distribution as any other order, and no sort is needed to evaluate it).
"""
from __future__ import annotations

import numpy as np


def _as_f64(logits: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(logits)
    if a.dtype == np.uint16:   # bf16 bits
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return a.astype(np.float64)


def kept_set(logits: np.ndarray, temperature: float, top_k: int, top_p: float) -> tuple[np.ndarray, np.ndarray]:
    """(kept indices in vocabulary order, p over the full row in fp64)."""
    x = _as_f64(logits)
    V = x.size
    if temperature <= 0 or top_k == 1:
        j = int(np.argmax(x))          # numpy: first maximal index
        p = np.zeros(V)
        p[j] = 1.0
        return np.array([j]), p
    z = x / temperature
    w = np.exp(z - z.max())
    p = w / w.sum()
    order = np.lexsort((np.arange(V), -x))          # logit descending, index ascending
    keep = order if not (0 < top_k < V) else order[:top_k]
    if 0 < top_p < 1:
        mass = p[keep]
        cum = np.cumsum(mass)
        n = int(np.searchsorted(cum, top_p * mass.sum(), side="left")) + 1   # shortest prefix with cum >= P*M
        keep = keep[:min(n, keep.size)]
    return np.sort(keep), p


def sample(logits: np.ndarray, temperature: float, top_k: int, top_p: float, u: float) -> int:
    """The sampled token id (see the module docstring)."""
    keep, p = kept_set(logits, temperature, top_k, top_p)
    if keep.size == 1:
        return int(keep[0])
    pk = p[keep]
    cum = np.cumsum(pk)
    j = int(np.searchsorted(cum, u * cum[-1], side="right"))   # first cum > u*M
    return int(keep[min(j, keep.size - 1)])


def interval(logits: np.ndarray, temperature: float, top_k: int, top_p: float, token: int) -> tuple[float, float]:
    """[lo, hi) of u that draws `token` (relative to the kept mass), or (nan, nan) if it is not kept."""
    keep, p = kept_set(logits, temperature, top_k, top_p)
    if token not in set(keep.tolist()):
        return float("nan"), float("nan")
    if keep.size == 1:
        return 0.0, 1.0
    pk = p[keep]
    cum = np.cumsum(pk) / pk.sum()
    i = int(np.flatnonzero(keep == token)[0])
    return (float(cum[i - 1]) if i else 0.0), float(cum[i])
