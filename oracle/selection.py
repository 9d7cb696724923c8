"""Query and KV selection in float64 (oracle; test infrastructure only).

Restates ``query_select.py:41-92``, ``block_probe.py:44-78`` and
``kv_select.py:49-195``. Functions take plain arrays (one head at a time or
lists of per-head vectors) rather than the reference's dataclasses.
"""

from __future__ import annotations

import math

import numpy as np

from paper_2511_12201_b200.errors import IntegrityError, LayoutError, ParameterError

from .numerics import block_lengths, colsum, f64, kurtosis, matmul, mean_pool_rows, softmax_rows

STOCHASTIC_ATOL = 1e-6  # kv_select.py:20


# ---------------------------------------------------------------- query side
def probe_keys(k: np.ndarray, n_vision: int, sink_index: int) -> tuple[np.ndarray, np.ndarray]:
    """``query_select.py:41-47``: (k_lazy = K[sink], k_act = mean(K[:nv]))."""
    if n_vision == 0:
        raise LayoutError("probe keys need at least one vision token")
    k = np.asarray(k)
    return np.array(k[sink_index], dtype=np.float64), np.asarray(
        f64(k[:n_vision]).mean(axis=0), dtype=np.float64
    )


def classify(q: np.ndarray, k_lazy: np.ndarray, k_act: np.ndarray, tau: float):
    """``query_select.py:50-68``: two-logit softmax; active iff p_act > tau
    (strict). Returns (p_act, active)."""
    if not 0.0 <= tau < 1.0:
        raise ValueError(f"tau must be in [0, 1), got {tau}")
    q = f64(q)
    refs = np.stack([f64(k_lazy), f64(k_act)])  # lazy column first
    logits = matmul(q, refs.T) * (1.0 / np.sqrt(q.shape[1]))
    p_act = softmax_rows(logits)[:, 1]
    return p_act, p_act > tau


def query_mask(q: np.ndarray, k_lazy, k_act, n_vision: int, tau: float, force_all: bool) -> np.ndarray:
    """``query_select.py:71-92`` for one head: vision rows classified, text and
    answer rows active; ``force_all`` is the first-head preservation."""
    _, verdict = classify(q[:n_vision], k_lazy, k_act, tau)
    active = np.ones(np.asarray(q).shape[0], dtype=bool)
    active[:n_vision] = verdict
    if force_all:
        active[:] = True
    return active


# ----------------------------------------------------------- block probe
def probe_map(q: np.ndarray, k: np.ndarray, block: int) -> np.ndarray:
    """``block_probe.py:44-64``: block-causal softmax of pooled Q pooled K^T."""
    if block < 1:
        raise ParameterError(f"block size must be >= 1, got {block}")
    pq = mean_pool_rows(q, block)
    pk = mean_pool_rows(k, block)
    s = matmul(pq, pk.T) * (1.0 / np.sqrt(np.asarray(q).shape[1]))
    nb = pq.shape[0]
    return softmax_rows(s, np.tril(np.ones((nb, nb), dtype=bool)))


def block_mass(pmap: np.ndarray) -> np.ndarray:
    """Column mass of a probe map (the ``colsum`` inside
    ``block_probe.py:76``)."""
    return colsum(pmap)


def token_scores_from_blocks(mass: np.ndarray, n: int, block: int) -> np.ndarray:
    """``block_probe.py:67-78``: block mass / true block length, repeated per
    token (sums to nb, not n)."""
    lens = block_lengths(n, block)
    if mass.shape[0] != lens.shape[0]:
        raise ParameterError(f"map covers {mass.shape[0]} blocks, asked for {lens.shape[0]}")
    return np.repeat(f64(mass) / lens.astype(np.float64), lens)


def exact_scores(attn: np.ndarray) -> np.ndarray:
    """``kv_select.py:56-73`` for one head: column sums of a row-stochastic
    map with the integrity checks."""
    attn = f64(attn)
    rs = attn.sum(axis=1)
    if np.abs(rs - 1.0).max() > STOCHASTIC_ATOL:
        worst = int(np.abs(rs - 1.0).argmax())
        raise IntegrityError(f"attention row {worst} sums to {rs[worst]:.9f}, not 1")
    if attn.min() < 0.0:
        raise IntegrityError("attention has negative entries")
    return colsum(attn)


# --------------------------------------------------------------- KV budget
def kurtoses(vectors: list[np.ndarray]) -> list[float]:
    """``kv_select.py:49-53``."""
    return [kurtosis(v) for v in vectors]


def flattest(kurt: list[float]) -> int:
    """``kv_select.py:76-80``: argmin, ties to the lowest index."""
    if len(kurt) < 1:
        raise ParameterError("need at least one head")
    return int(np.argmin(np.asarray(kurt, dtype=np.float64)))


def budget(a_star: np.ndarray, p: float, total_mass: float | None = None) -> tuple[int, float, float]:
    """``kv_select.py:87-120``: (b, retained, total) — b is the smallest
    descending-sorted prefix whose sequential cumsum reaches
    min(p * total, cum[-1]) (searchsorted-left + 1)."""
    if not 0.0 < p <= 1.0:
        raise ParameterError(f"retention p must be in (0, 1], got {p}")
    cum = np.cumsum(np.sort(f64(a_star))[::-1])
    total = float(total_mass) if total_mass is not None else float(cum[-1])
    thr = min(p * total, cum[-1])
    b = int(np.searchsorted(cum, thr, side="left")) + 1
    return b, float(cum[b - 1]), total


def top_b(a: np.ndarray, b: int) -> np.ndarray:
    """``kv_select.py:123-127``: ascending indices of the b largest scores,
    cutoff ties to the lower index."""
    a = f64(a)
    order = np.lexsort((np.arange(a.shape[0]), -a))
    return np.sort(order[:b]).astype(np.int64)


def key_masks(vectors: list[np.ndarray], b: int) -> list[np.ndarray]:
    """``kv_select.py:130-144`` (token granularity)."""
    n = vectors[0].shape[0]
    if not 1 <= b <= n:
        raise ParameterError(f"budget must be in [1, {n}], got {b}")
    return [top_b(a, b) for a in vectors]


def top_blocks(vectors: list[np.ndarray], b: int, block: int) -> list[np.ndarray]:
    """``kv_select.py:147-176`` (block granularity): whole blocks by summed
    mass (ties to the lower block), the marginal block contributes its lowest
    indices."""
    n = vectors[0].shape[0]
    if not 1 <= b <= n:
        raise ParameterError(f"budget must be in [1, {n}], got {b}")
    if block < 1:
        raise ParameterError(f"block size must be >= 1, got {block}")
    starts = np.arange(0, n, block)
    out = []
    for a in vectors:
        mass = np.add.reduceat(f64(a), starts)
        picked, left = [], b
        for j in np.lexsort((np.arange(starts.shape[0]), -mass)):
            lo = int(starts[j])
            take = min(min(lo + block, n) - lo, left)
            picked.append(np.arange(lo, lo + take, dtype=np.int64))
            left -= take
            if left == 0:
                break
        out.append(np.sort(np.concatenate(picked)))
    return out


def vision_keys(vectors: list[np.ndarray], b: int, n_vision: int) -> tuple[int, list[np.ndarray]]:
    """``kv_select.py:179-195``: per-head top keys inside the vision span, b
    capped at n_vision."""
    if n_vision < 1:
        raise ParameterError("vision span is empty")
    bb = min(b, n_vision)
    if bb < 1:
        raise ParameterError(f"budget must be positive, got {b}")
    return bb, [top_b(a[:n_vision], bb) for a in vectors]


def sparsity_gap(vectors: list[np.ndarray], p: float) -> float:
    """``kv_select.py:198-210``."""
    if len(vectors) < 2:
        raise ParameterError("sparsity gap needs at least two heads")
    kurt = kurtoses(vectors)
    flat, sharp = flattest(kurt), int(np.argmax(kurt))
    return (budget(vectors[flat], p)[0] - budget(vectors[sharp], p)[0]) / vectors[0].shape[0]


def num_blocks(n: int, block: int) -> int:
    return math.ceil(n / block)
