"""Sparse prefill attention and slimmed decode in float64 (oracle; tests only).

Restates ``prefill.py:89-122`` (``sparse_head_attention``),
``attention.py:94-134`` (dense causal oracle) and ``decode.py:82-228``
(cache build, decode classification, conditional-fetch decode, dense decode
oracle). Rows are processed in chunks so 32K-64K heads fit in host memory;
per-row arithmetic is unchanged by chunking.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2511_12201_b200.errors import DegenerateContextError, IntegrityError, ShapeError

from .numerics import f64, matmul, softmax_rows
from .selection import classify, probe_keys

VALUE_BYTES = 8  # metrics.py:23 (flat f64 memory model of the FetchLog)


def sparse_head_attention(q, k, v, selected, active, sink_index: int, row_chunk: int = 2048,
                          rows_subset: np.ndarray | None = None) -> np.ndarray:
    """``prefill.py:89-122``: active rows attend causally (original positions)
    to the selected keys, softmax renormalised over the visible ones; rows with
    no visible key copy ``v[sink]``; lazy rows are zero.

    ``rows_subset`` (test/bench sampling only) restricts the computed rows to a
    subset of the active rows; other rows stay zero.
    """
    q, k, v = f64(q), f64(k), f64(v)
    selected = np.asarray(selected, dtype=np.int64)
    out = np.zeros_like(v)
    rows = np.flatnonzero(np.asarray(active, dtype=bool))
    if rows_subset is not None:
        rows = np.intersect1d(rows, np.asarray(rows_subset, dtype=np.int64))
    if rows.size == 0 or selected.size == 0:
        return out
    k_sel, v_sel = k[selected], v[selected]
    scale = 1.0 / np.sqrt(q.shape[1])
    for lo in range(0, rows.size, row_chunk):
        r = rows[lo:lo + row_chunk]
        s = matmul(q[r], k_sel.T) * scale
        vis = selected[None, :] <= r[:, None]
        alive = vis.any(axis=1)
        probs = np.zeros_like(s)
        if alive.any():
            probs[alive] = softmax_rows(s[alive], vis[alive])
        o = matmul(probs, v_sel)
        if not alive.all():
            o[~alive] = v[sink_index]
        out[r] = o
    return out


def sparse_head_lse(q, k, selected, active, row_chunk: int = 2048) -> np.ndarray:
    """Natural-log softmax normaliser per active row over its visible selected
    keys (-inf for lazy rows and rows with no visible key). Not in the
    reference; used to check the forward kernel's LSE side output."""
    q, k = f64(q), f64(k)
    selected = np.asarray(selected, dtype=np.int64)
    lse = np.full(q.shape[0], -np.inf)
    rows = np.flatnonzero(np.asarray(active, dtype=bool))
    k_sel = k[selected]
    scale = 1.0 / np.sqrt(q.shape[1])
    for lo in range(0, rows.size, row_chunk):
        r = rows[lo:lo + row_chunk]
        s = (q[r] @ k_sel.T) * scale
        vis = selected[None, :] <= r[:, None]
        s = np.where(vis, s, -np.inf)
        mx = s.max(axis=1)
        ok = np.isfinite(mx)
        val = np.full(r.shape[0], -np.inf)
        val[ok] = mx[ok] + np.log(np.exp(s[ok] - mx[ok, None]).sum(axis=1))
        lse[r] = val
    return lse


def causal_attention(q, k, v) -> tuple[np.ndarray, np.ndarray]:
    """``attention.py:99-128``: dense causal map and output (small N only)."""
    q, k, v = f64(q), f64(k), f64(v)
    n = q.shape[0]
    a = softmax_rows(matmul(q, k.T) * (1.0 / np.sqrt(q.shape[1])), np.tril(np.ones((n, k.shape[0]), dtype=bool)))
    return a, matmul(a, v)


# -------------------------------------------------------------------- decode
@dataclass
class GroupCache:
    """``decode.py:33-42`` HeadCache, one per KV head (group)."""

    vision_k: np.ndarray
    vision_v: np.ndarray
    vision_indices: np.ndarray
    text_k: np.ndarray
    text_v: np.ndarray
    k_lazy: np.ndarray
    k_act: np.ndarray
    answer_k: list = field(default_factory=list)
    answer_v: list = field(default_factory=list)


@dataclass
class FetchLog:
    """``decode.py:45-61``."""

    vision_tokens: int = 0
    vision_bytes: int = 0
    text_answer_bytes: int = 0
    step_vision_tokens: list = field(default_factory=list)
    step_active_heads: list = field(default_factory=list)


def build_cache(keys, values, selected, budget: int, n_vision: int, n_text: int, sink_index: int) -> list[GroupCache]:
    """``decode.py:82-108``: gather exactly ``budget`` vision rows per head
    (group), copy the text span, freeze probe keys from the unpruned K."""
    out = []
    for i, (k, v) in enumerate(zip(keys, values)):
        idx = np.asarray(selected[i], dtype=np.int64)
        if idx.shape[0] != budget:
            raise IntegrityError(f"head {i} selection has {idx.shape[0]} keys, budget {budget}")
        if idx.size and (idx.min() < 0 or idx.max() >= n_vision):
            raise IntegrityError(f"head {i} selection indices fall outside the vision span")
        k64, v64 = f64(k), f64(v)
        kl, ka = probe_keys(k64, n_vision, sink_index)
        out.append(GroupCache(k64[idx].copy(), v64[idx].copy(), idx.copy(),
                              k64[n_vision:n_vision + n_text].copy(), v64[n_vision:n_vision + n_text].copy(), kl, ka))
    return out


def append_answer(cache: list[GroupCache], k_rows, v_rows, head_dim: int) -> None:
    """``decode.py:111-121``."""
    if len(k_rows) != len(cache) or len(v_rows) != len(cache):
        raise ShapeError("append needs one k and one v row per head")
    for gc, k, v in zip(cache, k_rows, v_rows):
        k, v = f64(k).reshape(-1), f64(v).reshape(-1)
        if k.shape[0] != head_dim or v.shape[0] != head_dim:
            raise ShapeError(f"answer rows must have length {head_dim}")
        gc.answer_k.append(k)
        gc.answer_v.append(v)


def _segments(gc: GroupCache, fetch_vision: bool):
    """``decode.py:143-154``."""
    ks = [gc.vision_k] if fetch_vision else []
    vs = [gc.vision_v] if fetch_vision else []
    if gc.text_k.shape[0]:
        ks.append(gc.text_k)
        vs.append(gc.text_v)
    if gc.answer_k:
        ks.append(np.vstack(gc.answer_k))
        vs.append(np.vstack(gc.answer_v))
    if not ks:
        raise DegenerateContextError("lazy head with no text and no answer KV")
    return np.vstack(ks), np.vstack(vs)


def decode_flags(q_heads, cache: list[GroupCache], tau: float, rep: int, preserve_first_head: bool) -> np.ndarray:
    """``decode.py:124-140`` generalised to rule B: Q head h is classified
    against its group's (h // rep) frozen probe keys; head 0 forced active."""
    hq = len(q_heads)
    flags = np.zeros(hq, dtype=bool)
    for h in range(hq):
        gc = cache[h // rep]
        _, verdict = classify(f64(q_heads[h]).reshape(1, -1), gc.k_lazy, gc.k_act, tau)
        flags[h] = bool(verdict[0])
    if preserve_first_head:
        flags[0] = True
    return flags


def decode_step(q_heads, cache: list[GroupCache], tau: float, rep: int, preserve_first_head: bool,
                log: FetchLog, flags=None, head_dim: int | None = None):
    """``decode.py:157-194`` under rule B. Per Q head: keys = [vision if the
    head is active] + text + answer; the group's vision segment is fetched once
    when any of its Q heads is active (OR-fetch); fetch bytes are metered per
    group with the reference's flat f64 model. At rep == 1 this is the
    reference exactly (one group per head)."""
    if flags is None:
        flags = decode_flags(q_heads, cache, tau, rep, preserve_first_head)
    flags = np.asarray(flags, dtype=bool)
    d = head_dim if head_dim is not None else cache[0].vision_k.shape[1]
    outs = []
    for h in range(len(q_heads)):
        q = f64(q_heads[h]).reshape(1, -1)
        if q.shape[1] != d:
            raise ShapeError(f"decode query must have length {d}")
        keys, vals = _segments(cache[h // rep], bool(flags[h]))
        probs = softmax_rows(matmul(q, keys.T) * (1.0 / np.sqrt(d)))
        outs.append(matmul(probs, vals)[0])
    step_vision = 0
    b = cache[0].vision_k.shape[0]
    for g, gc in enumerate(cache):
        fetched = bool(flags[g * rep:(g + 1) * rep].any())
        n_ta = gc.text_k.shape[0] + len(gc.answer_k)
        if fetched:
            step_vision += b
            log.vision_bytes += b * 2 * d * VALUE_BYTES
        log.text_answer_bytes += n_ta * 2 * d * VALUE_BYTES
    log.vision_tokens += step_vision
    log.step_vision_tokens.append(step_vision)
    log.step_active_heads.append(int(flags.sum()))
    return outs, flags


def decode_dense(q_heads, cache: list[GroupCache], flags, rep: int, zero_masked_vision: bool = False):
    """``decode.py:197-228``: dense oracle over the concatenated segments with
    -inf (exclusion) or literal zeroing of a lazy head's vision rows."""
    flags = np.asarray(flags, dtype=bool)
    outs = []
    for h in range(len(q_heads)):
        gc = cache[h // rep]
        q = f64(q_heads[h]).reshape(1, -1)
        keys, vals = _segments(gc, True)
        b = gc.vision_k.shape[0]
        if not flags[h] and zero_masked_vision:
            keys, vals = keys.copy(), vals.copy()
            keys[:b] = 0.0
            vals[:b] = 0.0
        s = (q @ keys.T) / np.sqrt(q.shape[1])
        if not flags[h] and not zero_masked_vision:
            s[0, :b] = -np.inf
        e = np.exp(s - s.max())
        e[~np.isfinite(s)] = 0.0
        outs.append(((e / e.sum()) @ vals)[0])
    return outs
