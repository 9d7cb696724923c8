"""Reference-named KV-selection operators on the GPU (reference
``kv_select.py:23-195``), all routed through K3b ``omni_select``.

Vectors are per-token scores (NumPy or torch); they are handed to the kernel
as ``block_size = 1`` column masses, so the same kernel that runs the 64K
probe path (block-constant scores) computes token-exact kurtosis, budget and
top-b here, in the reference's arithmetic order (module docstring of
``csrc/select.cu``): bit-exact with the reference on identical vectors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .errors import IntegrityError, ParameterError

STOCHASTIC_ATOL = 1e-6


@dataclass
class KeyScores:
    """Per-head accumulated key mass and kurtosis (kv_select.py:23-36)."""

    scores: list
    kurtoses: list

    @property
    def num_heads(self) -> int:
        return len(self.scores)

    @property
    def num_keys(self) -> int:
        return int(np.asarray(self.scores[0]).shape[0])


@dataclass
class SelectionResult:
    """kv_select.py:39-46."""

    budget: int
    selected: list
    flattest_head: int


def _mass(vectors) -> torch.Tensor:
    arr = np.stack([np.asarray(v.cpu() if isinstance(v, torch.Tensor) else v, dtype=np.float64) for v in vectors])
    return torch.from_numpy(arr).to("cuda")


def _run(vectors, p=0.5, budget_override=0, granularity="token", block=1, vision_limit=-1):
    m = _mass(vectors)
    h, n = m.shape
    if block > 1:  # block granularity needs block masses: reduce token scores per block first
        raise ParameterError("use select_top_blocks for block granularity")
    sel = ops.select(m, h, n, 1, p, granularity, vision_limit, budget_override)
    info = sel.info.cpu().numpy()
    stats = sel.stats.cpu().numpy()
    return sel, info, stats


def key_scores_from_vectors(vectors) -> KeyScores:
    """Kurtosis per head (kv_select.py:49-53) on the GPU."""
    for v in vectors:
        if np.asarray(v).size < 2:
            raise ParameterError("kurtosis needs at least 2 samples")
    _, info, stats = _run(vectors)
    return KeyScores([np.asarray(v, dtype=np.float64) for v in vectors], list(stats[: len(vectors)]))


def accumulated_key_scores(attn_matrices) -> KeyScores:
    """Column sums of row-stochastic maps (kv_select.py:56-73) with the
    reference's integrity checks."""
    vecs = []
    for i, a in enumerate(attn_matrices):
        a = torch.as_tensor(np.asarray(a, dtype=np.float64)).to("cuda")
        rs = a.sum(dim=1)
        dev = (rs - 1.0).abs()
        if float(dev.max()) > STOCHASTIC_ATOL:
            worst = int(dev.argmax())
            raise IntegrityError(f"head {i} attention row {worst} sums to {float(rs[worst]):.9f}, not 1")
        if float(a.min()) < 0.0:
            raise IntegrityError(f"head {i} attention has negative entries")
        vecs.append(a.sum(dim=0).cpu().numpy())
    return key_scores_from_vectors(vecs)


def flattest_head(scores: KeyScores) -> int:
    """argmin kurtosis, ties to the lowest index (kv_select.py:76-80)."""
    if scores.num_heads < 1:
        raise ParameterError("need at least one head")
    return int(np.argmin(np.asarray(scores.kurtoses, dtype=np.float64)))


def budget_with_retained_mass(a_star, p: float, total_mass: float | None = None) -> tuple:
    """kv_select.py:104-120: (b, retained, total) from the GPU budget search."""
    if not 0.0 < p <= 1.0:
        raise ParameterError(f"retention p must be in (0, 1], got {p}")
    if total_mass is not None:
        raise ParameterError("explicit total_mass is not supported on the GPU path (the pipeline uses the actual sum)")
    _, info, stats = _run([a_star], p=p)
    return int(info[0]), float(stats[1]), float(stats[2])


def determine_budget(a_star, p: float, total_mass: float | None = None) -> int:
    """kv_select.py:87-101."""
    return budget_with_retained_mass(a_star, p, total_mass)[0]


def top_b_indices(a, b: int) -> np.ndarray:
    """kv_select.py:123-127: ascending indices of the b largest, ties to the
    lower index."""
    n = np.asarray(a).shape[0]
    if not 1 <= b <= n:
        raise ParameterError(f"budget must be in [1, {n}], got {b}")
    sel, info, _ = _run([a], budget_override=b)
    return sel.selected[0, :b].cpu().numpy().astype(np.int64)


def build_key_masks(scores: KeyScores, budget: int) -> SelectionResult:
    """kv_select.py:130-144."""
    n = scores.num_keys
    if not 1 <= budget <= n:
        raise ParameterError(f"budget must be in [1, {n}], got {budget}")
    sel, info, _ = _run(scores.scores, budget_override=budget)
    s = sel.selected.cpu().numpy()
    return SelectionResult(budget, [s[g, :budget].astype(np.int64) for g in range(scores.num_heads)],
                           flattest_head(scores))


def select_vision_keys(scores: KeyScores, budget: int, n_vision: int) -> SelectionResult:
    """kv_select.py:179-195: top keys inside the vision span, b capped."""
    if n_vision < 1:
        raise ParameterError("vision span is empty")
    b = min(budget, n_vision)
    if b < 1:
        raise ParameterError(f"budget must be positive, got {budget}")
    sel, info, _ = _run(scores.scores, budget_override=b, vision_limit=n_vision)
    s = sel.selected.cpu().numpy()
    return SelectionResult(b, [s[g, :b].astype(np.int64) for g in range(scores.num_heads)], flattest_head(scores))


def select_top_blocks(scores: KeyScores, budget: int, block_size: int) -> SelectionResult:
    """kv_select.py:147-176: whole blocks ranked by summed token mass (ties to
    the lower block), the marginal block contributing its lowest indices —
    exactly ``budget`` keys per head. Block sums (np.add.reduceat order),
    ranking and the block table all run on the GPU (omni_block_sums,
    omni_top_blocks)."""
    n = scores.num_keys
    if not 1 <= budget <= n:
        raise ParameterError(f"budget must be in [1, {n}], got {budget}")
    if block_size < 1:
        raise ParameterError(f"block size must be >= 1, got {block_size}")
    h = scores.num_heads
    bm = ops.block_sums(_mass(scores.scores), block_size)  # np.add.reduceat order, on the device
    sel, _ = ops.top_blocks(bm, n, block_size, budget)
    s = sel.cpu().numpy()
    return SelectionResult(budget, [s[g, :budget].astype(np.int64) for g in range(h)], flattest_head(scores))


def sparsity_gap(scores: KeyScores, p: float) -> float:
    """kv_select.py:198-210: (b_flattest - b_sharpest) / N with each head's
    individual budget at retention ``p``."""
    if scores.num_heads < 2:
        raise ParameterError("sparsity gap needs at least two heads")
    flat = flattest_head(scores)
    sharp = int(np.argmax(scores.kurtoses))
    return (determine_budget(scores.scores[flat], p) - determine_budget(scores.scores[sharp], p)) / scores.num_keys
