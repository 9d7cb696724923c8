"""Row kernels in float64 (oracle; test infrastructure only).

Restates the reference kernel core contract: ``_core_py.py:13-44`` /
``_core_cy.pyx:17-113`` behind the validating wrappers of
``kernels.py:73-139``.
"""

from __future__ import annotations

import numpy as np

from paper_2511_12201_b200.errors import DegenerateRowError, ParameterError, ShapeError


def f64(x) -> np.ndarray:
    """Upcast to a C-contiguous float64 array (the reference's only precision,
    SURVEY §0 pitfall: fp32/bf16 values must reach the oracle as f64)."""
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """``kernels.py:73-81``: shape-checked dense product."""
    if a.shape[1] != b.shape[0]:
        raise ShapeError(f"matmul shapes incompatible: {a.shape} @ {b.shape}")
    out = a @ b
    if not np.isfinite(out).all():
        raise ParameterError("non-finite values after matmul")
    return out


def softmax_rows(m: np.ndarray, mask: np.ndarray | None = None) -> np.ndarray:
    """``kernels.py:84-112`` + ``_core_py.py:13-22``.

    Max-subtracted softmax over unmasked cells; masked cells are exactly 0; a
    row with no unmasked cell raises DegenerateRowError.
    """
    m = f64(m)
    if m.shape[1] == 0:
        raise DegenerateRowError("softmax over zero columns")
    if mask is None:
        e = np.exp(m - m.max(axis=1, keepdims=True))
        return e / e.sum(axis=1, keepdims=True)
    mask = np.asarray(mask, dtype=bool)
    if mask.shape != m.shape:
        raise ShapeError(f"mask shape {mask.shape} does not match matrix {m.shape}")
    alive = mask.any(axis=1)
    if not alive.all():
        raise DegenerateRowError(f"softmax row {int(np.flatnonzero(~alive)[0])} is fully masked")
    held = np.where(mask, m, -np.inf)
    e = np.exp(held - held.max(axis=1, keepdims=True))
    e[~mask] = 0.0
    return e / e.sum(axis=1, keepdims=True)


def block_lengths(n: int, block: int) -> np.ndarray:
    """``block_probe.py:36-41``: true lengths of the ceil(n/B) blocks."""
    nb = -(-n // block)
    lens = np.full(nb, block, dtype=np.int64)
    if n % block:
        lens[-1] = n % block
    return lens


def mean_pool_rows(m: np.ndarray, block: int) -> np.ndarray:
    """``kernels.py:115-122`` + ``_core_py.py:25-30``: block means, short tail
    averaged over its true length."""
    if block < 1:
        raise ParameterError(f"pooling block must be >= 1, got {block}")
    m = f64(m)
    starts = np.arange(0, m.shape[0], block)
    lens = block_lengths(m.shape[0], block).astype(np.float64)
    return np.add.reduceat(m, starts, axis=0) / lens[:, None]


def kurtosis(v: np.ndarray) -> float:
    """``kernels.py:125-134`` + ``_core_py.py:33-40``: Pearson m4/m2^2 with 1/n
    moments; zero variance -> 0.0."""
    v = f64(v).ravel()
    if v.size < 2:
        raise ParameterError(f"kurtosis needs at least 2 samples, got {v.size}")
    d = v - v.mean()
    m2 = float(np.mean(d * d))
    if m2 == 0.0:
        return 0.0
    m4 = float(np.mean(d * d * d * d))
    return m4 / (m2 * m2)


def colsum(m: np.ndarray) -> np.ndarray:
    """``kernels.py:137-139`` + ``_core_py.py:43-44``."""
    return f64(m).sum(axis=0)
