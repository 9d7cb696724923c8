"""Attention recall in float64 (oracle; tests only).

Restates ``metrics.py:26-39`` (``attention_recall``): the share of the dense
attention mass of the active query rows that lands on the selected keys;
a head with no active rows recalls 1.0.
"""

from __future__ import annotations

import numpy as np

from .attention import causal_attention


def attention_recall(full_attention, selected, active=None) -> float:
    """metrics.py:26-39 on an explicit map."""
    a = np.asarray(full_attention, dtype=np.float64)
    if active is not None:
        a = a[np.asarray(active, dtype=bool)]
    if a.shape[0] == 0:
        return 1.0
    return float(a[:, np.asarray(selected, dtype=np.int64)].sum()) / float(a.sum())


def head_recall(q, k, selected, active) -> float:
    """Recall of one head from Q / K (dense causal map, small N)."""
    a, _ = causal_attention(q, k, k)
    return attention_recall(a, selected, active)
