"""Gradient oracle for the sparse attention forward (tests only).

The reference has no autograd (``SPEC.md`` numerics non-goals: "auto-
differentiation"), so gradient parity is unpinned by the reference. This is a
float64 torch-autograd restatement of ``prefill.py:89-122``: gather active rows
and selected keys, staircase mask in original positions, softmax renormalised
over visible keys, times V_sel; rows with no visible key copy ``v[sink]``
(so their gradient flows into ``dV[sink]``); lazy rows are constant zero.
Its forward is pinned to :func:`oracle.attention.sparse_head_attention`
(tests/test_oracle_golden.py), and its gradients are the oracle for the
backward kernel.
"""

from __future__ import annotations

import numpy as np
import torch


def sparse_attention_t(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, selected, active, sink_index: int,
                       rows_subset=None) -> torch.Tensor:
    """Differentiable f64 forward for one Q head over its group's K/V."""
    sel = torch.as_tensor(np.asarray(selected, dtype=np.int64))
    rows = np.flatnonzero(np.asarray(active, dtype=bool))
    if rows_subset is not None:
        rows = np.intersect1d(rows, np.asarray(rows_subset, dtype=np.int64))
    rows_t = torch.as_tensor(rows)
    out = torch.zeros_like(v)
    if rows.size == 0 or sel.numel() == 0:
        return out + 0.0 * (q.sum() + k.sum() + v.sum())
    s = (q[rows_t] @ k[sel].T) * (1.0 / np.sqrt(q.shape[1]))
    vis = sel[None, :] <= rows_t[:, None]
    alive = vis.any(dim=1)
    s = s.masked_fill(~vis, float("-inf"))
    s = torch.where(alive[:, None], s, torch.zeros_like(s))
    p = torch.softmax(s, dim=1) * alive[:, None]
    o = p @ v[sel]
    o = torch.where(alive[:, None], o, v[sink_index].expand_as(o))
    return out.index_copy(0, rows_t, o)


def sparse_attention_grads(Q, K, V, selected_per_group, active, sink_index: int, dO, rows_subset=None):
    """Gradients of sum(O * dO) w.r.t. Q [Hq,N,d], K/V [Hkv,N,d] (f64 numpy),
    rule-B grouping (Q head h uses group h // rep)."""
    hq, hkv = len(Q), len(K)
    rep = hq // hkv
    q = torch.tensor(np.asarray(Q, dtype=np.float64), requires_grad=True)
    k = torch.tensor(np.asarray(K, dtype=np.float64), requires_grad=True)
    v = torch.tensor(np.asarray(V, dtype=np.float64), requires_grad=True)
    go = torch.tensor(np.asarray(dO, dtype=np.float64))
    total = 0.0
    outs = []
    for h in range(hq):
        g = h // rep
        o = sparse_attention_t(q[h], k[g], v[g], selected_per_group[g], active[h], sink_index, rows_subset)
        outs.append(o.detach().numpy())
        total = total + (o * go[h]).sum()
    total.backward()
    return np.stack(outs), q.grad.numpy(), k.grad.numpy(), v.grad.numpy()
