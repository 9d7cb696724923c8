"""Training path: sparse attention as a torch.autograd.Function (K4 forward,
K5 backward). Selection (query masks, budget, top-b) is non-differentiable
and runs under no_grad, exactly as the reference's selection is a
preprocessing step of ``sparse_prefill`` (prefill.py:161-169)."""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import ops
from .pipeline import SparsityConfig, check_qkv, select_device


@dataclass
class SparsePlan:
    """Device-resident masks and index sets one attention call consumes."""

    rows: torch.Tensor        # i32 [Hq, N]
    counts: torch.Tensor      # i32 [Hq]
    selected: torch.Tensor    # i32 [Hkv, N]
    sel_counts: torch.Tensor  # i32 [Hkv]
    sink_index: int


class SparseAttentionFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, Q, K, V, plan: SparsePlan):
        hq, n, d = Q.shape
        cap = ops.round_up(n, ops.TILE)
        Qb, Kb, Vb = (x.detach().to(torch.bfloat16).contiguous() for x in (Q, K, V))
        K_sel = ops.gather_rows(Kb, plan.selected, plan.sel_counts, cap, ops.TILE)
        V_sel = ops.gather_rows(Vb, plan.selected, plan.sel_counts, cap, ops.TILE)
        O = torch.zeros_like(Qb)
        lse = torch.empty(hq, n, device=Q.device, dtype=torch.float32)
        ops.sparse_attn_fwd(Qb, K_sel, V_sel, Vb, plan.rows, plan.counts, plan.selected, plan.sel_counts,
                            plan.sink_index, O, lse)
        ctx.save_for_backward(Qb, K_sel, V_sel, O, lse)
        ctx.plan = plan
        ctx.dtypes = (Q.dtype, K.dtype, V.dtype)
        return O.to(Q.dtype)

    @staticmethod
    def backward(ctx, dO):
        Qb, K_sel, V_sel, O, lse = ctx.saved_tensors
        plan = ctx.plan
        hkv = K_sel.shape[0]
        n = Qb.shape[1]
        qd, kd, vd = ctx.dtypes
        dQ, dKs, dVs, dVsink = ops.sparse_attn_bwd(Qb, K_sel, V_sel, O, dO.to(torch.bfloat16).contiguous(), lse,
                                                   plan.rows, plan.counts, plan.selected, plan.sel_counts,
                                                   dq_dtype=torch.bfloat16 if qd == torch.bfloat16 else torch.float32)
        # compacted key gradients back to their original positions (device
        # counts: no host round trip)
        dK = ops.scatter_rows(dKs, plan.selected, plan.sel_counts,
                              torch.zeros(hkv, n, Qb.shape[2], device=Qb.device, dtype=torch.float32))
        dV = ops.scatter_rows(dVs, plan.selected, plan.sel_counts, torch.zeros_like(dK))
        dV[:, plan.sink_index] += dVsink
        return dQ.to(qd), dK.to(kd), dV.to(vd), None


def plan_from_selection(active_rows, counts, selection, sink_index: int) -> SparsePlan:
    return SparsePlan(active_rows, counts, selection.selected, selection.counts, sink_index)


def sparse_attention(Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, n_vision: int,
                     cfg: SparsityConfig = SparsityConfig()) -> torch.Tensor:
    """Differentiable OmniSparse attention for a training step: selection
    under no_grad, then the tcgen05 forward with a K5 backward."""
    check_qkv(Q, K, V)
    with torch.no_grad():
        _, _, _, _, _, _, rows, counts, _, sel = select_device(Q.detach(), K.detach(), n_vision, cfg)
    return SparseAttentionFn.apply(Q, K, V, plan_from_selection(rows, counts, sel, cfg.sink_index))
