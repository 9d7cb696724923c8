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
    # optional output buffer [Hq, N, d] bf16 whose lazy rows the selection's
    # K2 already zeroed (select_device(..., O_zero=out)): the forward then
    # writes only the active rows instead of zero-filling the whole output
    out: torch.Tensor | None = None


class SparseAttentionFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, Q, K, V, plan: SparsePlan):
        hq, n, d = Q.shape
        cap = ops.round_up(n, ops.TILE)
        Qb, Kb, Vb = (x.detach().to(torch.bfloat16).contiguous() for x in (Q, K, V))
        K_sel = ops.gather_rows(Kb, plan.selected, plan.sel_counts, cap, ops.TILE)
        V_sel = ops.gather_rows(Vb, plan.selected, plan.sel_counts, cap, ops.TILE)
        O = plan.out if plan.out is not None else torch.zeros_like(Qb)
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
        # compacted key gradients back to their original positions in the
        # leaves' dtype, the sink row's extra dV folded in before rounding
        # (device counts: no host round trip)
        def key_grad(src, dt, **kw):
            tgt = dt if dt in (torch.float32, torch.bfloat16) else torch.float32
            out = torch.zeros(hkv, n, Qb.shape[2], device=Qb.device, dtype=tgt)
            return ops.scatter_key_grads(src, plan.selected, plan.sel_counts, out, **kw).to(dt)

        dK = key_grad(dKs, kd)
        dV = key_grad(dVs, vd, sink_index=plan.sink_index, sink_add=dVsink)
        return dQ.to(qd), dK, dV, None


def plan_from_selection(active_rows, counts, selection, sink_index: int, out: torch.Tensor | None = None) -> SparsePlan:
    return SparsePlan(active_rows, counts, selection.selected, selection.counts, sink_index, out)


def sparse_attention(Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, n_vision: int,
                     cfg: SparsityConfig = SparsityConfig()) -> torch.Tensor:
    """Differentiable OmniSparse attention for a training step: selection
    under no_grad, then the tcgen05 forward with a K5 backward."""
    check_qkv(Q, K, V)
    # the output buffer's lazy rows are zeroed by K2 during the selection
    out = torch.empty(Q.shape, device=Q.device, dtype=torch.bfloat16)
    with torch.no_grad():
        _, _, _, _, _, _, rows, counts, _, sel = select_device(Q.detach(), K.detach(), n_vision, cfg, O_zero=out)
    return SparseAttentionFn.apply(Q, K, V, plan_from_selection(rows, counts, sel, cfg.sink_index, out))
