"""Multi-GPU sharding (one process per GPU, torch.distributed): head-sharded
prefill and training, sequence-sharded decode.

SURVEY §8e: work shards by KV group. A rank owns a contiguous range of KV
groups (world <= Hkv) or a contiguous slice of one group's Q heads (world >
Hkv, e.g. 8 GPUs over 4 groups: 3 + 4 Q heads per rank with the group's K/V
replicated). K1/K2/K3a run locally; the only exchange is ONE all_gather of
the per-Q-head block column masses (28 x nb x 8 B = 57 KB at 64K), after
which every rank redundantly runs the selection (flattest group, budget,
top-b) on identical inputs in canonical head order — bit-identical to the
single-GPU path. A per-rank all-reduce(max) of budgets would be wrong: the
budget is the FLATTEST group's b (kv_select.py:76-80), not the largest.

Training (SURVEY §8e "Training backward"): the same head sharding; dQ stays
with its Q head and dK / dV with the rank owning the KV group. When a group
is split across ranks (world > Hkv: 8 GPUs over 4 groups), each rank's dK /
dV of that group is a partial sum over its own Q heads, so the group's ranks
all-reduce it once (``kv_grad_group`` + ``ReduceGradOverGroup``).

Decode: sequences shard contiguously across ranks (C5: 32
sequences, 4 per GPU at 8 GPUs); each rank decodes its own sequences from its
own slim caches with no collective; ``gather_decode_outputs`` reassembles a
step's outputs where a caller needs them in one place.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import ops
from .errors import ShapeError
from .pipeline import DevicePrefill, SparsityConfig, check_qkv


@dataclass(frozen=True)
class ShardPlan:
    q_start: int
    q_stop: int
    g_start: int
    g_stop: int
    n_q_heads: int
    n_kv_heads: int

    @property
    def q_heads(self) -> int:
        return self.q_stop - self.q_start

    @property
    def kv_groups(self) -> int:
        return self.g_stop - self.g_start


def shard_plan(n_q_heads: int, n_kv_heads: int, world: int, rank: int) -> ShardPlan:
    """Contiguous head ranges per rank (rule-B groups never straddle ranks
    unless world > Hkv, in which case each group spans world / Hkv ranks)."""
    if n_q_heads % n_kv_heads:
        raise ShapeError("n_q_heads must be a multiple of n_kv_heads")
    rep = n_q_heads // n_kv_heads
    if world <= n_kv_heads:
        if n_kv_heads % world:
            raise ShapeError(f"{n_kv_heads} KV groups do not split over {world} ranks")
        per = n_kv_heads // world
        g0 = rank * per
        return ShardPlan(g0 * rep, (g0 + per) * rep, g0, g0 + per, n_q_heads, n_kv_heads)
    if world % n_kv_heads:
        raise ShapeError(f"world {world} must be a multiple of {n_kv_heads} KV groups")
    per_group = world // n_kv_heads
    if per_group > rep:
        raise ShapeError("more ranks per group than Q heads in the group")
    g = rank // per_group
    part = rank % per_group
    base, extra = divmod(rep, per_group)
    # the extra heads go to the LAST parts of a group: the first part of
    # group 0 holds Q head 0, which preserve_first_head keeps fully active
    # (about twice a lazy-masked head's work), so it takes one head fewer
    # (8 GPUs, 28/4 heads: 3 + 4 per group, max per-rank work 4 head-units
    # instead of 5)
    lead = per_group - extra
    start = part * base + max(0, part - lead)
    stop = start + base + (1 if part >= lead else 0)
    return ShardPlan(g * rep + start, g * rep + stop, g, g + 1, n_q_heads, n_kv_heads)


def gather_block_mass(local: torch.Tensor, plan: ShardPlan, world: int, group=None) -> torch.Tensor:
    """all_gather of the per-Q-head block column masses into [Hq, nb] in
    global head order (works on gloo/CPU and NCCL/CUDA tensors)."""
    nb = local.shape[1]
    plans = [shard_plan(plan.n_q_heads, plan.n_kv_heads, world, r) for r in range(world)]
    width = max(p.q_heads for p in plans)
    buf = torch.zeros(width, nb, dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    full = torch.empty(plan.n_q_heads, nb, dtype=local.dtype, device=local.device)
    for p, t in zip(plans, parts):
        full[p.q_start:p.q_stop] = t[: p.q_heads]
    return full


def select_sharded(Q_loc: torch.Tensor, K_loc: torch.Tensor, plan: ShardPlan, n_vision: int, world: int,
                   cfg: SparsityConfig = SparsityConfig(), O_zero: torch.Tensor | None = None, group=None):
    """This rank's masks + the replicated global selection: K1/K2/K3a on the
    local heads, one all_gather of block masses, K3b on every rank.
    Returns (k_lazy, k_act, pooled_k, active, pooled_q, rows, counts, mass,
    selection, local selected index lists, local counts)."""
    n = Q_loc.shape[1]
    k_lazy, k_act, pk = ops.kv_probe(K_loc, n_vision, cfg.sink_index, cfg.block_size)
    preserve = cfg.preserve_first_head and plan.q_start == 0  # only global head 0 is preserved
    active, _, pq, bact = ops.q_score(Q_loc, k_lazy, k_act, n_vision, cfg.tau, preserve, cfg.block_size,
                                      O_zero=O_zero)
    rows, counts = ops.compact_rows(active, bact, cfg.block_size)
    mass_loc = ops.probe_mass(pq, pk)
    mass = gather_block_mass(mass_loc, plan, world, group) if world > 1 else mass_loc
    sel = ops.select(mass, plan.n_kv_heads, n, cfg.block_size, cfg.p, cfg.granularity)
    sel_loc = sel.selected[plan.g_start:plan.g_stop]
    cnt_loc = sel.info[4 + plan.g_start: 4 + plan.g_stop]
    return k_lazy, k_act, pk, active, pq, rows, counts, mass, sel, sel_loc, cnt_loc


def sparse_prefill_sharded(Q_loc: torch.Tensor, K_loc: torch.Tensor, V_loc: torch.Tensor, plan: ShardPlan,
                           n_vision: int, world: int, cfg: SparsityConfig = SparsityConfig(),
                           out: torch.Tensor | None = None, group=None) -> DevicePrefill:
    """This rank's share of the sparse prefill: Q_loc = Q[q_start:q_stop],
    K_loc / V_loc = K/V[g_start:g_stop]. Returns outputs for the local Q heads
    plus the (replicated) global selection."""
    check_qkv(Q_loc, K_loc, V_loc)
    hq_l, n, d = Q_loc.shape
    O = out if out is not None else torch.empty_like(Q_loc)
    k_lazy, k_act, pk, active, pq, rows, counts, mass, sel, sel_loc, cnt_loc = select_sharded(
        Q_loc, K_loc, plan, n_vision, world, cfg, O_zero=O, group=group)
    cap = ops.round_up(n, ops.TILE)
    K_sel = ops.gather_rows(K_loc, sel_loc, cnt_loc, cap, ops.TILE)
    V_sel = ops.gather_rows(V_loc, sel_loc, cnt_loc, cap, ops.TILE)
    lse = torch.empty(hq_l, n, device=Q_loc.device, dtype=torch.float32)
    ops.sparse_attn_fwd(Q_loc, K_sel, V_sel, V_loc, rows, counts, sel_loc, cnt_loc, cfg.sink_index, O, lse)
    return DevicePrefill(O, lse, active, rows, counts, sel, k_lazy, k_act, pq, pk, mass, K_sel, V_sel)


# ------------------------------------------------------------------ training
def kv_grad_group(n_q_heads: int, n_kv_heads: int, world: int, rank: int):
    """The process group of the ranks that share this rank's KV group when
    groups are split across ranks (world > Hkv), else None. Every rank must
    call it (dist.new_group is collective), in the same order."""
    if world <= n_kv_heads:
        return None
    per_group = world // n_kv_heads
    mine = None
    for g in range(n_kv_heads):
        ranks = list(range(g * per_group, (g + 1) * per_group))
        pg = dist.new_group(ranks)
        if rank in ranks:
            mine = pg
    return mine


class ReduceGradOverGroup(torch.autograd.Function):
    """Identity in the forward pass; the backward all-reduces (sums) the
    gradient over ``group`` — the partial dK / dV of a KV group whose Q
    heads are spread over several ranks."""

    @staticmethod
    def forward(ctx, x, group):
        ctx.group = group
        return x.view_as(x)

    @staticmethod
    def backward(ctx, g):
        g = g.contiguous()
        dist.all_reduce(g, op=dist.ReduceOp.SUM, group=ctx.group)
        return g, None


def sparse_attention_sharded(Q_loc: torch.Tensor, K_loc: torch.Tensor, V_loc: torch.Tensor, plan: ShardPlan,
                             n_vision: int, world: int, cfg: SparsityConfig = SparsityConfig(), group=None,
                             kv_group=None) -> torch.Tensor:
    """Differentiable head-sharded OmniSparse attention (training forward +
    backward on this rank's Q heads): the sharded selection under no_grad,
    then the K4 forward / K5 backward locally; ``kv_group`` (from
    ``kv_grad_group``) reduces a split group's dK / dV."""
    from .autograd import SparseAttentionFn, SparsePlan

    check_qkv(Q_loc, K_loc, V_loc)
    o_buf = torch.empty(Q_loc.shape, device=Q_loc.device, dtype=torch.bfloat16)  # lazy rows zeroed by K2
    with torch.no_grad():
        out = select_sharded(Q_loc.detach(), K_loc.detach(), plan, n_vision, world, cfg, O_zero=o_buf, group=group)
    rows, counts, sel_loc, cnt_loc = out[5], out[6], out[9], out[10]
    if kv_group is not None:
        # reduce the split group's partial dK / dV in fp32, before the
        # rounding to the leaves' dtype
        K_loc = ReduceGradOverGroup.apply(K_loc.float(), kv_group)
        V_loc = ReduceGradOverGroup.apply(V_loc.float(), kv_group)
    return SparseAttentionFn.apply(Q_loc, K_loc, V_loc, SparsePlan(rows, counts, sel_loc.contiguous(),
                                                                   cnt_loc.contiguous(), cfg.sink_index, o_buf))


# ------------------------------------------------------------------ decode
def sequence_shard(batch: int, world: int, rank: int) -> range:
    """Contiguous, balanced sequence range of this rank (the first
    batch % world ranks take one sequence more)."""
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def gather_decode_outputs(out_loc: torch.Tensor, batch: int, world: int, group=None) -> torch.Tensor:
    """all_gather of the ranks' decode outputs [B_r, Hq, d] into [B, Hq, d]
    in sequence order (works on gloo/CPU and NCCL/CUDA tensors)."""
    width = max(len(sequence_shard(batch, world, r)) for r in range(world))
    buf = torch.zeros((width,) + tuple(out_loc.shape[1:]), dtype=out_loc.dtype, device=out_loc.device)
    buf[: out_loc.shape[0]] = out_loc
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[: len(sequence_shard(batch, world, r))] for r, p in enumerate(parts)])
