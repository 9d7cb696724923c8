"""Head-sharded multi-GPU prefill (one process per GPU, torch.distributed).

SURVEY §8e: work shards by KV group. A rank owns a contiguous range of KV
groups (world <= Hkv) or a contiguous slice of one group's Q heads (world >
Hkv, e.g. 8 GPUs over 4 groups: 3 + 4 Q heads per rank with the group's K/V
replicated). K1/K2/K3a run locally; the only exchange is ONE all_gather of
the per-Q-head block column masses (28 x nb x 8 B = 57 KB at 64K), after
which every rank redundantly runs the selection (flattest group, budget,
top-b) on identical inputs in canonical head order — bit-identical to the
single-GPU path. A per-rank all-reduce(max) of budgets would be wrong: the
budget is the FLATTEST group's b (kv_select.py:76-80), not the largest.
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


def sparse_prefill_sharded(Q_loc: torch.Tensor, K_loc: torch.Tensor, V_loc: torch.Tensor, plan: ShardPlan,
                           n_vision: int, world: int, cfg: SparsityConfig = SparsityConfig(),
                           out: torch.Tensor | None = None, group=None) -> DevicePrefill:
    """This rank's share of the sparse prefill: Q_loc = Q[q_start:q_stop],
    K_loc / V_loc = K/V[g_start:g_stop]. Returns outputs for the local Q heads
    plus the (replicated) global selection."""
    check_qkv(Q_loc, K_loc, V_loc)
    hq_l, n, d = Q_loc.shape
    O = out if out is not None else torch.empty_like(Q_loc)
    k_lazy, k_act, pk = ops.kv_probe(K_loc, n_vision, cfg.sink_index, cfg.block_size)
    preserve = cfg.preserve_first_head and plan.q_start == 0  # only global head 0 is preserved
    active, _, pq, bact = ops.q_score(Q_loc, k_lazy, k_act, n_vision, cfg.tau, preserve, cfg.block_size, O_zero=O)
    rows, counts = ops.compact_rows(active, bact, cfg.block_size)
    mass_loc = ops.probe_mass(pq, pk)
    mass = gather_block_mass(mass_loc, plan, world, group) if world > 1 else mass_loc
    sel = ops.select(mass, plan.n_kv_heads, n, cfg.block_size, cfg.p, cfg.granularity)
    sel_loc = sel.selected[plan.g_start:plan.g_stop]
    cnt_loc = sel.info[4 + plan.g_start: 4 + plan.g_stop]
    cap = ops.round_up(n, ops.TILE)
    K_sel = ops.gather_rows(K_loc, sel_loc, cnt_loc, cap, ops.TILE)
    V_sel = ops.gather_rows(V_loc, sel_loc, cnt_loc, cap, ops.TILE)
    lse = torch.empty(hq_l, n, device=Q_loc.device, dtype=torch.float32)
    ops.sparse_attn_fwd(Q_loc, K_sel, V_sel, V_loc, rows, counts, sel_loc, cnt_loc, cfg.sink_index, O, lse)
    return DevicePrefill(O, lse, active, rows, counts, sel, k_lazy, k_act, pq, pk, mass, K_sel, V_sel)
