"""Accounting and reporting (reference ``metrics.py``): attention recall on the
GPU, the closed-form multiply-add and KV models, and the JSON report (schema
version 1) tying a run together.

Recall without attention maps. The reference measures recall as the share of
the dense causal attention mass of the active rows that lands on the selected
keys (``metrics.py:26-39``), which needs every N x N map. Per row that share
is exp(LSE_sel - LSE_all): LSE_sel is the log normaliser over the row's
visible selected keys (the sparse kernel K4 emits it as a side output) and
LSE_all the one over all of the row's causal keys — the same kernel run with
the identity selection. ``attention_recall_device`` therefore costs one extra
K4 launch over all keys (dense work on the active rows only) and never forms a
map; heads with no active rows recall 1.0 (reference convention).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import Any

import torch

from . import ops
from .errors import ParameterError

SCHEMA_VERSION = 1
VALUE_BYTES = 8  # the reference's float64 flat memory model (bytes = values x 8)


def attention_recall_device(res, Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, sink_index: int = 0
                            ) -> torch.Tensor:
    """Per-Q-head recall (float64 [Hq]) of a ``pipeline.DevicePrefill``.

    Q [Hq, N, 128], K / V [Hkv, N, 128] bf16 on the GPU (the prefill inputs)."""
    hq, n, d = Q.shape
    hkv = K.shape[0]
    cap = ops.round_up(n, ops.TILE)
    ident = torch.arange(n, device=Q.device, dtype=torch.int32).repeat(hkv, 1).contiguous()
    cnt = torch.full((hkv,), n, device=Q.device, dtype=torch.int32)
    K_all = ops.gather_rows(K, ident, cnt, cap, ops.TILE)
    V_all = ops.gather_rows(V, ident, cnt, cap, ops.TILE)
    O_tmp = torch.empty_like(Q)
    lse_all = torch.empty(hq, n, device=Q.device, dtype=torch.float32)
    ops.sparse_attn_fwd(Q, K_all, V_all, V, res.rows, res.counts, ident, cnt, sink_index, O_tmp, lse_all)
    act = res.active.bool()
    share = torch.exp(res.lse.double() - lse_all.double())  # rows with no visible selected key: exp(-inf) = 0
    share = torch.where(act, share, torch.zeros_like(share))
    n_act = act.sum(dim=1)
    rec = share.sum(dim=1) / n_act.clamp(min=1).double()
    return torch.where(n_act > 0, rec, torch.ones_like(rec))


def sparsity_gap_device(mass: torch.Tensor, selection, n_kv_heads: int, seq_len: int, block_size: int,
                        p: float) -> float:
    """kv_select.py:198-210 under rule B: (b_flattest - b_sharpest) / N, each
    group's individual budget at retention ``p``. The sharpest group is the
    argmax of the kurtoses K3b already produced (ties to the lowest index, as
    np.argmax); each budget is K3b run on that group's Q heads alone, so it
    is the same arithmetic that set the shared budget. ``mass`` is the
    per-Q-head column mass the selection consumed ([Hq, nb]; nb = N is the
    exact / token path, block size 1)."""
    if n_kv_heads < 2:
        raise ParameterError("sparsity gap needs at least two heads")
    hq = mass.shape[0]
    rep = hq // n_kv_heads
    bs = 1 if mass.shape[1] == seq_len else block_size
    kurt = selection.stats[:n_kv_heads].cpu().tolist()
    flat = int(selection.info[1])
    sharp = max(range(n_kv_heads), key=lambda g: (kurt[g], -g))

    def own_budget(g: int) -> int:
        sub = mass[g * rep:(g + 1) * rep].contiguous()
        return int(ops.select(sub, 1, seq_len, bs, p, "token").info[0])

    return (own_budget(flat) - own_budget(sharp)) / seq_len


@dataclass(frozen=True)
class FlopsBreakdown:
    """Multiply-add counts of the full, sparse and probe paths."""

    full: int
    sparse: int
    probe_overhead: int

    @property
    def reduction(self) -> float:
        return 1.0 - (self.sparse + self.probe_overhead) / self.full


def analytic_flops(n_tokens: int, n_vision: int, head_dim: int, active_per_head: list, budget: int,
                   block_size: int | None = None, probe_scores: bool = False) -> FlopsBreakdown:
    """The reference's closed-form multiply-add model (metrics.py:55-81):
    dense QK^T + AV over the full N x N rectangle per head; sparse the same
    over active rows x budget keys; probe = the two classification logits per
    vision query, plus (block probe) pooling of Q and K and the pooled product."""
    heads = len(active_per_head)
    full = heads * 2 * n_tokens * n_tokens * head_dim
    sparse = 2 * budget * head_dim * sum(int(a) for a in active_per_head)
    probe = heads * 2 * n_vision * head_dim
    if probe_scores:
        if block_size is None:
            raise ValueError("probe accounting needs the block size")
        n_blocks = -(-n_tokens // block_size)
        probe += heads * (2 * n_tokens * head_dim + n_blocks * n_blocks * head_dim)
    return FlopsBreakdown(full, sparse, probe)


@dataclass(frozen=True)
class KVReduction:
    """Vision-segment residency and per-step fetch savings."""

    resident_reduction: float
    fetch_reduction: float
    predicted_vision_tokens: int
    predicted_vision_bytes: int


def kv_reduction(n_vision: int, budget: int, head_dim: int, active_head_steps: int, total_head_steps: int
                 ) -> KVReduction:
    """metrics.py:94-120: residency falls by 1 - b/Nv; fetches additionally by
    the active head-step fraction; byte predictions at VALUE_BYTES per value
    (K and V rows)."""
    if budget > n_vision:
        raise ValueError(f"budget {budget} exceeds vision span {n_vision}")
    frac = active_head_steps / total_head_steps if total_head_steps else 0.0
    tokens = budget * active_head_steps
    return KVReduction(resident_reduction=1.0 - budget / n_vision,
                       fetch_reduction=1.0 - (budget / n_vision) * frac,
                       predicted_vision_tokens=tokens,
                       predicted_vision_bytes=tokens * 2 * head_dim * VALUE_BYTES)


_REPORT_FIELDS = ("mode", "config", "workload", "flops_full", "flops_sparse", "flops_probe_overhead",
                  "flops_reduction", "exponentials_full", "exponentials_sparse", "recall_per_head", "recall_min",
                  "recall_flattest", "flattest_retained_mass", "flattest_total_mass", "budget", "flattest_head",
                  "lazy_query_fraction", "sparsity_gap", "kv_resident_reduction", "kv_fetch_reduction",
                  "lazy_head_fraction_decode", "decode")


@dataclass
class MetricsReport:
    """One run's report, JSON schema version 1 (reference metrics.py:122-196):
    same field names, same defaults, same sorted-key serialisation."""

    mode: str
    config: dict
    workload: dict
    flops_full: int
    flops_sparse: int
    flops_probe_overhead: int
    flops_reduction: float
    exponentials_full: int
    exponentials_sparse: int
    recall_per_head: list
    recall_min: float
    recall_flattest: float
    flattest_retained_mass: float
    flattest_total_mass: float
    budget: int
    flattest_head: int
    lazy_query_fraction: float
    sparsity_gap: float | None
    kv_resident_reduction: float | None = None
    kv_fetch_reduction: float | None = None
    lazy_head_fraction_decode: float | None = None
    decode: dict | None = None
    schema_version: int = SCHEMA_VERSION

    def to_dict(self) -> dict[str, Any]:
        d = {"schema_version": self.schema_version}
        d.update({k: getattr(self, k) for k in _REPORT_FIELDS})
        return d

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True, indent=2) + "\n"

    @classmethod
    def from_dict(cls, d: dict[str, Any]) -> "MetricsReport":
        d = dict(d)
        version = d.pop("schema_version")
        if version != SCHEMA_VERSION:
            raise ValueError(f"unsupported report schema {version}")
        return cls(schema_version=version, **d)

    @classmethod
    def from_json(cls, text: str) -> "MetricsReport":
        return cls.from_dict(json.loads(text))


def prefill_report(res, Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, n_vision: int, cfg,
                   with_recall: bool = True) -> MetricsReport:
    """MetricsReport of a device prefill (``pipeline.DevicePrefill``): the
    analytic model on its masks and budget, GPU recall per Q head, and the
    flattest group's retained / total mass (GQA rule B: the flattest entry is
    a KV group; recall_flattest is its retained share, as on the exact path)."""
    hq, n, d = Q.shape
    hkv = K.shape[0]
    info = res.selection.info.cpu().tolist()
    stats = res.selection.stats.cpu().tolist()
    b, flat = int(info[0]), int(info[1])
    active = res.active.bool()
    act_per_head = active.sum(dim=1).cpu().tolist()
    fl = analytic_flops(n, n_vision, d, act_per_head, b, block_size=cfg.block_size, probe_scores=True)
    rec = attention_recall_device(res, Q, K, V, cfg.sink_index).cpu().tolist() if with_recall else [1.0] * hq
    retained, total = float(stats[hkv]), float(stats[hkv + 1])
    return MetricsReport(
        mode="sparse",
        config={"tau": cfg.tau, "p": cfg.p, "block_size": cfg.block_size, "granularity": cfg.granularity,
                "preserve_first_head": cfg.preserve_first_head, "score_source": "probe"},
        workload={"heads": hq, "kv_heads": hkv, "head_dim": d, "n_tokens": n, "n_vision": n_vision,
                  "n_text": n - n_vision},
        flops_full=fl.full, flops_sparse=fl.sparse, flops_probe_overhead=fl.probe_overhead,
        flops_reduction=fl.reduction,
        exponentials_full=hq * n * (n + 1) // 2,
        exponentials_sparse=int(sum(act_per_head)) * b,
        recall_per_head=rec, recall_min=min(rec),
        recall_flattest=retained / total if total > 0 else 1.0,
        flattest_retained_mass=retained, flattest_total_mass=total, budget=b, flattest_head=flat,
        lazy_query_fraction=1.0 - float(active[:, :n_vision].float().mean()) if n_vision else 0.0,
        sparsity_gap=sparsity_gap_device(res.block_mass, res.selection, hkv, n, cfg.block_size, cfg.p)
        if hkv >= 2 else None)
