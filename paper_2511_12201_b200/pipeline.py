"""Device-resident OmniSparse prefill: K1 -> K2 -> compaction -> K3a -> K3b ->
gather -> K4, all on one CUDA stream with no host synchronisation.

This is the composite behind ``prefill.sparse_prefill`` and the benchmark.
It follows the glue of ``prefill.py:160-175`` (minus the always-on dense
oracle and recall instrumentation) under GQA rule B
(DESIGN.md): masks per Q head, probe scores summed per KV group, one budget
from the flattest group, one top-b set per group shared by its Q heads.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import ops
from .errors import LayoutError, ParameterError, ShapeError


@dataclass(frozen=True)
class SparsityConfig:
    """``prefill.py:38-65``: every sparsity knob, validated on construction."""

    tau: float = 0.08
    p: float = 0.82
    block_size: int = 256
    granularity: str = "token"
    preserve_first_head: bool = True
    sink_index: int = 0
    seed: int = 0

    def __post_init__(self):
        if not 0.0 <= self.tau < 1.0:
            raise ParameterError(f"tau must be in [0, 1), got {self.tau}")
        if not 0.0 < self.p <= 1.0:
            raise ParameterError(f"p must be in (0, 1], got {self.p}")
        if self.block_size < 1:
            raise ParameterError(f"block_size must be >= 1, got {self.block_size}")
        if self.granularity not in ("token", "block"):
            raise ParameterError("granularity must be one of ('token', 'block')")


@dataclass
class DevicePrefill:
    """All device tensors of one prefill (outputs + every intermediate)."""

    outputs: torch.Tensor       # bf16 [Hq, N, d]; lazy rows zero
    lse: torch.Tensor           # f32 [Hq, N] softmax normaliser of active rows
    active: torch.Tensor        # u8 [Hq, N]
    rows: torch.Tensor          # i32 [Hq, N] compacted active rows
    counts: torch.Tensor        # i32 [Hq]
    selection: ops.Selection
    k_lazy: torch.Tensor
    k_act: torch.Tensor
    pooled_q: torch.Tensor
    pooled_k: torch.Tensor
    block_mass: torch.Tensor    # f64 [Hq, nb]
    K_sel: torch.Tensor         # bf16 [Hkv, cap, d]
    V_sel: torch.Tensor
    p_act: torch.Tensor | None = None


def check_qkv(Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor) -> None:
    for name, t in (("Q", Q), ("K", K), ("V", V)):
        if not t.is_cuda or t.dim() != 3:
            raise ShapeError(f"{name} must be a CUDA [heads, tokens, dim] tensor")
    if K.shape != V.shape or Q.shape[1:] != K.shape[1:]:
        raise ShapeError(f"Q {tuple(Q.shape)} / K {tuple(K.shape)} / V {tuple(V.shape)} disagree")
    if Q.shape[0] % K.shape[0]:
        raise ShapeError("Q heads must be a multiple of KV heads (GQA rule B)")


def select_device(Q: torch.Tensor, K: torch.Tensor, n_vision: int, cfg: SparsityConfig, want_prob: bool = False,
                  O_zero: torch.Tensor | None = None, score_source: str = "probe"):
    """Masks + key scores + flattest/budget/top-b (no attention).

    score_source "probe" (hot path): block-probe column masses (K3a).
    score_source "exact": column masses of the full causal maps (K3x, O(N^2 d)
    float64) and a token-level selection (the general K3b path)."""
    hq, n, d = Q.shape
    if not 1 <= n_vision <= n:
        raise LayoutError(f"n_vision {n_vision} outside [1, {n}]")
    if not 0 <= cfg.sink_index < n:
        raise LayoutError(f"sink_index {cfg.sink_index} outside the prompt")
    if score_source not in ("exact", "probe"):
        raise ParameterError("score source must be one of ('exact', 'probe')")
    k_lazy, k_act, pk = ops.kv_probe(K, n_vision, cfg.sink_index, cfg.block_size)
    active, p_act, pq, bact = ops.q_score(Q, k_lazy, k_act, n_vision, cfg.tau, cfg.preserve_first_head,
                                          cfg.block_size, want_prob=want_prob, O_zero=O_zero)
    rows, counts = ops.compact_rows(active, bact, cfg.block_size)
    if score_source == "probe":
        mass = ops.probe_mass(pq, pk)
        sel = ops.select(mass, K.shape[0], n, cfg.block_size, cfg.p, cfg.granularity)
    else:
        mass = ops.exact_mass(Q, K)
        sel = ops.select(mass, K.shape[0], n, 1, cfg.p, "token")
        if cfg.granularity == "block":
            # select_top_blocks over the same budget (prefill.py:168-169,
            # kv_select.py:147-176): np.add.reduceat block sums of the
            # token-level group scores, ranked on the device; the key scores
            # and kurtoses stay token-level, as the reference returns them
            blk = ops.block_sums(sel.group_scores, cfg.block_size)
            sel.selected, bcounts = ops.top_blocks(blk, n, cfg.block_size, int(sel.info[0]))
            sel.info[4:] = bcounts
    return k_lazy, k_act, pk, active, p_act, pq, rows, counts, mass, sel


class PrefillStreamer:
    """Host-buffer serving API: pinned host Q/K/V in, host O out, with the
    host<->device copies of neighbouring requests overlapped with compute.

    Request i's H2D copy runs on a copy stream while request i-1 computes and
    request i-2's output drains on a second copy stream (``depth`` device
    buffer sets rotate; depth 3 lets the three stages run concurrently, so the
    period approaches the slowest stage — the H2D copy at PCIe rate). Every
    request still pays its own copies; only their latency is hidden behind
    other requests' kernels."""

    def __init__(self, hq: int, hkv: int, n: int, d: int, n_vision: int, cfg: SparsityConfig = SparsityConfig(),
                 depth: int = 3, device="cuda"):
        self.n_vision, self.cfg = n_vision, cfg
        bf = dict(device=device, dtype=torch.bfloat16)
        self.bufs = [dict(Q=torch.empty(hq, n, d, **bf), K=torch.empty(hkv, n, d, **bf),
                          V=torch.empty(hkv, n, d, **bf), O=torch.empty(hq, n, d, **bf),
                          free=torch.cuda.Event(), loaded=torch.cuda.Event(), done=torch.cuda.Event())
                     for _ in range(depth)]
        for b in self.bufs:
            b["free"].record()
        self.h2d, self.d2h = torch.cuda.Stream(), torch.cuda.Stream()
        self.comp = torch.cuda.current_stream()

    def run(self, requests, outputs) -> None:
        """requests: iterable of pinned (Q, K, V) host tensors; outputs: pinned
        host tensors receiving O. Returns when all copies are enqueued."""
        for i, ((hq_, hk_, hv_), ho) in enumerate(zip(requests, outputs)):
            b = self.bufs[i % len(self.bufs)]
            self.h2d.wait_event(b["free"])
            with torch.cuda.stream(self.h2d):
                b["Q"].copy_(hq_, non_blocking=True)
                b["K"].copy_(hk_, non_blocking=True)
                b["V"].copy_(hv_, non_blocking=True)
                b["loaded"].record()
            self.comp.wait_event(b["loaded"])
            with torch.cuda.stream(self.comp):
                sparse_prefill_device(b["Q"], b["K"], b["V"], self.n_vision, self.cfg, out=b["O"])
                b["done"].record()
            self.d2h.wait_event(b["done"])
            with torch.cuda.stream(self.d2h):
                ho.copy_(b["O"], non_blocking=True)
                b["free"].record()

    def synchronize(self) -> None:
        self.d2h.synchronize()
        self.comp.synchronize()


def sparse_prefill_device(Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, n_vision: int,
                          cfg: SparsityConfig = SparsityConfig(), want_prob: bool = False,
                          out: torch.Tensor | None = None, score_source: str = "probe") -> DevicePrefill:
    """Full sparse prefill of one attention layer on the GPU.

    Q [Hq, N, 128] bf16 (or fp32 for selection-only validation — attention
    then needs bf16 copies), K/V [Hkv, N, 128]."""
    check_qkv(Q, K, V)
    hq, n, d = Q.shape
    hkv = K.shape[0]
    Qb = Q if Q.dtype == torch.bfloat16 else Q.to(torch.bfloat16)
    Kb = K if K.dtype == torch.bfloat16 else K.to(torch.bfloat16)
    Vb = V if V.dtype == torch.bfloat16 else V.to(torch.bfloat16)
    O = out if out is not None else torch.empty_like(Qb)
    k_lazy, k_act, pk, active, p_act, pq, rows, counts, mass, sel = select_device(Q, K, n_vision, cfg, want_prob, O,
                                                                                  score_source)
    cap = ops.round_up(n, ops.TILE)
    K_sel = ops.gather_rows(Kb, sel.selected, sel.counts, cap, ops.TILE)
    V_sel = ops.gather_rows(Vb, sel.selected, sel.counts, cap, ops.TILE)
    lse = torch.empty(hq, n, device=Q.device, dtype=torch.float32)
    ops.sparse_attn_fwd(Qb, K_sel, V_sel, Vb, rows, counts, sel.selected, sel.counts, cfg.sink_index, O, lse)
    return DevicePrefill(O, lse, active, rows, counts, sel, k_lazy, k_act, pq, pk, mass, K_sel, V_sel, p_act)
