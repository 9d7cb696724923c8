"""Workload types of the operator API (reference ``attention.py:18-84``).

``AttentionWorkload`` keeps the reference's per-head list form (NumPy arrays
or torch tensors) and adds GQA: ``keys`` / ``values`` may hold fewer heads
than ``queries`` (Hq a multiple of Hkv, rule B). ``device_tensors()`` packs
them into the [H, N, d] bf16 CUDA layout the kernels consume.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import LayoutError, ShapeError


@dataclass(frozen=True)
class TokenLayout:
    """Vision -> text -> answer spans; ``sink_index`` inside the prompt
    (reference attention.py:18-43)."""

    n_vision: int
    n_text: int
    n_answer: int = 0
    sink_index: int = 0

    def __post_init__(self):
        if self.n_vision < 0 or self.n_text < 0 or self.n_answer < 0:
            raise LayoutError("span lengths must be non-negative")
        if not 0 <= self.sink_index < self.n_vision + self.n_text:
            raise LayoutError(f"sink_index {self.sink_index} outside prompt of length {self.n_vision + self.n_text}")

    @property
    def total(self) -> int:
        return self.n_vision + self.n_text + self.n_answer


def _shape(t):
    return tuple(t.shape)


@dataclass
class AttentionWorkload:
    """Per-head Q/K/V ([N, d] each) plus the token layout (reference
    attention.py:46-84), GQA-extended."""

    queries: list
    keys: list
    values: list
    layout: TokenLayout

    def __post_init__(self):
        if len(self.keys) != len(self.values):
            raise ShapeError("per-head tensor lists differ in length")
        if not self.queries or not self.keys:
            raise ShapeError("workload needs at least one head")
        if len(self.queries) % len(self.keys):
            raise ShapeError("query heads must be a multiple of key/value heads")
        shape = _shape(self.queries[0])
        for name, group in (("Q", self.queries), ("K", self.keys), ("V", self.values)):
            for i, t in enumerate(group):
                if _shape(t) != shape:
                    raise ShapeError(f"head {i} {name} shape {_shape(t)} != {shape}")
        if shape[0] != self.layout.total:
            raise ShapeError(f"layout covers {self.layout.total} tokens but tensors have {shape[0]} rows")

    @property
    def num_heads(self) -> int:
        return len(self.queries)

    @property
    def num_kv_heads(self) -> int:
        return len(self.keys)

    @property
    def head_dim(self) -> int:
        return _shape(self.queries[0])[1]

    @property
    def seq_len(self) -> int:
        return _shape(self.queries[0])[0]

    def source_dtype(self) -> torch.dtype:
        """The device dtype that keeps the caller's precision for the
        selection stages: the reference computes in float64, so
        float64 workloads (the reference's own arrays) select in float64,
        fp32 in fp32 and bf16 in bf16; attention always runs on bf16 copies."""
        x = self.queries[0]
        dt = x.dtype if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x)[:1]).dtype
        return dt if dt in (torch.float64, torch.float32, torch.bfloat16) else torch.float32

    def device_tensors(self, dtype=torch.bfloat16, device="cuda"):
        """(Q [Hq,N,d], K [Hkv,N,d], V [Hkv,N,d]) on the GPU."""
        def pack(xs):
            return torch.stack([torch.as_tensor(np.asarray(x) if not isinstance(x, torch.Tensor) else x)
                                .to(device=device, dtype=dtype) for x in xs]).contiguous()
        return pack(self.queries), pack(self.keys), pack(self.values)


@dataclass
class MultiheadOutput:
    """reference attention.py:87-91: per-head outputs, their horizontal
    concatenation (optionally projected) and, on request, the maps."""

    head_outputs: torch.Tensor        # [Hq, N, d]
    concatenated: torch.Tensor        # [N, Hq * d] or [N, out] after the projection
    attention: list | None = None


def concat_heads(outputs: torch.Tensor, output_proj: torch.Tensor | None = None) -> torch.Tensor:
    """Head outputs [Hq, N, d] concatenated in head order ([N, Hq * d],
    attention.py:131) and multiplied by ``output_proj`` [Hq * d, out] when
    given (:132-133). fp32 on the GPU (cuBLAS), whatever the head dtype."""
    hq, n, d = outputs.shape
    concat = outputs.float().transpose(0, 1).reshape(n, hq * d)
    if output_proj is None:
        return concat
    W = torch.as_tensor(output_proj, device=outputs.device, dtype=torch.float32)
    if W.shape[0] != hq * d:
        raise ShapeError(f"output projection has {W.shape[0]} rows, concatenation has {hq * d} columns")
    return concat @ W


def full_multihead(w: AttentionWorkload, causal: bool = True, output_proj=None, keep_attention: bool = False
                   ) -> MultiheadOutput:
    """Exact multi-head attention over a workload (attention.py:111-134).

    Causal: K4 (the sparse kernel) with every row active and the identity key
    selection is dense causal attention. Non-causal runs cuDNN SDPA (a
    comparator, not part of the hot path). ``keep_attention`` materialises
    the fp32 maps (validation sizes only)."""
    from . import ops

    Q, K, V = w.device_tensors()
    hq, n, d = Q.shape
    hkv = K.shape[0]
    rep = hq // hkv
    if causal:
        ident = torch.arange(n, device=Q.device, dtype=torch.int32).repeat(hkv, 1).contiguous()
        cnt = torch.full((hkv,), n, device=Q.device, dtype=torch.int32)
        rows = torch.arange(n, device=Q.device, dtype=torch.int32).repeat(hq, 1).contiguous()
        rcnt = torch.full((hq,), n, device=Q.device, dtype=torch.int32)
        cap = ops.round_up(n, ops.TILE)
        O = torch.empty_like(Q)
        ops.sparse_attn_fwd(Q, ops.gather_rows(K, ident, cnt, cap, ops.TILE),
                            ops.gather_rows(V, ident, cnt, cap, ops.TILE), V, rows, rcnt, ident, cnt, 0, O, None)
    else:
        Ke, Ve = K.repeat_interleave(rep, dim=0), V.repeat_interleave(rep, dim=0)
        O = torch.nn.functional.scaled_dot_product_attention(Q[None], Ke[None], Ve[None])[0]
    maps = None
    if keep_attention:
        if n > 8192:
            raise ShapeError("keep_attention materialises N x N maps; N <= 8192")
        maps = []
        for h in range(hq):
            s = (Q[h].float() @ K[h // rep].float().T) / d ** 0.5
            if causal:
                s = s.masked_fill(torch.ones(n, n, dtype=torch.bool, device=Q.device).triu(1), float("-inf"))
            maps.append(torch.softmax(s, dim=1))
    return MultiheadOutput(O, concat_heads(O, output_proj), maps)
