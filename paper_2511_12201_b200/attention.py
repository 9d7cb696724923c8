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

    def device_tensors(self, dtype=torch.bfloat16, device="cuda"):
        """(Q [Hq,N,d], K [Hkv,N,d], V [Hkv,N,d]) on the GPU."""
        def pack(xs):
            return torch.stack([torch.as_tensor(np.asarray(x) if not isinstance(x, torch.Tensor) else x)
                                .to(device=device, dtype=dtype) for x in xs]).contiguous()
        return pack(self.queries), pack(self.keys), pack(self.values)
