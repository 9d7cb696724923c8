"""Model-side drop-in: a Qwen2 / LLaVA-Video style attention layer whose
attention core is the OmniSparse path.

The reference stops at per-head outputs plus an optional output projection
of their concatenation (``attention.py:111-134``); the paper applies the
method inside the attention layers of Qwen2-based video LLMs
(``PAPER.md:308``). This module is that caller: Q/K/V projections (with the
Qwen2 biases), rotary position embedding, the sparse attention of each
packed sequence (selection under no_grad, K4 forward, K5 backward), the head
concatenation in head order and the output projection. Projections and RoPE
are plain cuBLAS / elementwise torch ops; the attention core has no
fallback.

Packing: ``cu_seqlens`` (host list of cumulative lengths, as varlen flash
attention takes) splits a [T, hidden] token stream into independent
sequences, each laid out vision -> text with its own ``n_vision``.
"""

from __future__ import annotations

import torch

from .autograd import sparse_attention
from .errors import LayoutError, ShapeError
from .pipeline import SparsityConfig


def rope_cos_sin(n: int, head_dim: int, theta: float, device, offset: int = 0):
    """Rotary tables [n, head_dim] (rotate-half convention, fp32)."""
    inv = 1.0 / (theta ** (torch.arange(0, head_dim, 2, device=device, dtype=torch.float32) / head_dim))
    pos = torch.arange(offset, offset + n, device=device, dtype=torch.float32)
    f = torch.outer(pos, inv)
    emb = torch.cat([f, f], dim=1)
    return emb.cos(), emb.sin()


def apply_rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """x [H, n, d] -> x * cos + rotate_half(x) * sin (computed in fp32)."""
    xf = x.float()
    h = xf.shape[-1] // 2
    rot = torch.cat([-xf[..., h:], xf[..., :h]], dim=-1)
    return (xf * cos + rot * sin).to(x.dtype)


class OmniSparseAttention(torch.nn.Module):
    """Attention layer with OmniSparse prefill.

    Defaults are Qwen2-7B's attention shapes (hidden 3584, 28 Q heads, 4 KV
    heads, head_dim 128, rope_theta 1e6, q/k/v biases, no o_proj bias)."""

    def __init__(self, hidden_size: int = 3584, num_heads: int = 28, num_kv_heads: int = 4, head_dim: int = 128,
                 rope_theta: float | None = 1.0e6, qkv_bias: bool = True, cfg: SparsityConfig = SparsityConfig(),
                 device=None, dtype=torch.bfloat16):
        super().__init__()
        if num_heads % num_kv_heads:
            raise ShapeError("num_heads must be a multiple of num_kv_heads")
        if head_dim != 128:
            raise ShapeError("the sparse attention kernels take head_dim 128")
        kw = dict(device=device, dtype=dtype)
        self.hq, self.hkv, self.d = num_heads, num_kv_heads, head_dim
        self.rope_theta, self.cfg = rope_theta, cfg
        self.q_proj = torch.nn.Linear(hidden_size, num_heads * head_dim, bias=qkv_bias, **kw)
        self.k_proj = torch.nn.Linear(hidden_size, num_kv_heads * head_dim, bias=qkv_bias, **kw)
        self.v_proj = torch.nn.Linear(hidden_size, num_kv_heads * head_dim, bias=qkv_bias, **kw)
        self.o_proj = torch.nn.Linear(num_heads * head_dim, hidden_size, bias=False, **kw)

    def qkv(self, x: torch.Tensor):
        """[n, hidden] -> Q [Hq, n, d], K / V [Hkv, n, d] (RoPE applied)."""
        n = x.shape[0]
        q = self.q_proj(x).view(n, self.hq, self.d).transpose(0, 1)
        k = self.k_proj(x).view(n, self.hkv, self.d).transpose(0, 1)
        v = self.v_proj(x).view(n, self.hkv, self.d).transpose(0, 1)
        if self.rope_theta is not None:
            cos, sin = rope_cos_sin(n, self.d, self.rope_theta, x.device)
            q, k = apply_rope(q, cos, sin), apply_rope(k, cos, sin)
        return q.contiguous(), k.contiguous(), v.contiguous()

    def attend(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, n_vision: int) -> torch.Tensor:
        """One sequence's attention core: [Hq, n, d] -> [n, Hq * d]."""
        o = sparse_attention(q, k, v, n_vision, self.cfg)
        return o.transpose(0, 1).reshape(q.shape[1], self.hq * self.d)

    def forward(self, hidden_states: torch.Tensor, n_vision, cu_seqlens: list | None = None) -> torch.Tensor:
        """hidden_states [T, hidden] (packed; ``cu_seqlens`` = [0, l0, l0+l1,
        ..., T]) or [B, S, hidden] (B sequences of S tokens). ``n_vision``: one
        int for every sequence or a list, one per sequence."""
        batched = hidden_states.dim() == 3
        x = hidden_states.reshape(-1, hidden_states.shape[-1]) if batched else hidden_states
        if x.dim() != 2:
            raise ShapeError("hidden_states must be [T, hidden] or [B, S, hidden]")
        T = x.shape[0]
        if cu_seqlens is None:
            cu_seqlens = list(range(0, T + 1, hidden_states.shape[1])) if batched else [0, T]
        cu = [int(c) for c in cu_seqlens]
        if cu[0] != 0 or cu[-1] != T or any(b <= a for a, b in zip(cu, cu[1:])):
            raise LayoutError("cu_seqlens must rise strictly from 0 to the token count")
        nseq = len(cu) - 1
        nv = list(n_vision) if isinstance(n_vision, (list, tuple)) else [int(n_vision)] * nseq
        if len(nv) != nseq:
            raise LayoutError("one n_vision per packed sequence")
        outs = []
        for s in range(nseq):
            q, k, v = self.qkv(x[cu[s]:cu[s + 1]])
            outs.append(self.attend(q, k, v, nv[s]))
        y = self.o_proj(torch.cat(outs, dim=0).to(self.o_proj.weight.dtype))
        return y.view(hidden_states.shape[:-1] + (y.shape[-1],)) if batched else y
