"""Slimmed decode: batched slim KV cache (K6) and decode attention (K7).

Mirrors ``decode.py`` of the reference (HeadCache / SlimKVCache / FetchLog,
``build_cache`` :82-108, ``append_answer`` :111-121, ``classify_decode_query``
:124-140, ``decode_attention`` :157-194) with a batch dimension and GQA rule
B: one pruned vision segment of exactly ``b`` rows per (sequence, KV group),
the group's vision rows are fetched iff any of its Q heads is active, lazy Q
heads attend over text + answer only (exclusion semantics).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import ops
from .errors import IntegrityError, ShapeError

VALUE_BYTES_BF16 = 2


@dataclass
class FetchLog:
    """``decode.py:45-61`` with bytes metered at the cache's storage width
    (bf16 = 2 bytes; the reference's flat model uses 8-byte float64)."""

    vision_tokens: int = 0
    vision_bytes: int = 0
    text_answer_bytes: int = 0
    step_vision_tokens: list = field(default_factory=list)
    step_active_heads: list = field(default_factory=list)

    @property
    def steps(self) -> int:
        return len(self.step_active_heads)


@dataclass
class SlimKVCache:
    """Batched device cache: [B, Hkv, cap, d] segments + frozen probe keys."""

    vision_k: torch.Tensor
    vision_v: torch.Tensor
    vision_len: torch.Tensor      # i32 [B] = b per sequence
    vision_indices: torch.Tensor  # i32 [B, Hkv, vcap] original positions
    text_k: torch.Tensor
    text_v: torch.Tensor
    answer_k: torch.Tensor
    answer_v: torch.Tensor
    k_lazy: torch.Tensor          # f64 [B, Hkv, d]
    k_act: torch.Tensor
    n_q_heads: int
    preserve_first_head: bool
    n_answer: int = 0
    fetch: FetchLog = field(default_factory=FetchLog)
    budgets: list = field(default_factory=list)  # host copy of vision_len

    @property
    def batch(self) -> int:
        return self.vision_k.shape[0]

    @property
    def n_kv_heads(self) -> int:
        return self.vision_k.shape[1]

    @property
    def head_dim(self) -> int:
        return self.vision_k.shape[3]

    @property
    def n_text(self) -> int:
        return self.text_k.shape[2]

    def resident_bytes(self) -> int:
        """Bytes a step would read with every group active (slimmed cache)."""
        b = sum(self.budgets)
        return (b * self.n_kv_heads + self.batch * self.n_kv_heads * (self.n_text + self.n_answer)) * 2 * \
            self.head_dim * VALUE_BYTES_BF16


def build_cache(K: torch.Tensor, V: torch.Tensor, vision_selected: torch.Tensor, budget: int, n_vision: int,
                n_text: int, k_lazy: torch.Tensor, k_act: torch.Tensor, n_q_heads: int,
                preserve_first_head: bool = True, answer_capacity: int = 64, vision_capacity: int | None = None
                ) -> SlimKVCache:
    """One sequence's slim cache (decode.py:82-108): prune + regroup the
    vision KV of every group to its ``budget`` selected rows (K6 gather),
    copy the text span, freeze the probe keys built from the unpruned K."""
    hkv, n, d = K.shape
    if vision_selected.shape[0] != hkv:
        raise IntegrityError("one selection per KV group required")
    if not 1 <= budget <= n_vision:
        raise IntegrityError(f"budget {budget} outside the vision span")
    vcap = vision_capacity or ops.round_up(n_vision, 128)
    if budget > vcap:
        raise ShapeError("vision capacity below the budget")
    Kb = K if K.dtype == torch.bfloat16 else K.to(torch.bfloat16)
    Vb = V if V.dtype == torch.bfloat16 else V.to(torch.bfloat16)
    # rows [budget, vcap) are zero-filled: the TMA-staged decode kernel reads
    # whole 64-key tiles and masks keys past the budget (P = 0 needs finite V)
    vk = ops.gather_rows(Kb, vision_selected, budget, vcap, vcap).unsqueeze(0)
    vv = ops.gather_rows(Vb, vision_selected, budget, vcap, vcap).unsqueeze(0)
    idx = torch.zeros(1, hkv, vcap, dtype=torch.int32, device=K.device)
    idx[0, :, :budget] = vision_selected[:, :budget]
    tk = Kb[:, n_vision:n_vision + n_text].contiguous().unsqueeze(0)
    tv = Vb[:, n_vision:n_vision + n_text].contiguous().unsqueeze(0)
    ak = torch.zeros(1, hkv, answer_capacity, d, dtype=torch.bfloat16, device=K.device)
    av = torch.zeros_like(ak)
    vl = torch.tensor([budget], dtype=torch.int32, device=K.device)
    return SlimKVCache(vk, vv, vl, idx, tk, tv, ak, av, k_lazy.unsqueeze(0).contiguous(),
                       k_act.unsqueeze(0).contiguous(), n_q_heads, preserve_first_head, budgets=[budget])


def stack_caches(caches: list[SlimKVCache]) -> SlimKVCache:
    """Batch per-sequence caches (equal capacities) into one device cache."""
    c0 = caches[0]
    cat = lambda name: torch.cat([getattr(c, name) for c in caches], dim=0).contiguous()
    return SlimKVCache(cat("vision_k"), cat("vision_v"), cat("vision_len"), cat("vision_indices"), cat("text_k"),
                       cat("text_v"), cat("answer_k"), cat("answer_v"), cat("k_lazy"), cat("k_act"), c0.n_q_heads,
                       c0.preserve_first_head, budgets=[b for c in caches for b in c.budgets])


def append_answer(cache: SlimKVCache, k_rows: torch.Tensor, v_rows: torch.Tensor) -> None:
    """decode.py:111-121: grow every group's answer segment by one token
    (k_rows / v_rows: [B, Hkv, d])."""
    if k_rows.shape != (cache.batch, cache.n_kv_heads, cache.head_dim) or v_rows.shape != k_rows.shape:
        raise ShapeError("append needs one k and one v row per (sequence, KV head)")
    if cache.n_answer >= cache.answer_k.shape[2]:
        raise ShapeError("answer capacity exhausted")
    cache.answer_k[:, :, cache.n_answer] = k_rows.to(torch.bfloat16)
    cache.answer_v[:, :, cache.n_answer] = v_rows.to(torch.bfloat16)
    cache.n_answer += 1


def decode_attention(q: torch.Tensor, cache: SlimKVCache, tau: float, flags: torch.Tensor | None = None,
                     log: bool = True):
    """decode.py:157-194 for a batch: returns (out f32 [B, Hq, d], flags u8
    [B, Hq]); ``flags`` overrides classification (decode.py:170-173)."""
    if q.shape != (cache.batch, cache.n_q_heads, cache.head_dim):
        raise ShapeError(f"decode query must be [B, Hq, d], got {tuple(q.shape)}")
    qb = q if q.dtype == torch.bfloat16 else q.to(torch.bfloat16)
    fo = None if flags is None else flags.to(device=q.device, dtype=torch.uint8).contiguous()
    out, fl = ops.decode_step(qb.contiguous(), cache.vision_k, cache.vision_v, cache.vision_len, cache.text_k,
                              cache.text_v, cache.n_text, cache.answer_k, cache.answer_v, cache.n_answer,
                              cache.k_lazy, cache.k_act, tau, cache.preserve_first_head, fo)
    if log:
        account(cache, fl)
    return out, fl


def step_bytes(cache: SlimKVCache, flags: torch.Tensor) -> tuple[int, int, int]:
    """(vision tokens, vision bytes, text+answer bytes) one step reads."""
    rep = cache.n_q_heads // cache.n_kv_heads
    fetched = flags.view(cache.batch, cache.n_kv_heads, rep).any(dim=2).cpu()
    row = 2 * cache.head_dim * VALUE_BYTES_BF16
    vt = int(sum(int(fetched[s].sum()) * cache.budgets[s] for s in range(cache.batch)))
    ta = cache.batch * cache.n_kv_heads * (cache.n_text + cache.n_answer) * row
    return vt, vt * row, ta


def account(cache: SlimKVCache, flags: torch.Tensor) -> None:
    vt, vb, tb = step_bytes(cache, flags)
    f = cache.fetch
    f.vision_tokens += vt
    f.vision_bytes += vb
    f.text_answer_bytes += tb
    f.step_vision_tokens.append(vt)
    f.step_active_heads.append(int(flags.sum()))
