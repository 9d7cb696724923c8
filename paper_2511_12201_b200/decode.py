"""Slimmed decode: batched slim KV cache (K6) and decode attention (K7).

Mirrors ``decode.py`` of the reference (HeadCache / SlimKVCache / FetchLog,
``build_cache`` :82-108, ``append_answer`` :111-121, ``classify_decode_query``
:124-140, ``decode_attention`` :157-194) with a batch dimension and GQA rule
B: one pruned vision segment of exactly ``b`` rows per (sequence, KV group),
the group's vision rows are fetched iff any of its Q heads is active, lazy Q
heads attend over text + answer only (exclusion semantics).

Serving lifecycle (beyond the reference's one growable list per head,
decode.py:111-121, and its batch-of-one scope): a batch holds
sequences with their own budget, prompt-text length and answer length
(``ragged`` caches, per-sequence lengths on the device); ``admit`` adds
sequences, ``evict`` drops finished ones, and ``append_answer`` grows the
answer capacity geometrically when it runs out.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import ops
from .errors import DegenerateContextError, IntegrityError, ShapeError

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
    # ragged batches: per-sequence text / answer lengths (host lists + device
    # i32 [B] copies); None = every sequence has n_text text and n_answer answer rows
    text_lens: list | None = None
    answer_lens: list | None = None
    text_len_dev: torch.Tensor | None = None
    answer_len_dev: torch.Tensor | None = None
    status: torch.Tensor | None = None  # i32 [1] degenerate-context flag of the last ragged step

    @property
    def ragged(self) -> bool:
        return self.text_lens is not None

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

    def seq_text_answer(self) -> list:
        """Per sequence (text rows, answer rows)."""
        if self.ragged:
            return list(zip(self.text_lens, self.answer_lens))
        return [(self.n_text, self.n_answer)] * self.batch

    def resident_bytes(self) -> int:
        """Bytes a step would read with every group active (slimmed cache)."""
        ta = sum(t + a for t, a in self.seq_text_answer())
        return (sum(self.budgets) + ta) * self.n_kv_heads * 2 * self.head_dim * VALUE_BYTES_BF16


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
    vk, vv = (t.unsqueeze(0) for t in ops.slim_cache(Kb, Vb, vision_selected, budget, vcap))
    idx = torch.zeros(1, hkv, vcap, dtype=torch.int32, device=K.device)
    idx[0, :, :budget] = vision_selected[:, :budget]
    tk = Kb[:, n_vision:n_vision + n_text].contiguous().unsqueeze(0)
    tv = Vb[:, n_vision:n_vision + n_text].contiguous().unsqueeze(0)
    ak = torch.zeros(1, hkv, answer_capacity, d, dtype=torch.bfloat16, device=K.device)
    av = torch.zeros_like(ak)
    vl = torch.tensor([budget], dtype=torch.int32, device=K.device)
    return SlimKVCache(vk, vv, vl, idx, tk, tv, ak, av, k_lazy.unsqueeze(0).contiguous(),
                       k_act.unsqueeze(0).contiguous(), n_q_heads, preserve_first_head, budgets=[budget])


def _pad_rows(t: torch.Tensor, cap: int) -> torch.Tensor:
    """Zero-pad dim 2 ([B, Hkv, rows, ...]) to ``cap`` rows (TMA tiles read
    whole 64-row boxes; rows past a segment must be finite)."""
    if t.shape[2] == cap:
        return t
    pad = [0, 0] * (t.dim() - 3) + [0, cap - t.shape[2]]
    return torch.nn.functional.pad(t, pad)


def stack_caches(caches: list[SlimKVCache]) -> SlimKVCache:
    """Batch sequences into one device cache. Capacities are padded to the
    largest; the result is ragged unless every sequence has the same text and
    answer lengths."""
    c0 = caches[0]
    for c in caches[1:]:
        if (c.n_q_heads, c.n_kv_heads, c.head_dim, c.preserve_first_head) != \
                (c0.n_q_heads, c0.n_kv_heads, c0.head_dim, c0.preserve_first_head):
            raise ShapeError("caches of one batch must share head layout and preserve_first_head")
    vcap = max(c.vision_k.shape[2] for c in caches)
    tcap = max(c.text_k.shape[2] for c in caches)
    acap = max(c.answer_k.shape[2] for c in caches)
    cat = lambda name, cap: torch.cat([_pad_rows(getattr(c, name), cap) for c in caches], dim=0).contiguous()
    lens = [tl for c in caches for tl in c.seq_text_answer()]
    ragged = len(set(lens)) > 1 or lens[0][0] != tcap
    out = SlimKVCache(cat("vision_k", vcap), cat("vision_v", vcap),
                      torch.cat([c.vision_len for c in caches]).contiguous(), cat("vision_indices", vcap),
                      cat("text_k", tcap), cat("text_v", tcap), cat("answer_k", acap), cat("answer_v", acap),
                      torch.cat([c.k_lazy for c in caches]).contiguous(),
                      torch.cat([c.k_act for c in caches]).contiguous(), c0.n_q_heads, c0.preserve_first_head,
                      n_answer=max(a for _, a in lens), budgets=[b for c in caches for b in c.budgets])
    if ragged:
        _set_lens(out, [t for t, _ in lens], [a for _, a in lens])
    return out


def _set_lens(cache: SlimKVCache, text_lens: list, answer_lens: list) -> None:
    dev = cache.vision_k.device
    cache.text_lens, cache.answer_lens = list(text_lens), list(answer_lens)
    cache.text_len_dev = torch.tensor(text_lens, dtype=torch.int32, device=dev)
    cache.answer_len_dev = torch.tensor(answer_lens, dtype=torch.int32, device=dev)
    cache.n_answer = max(answer_lens)
    if cache.status is None:
        cache.status = torch.zeros(1, dtype=torch.int32, device=dev)


def admit(cache: SlimKVCache, new: SlimKVCache | list) -> SlimKVCache:
    """Add sequences (built with ``build_cache``) to a running batch. Fetch
    accounting continues on the returned cache."""
    out = stack_caches([cache] + (list(new) if isinstance(new, list) else [new]))
    out.fetch = cache.fetch
    return out


def evict(cache: SlimKVCache, keep: list) -> SlimKVCache:
    """Drop finished sequences: keep the batch rows ``keep`` (in that order).
    Capacities stay; fetch accounting continues on the returned cache."""
    if not keep:
        raise ShapeError("evict would leave an empty batch")
    if any(not 0 <= s < cache.batch for s in keep):
        raise ShapeError("evict: sequence index outside the batch")
    idx = torch.tensor(keep, dtype=torch.long, device=cache.vision_k.device)
    pick = lambda t: t.index_select(0, idx).contiguous()
    lens = cache.seq_text_answer()
    out = SlimKVCache(pick(cache.vision_k), pick(cache.vision_v), pick(cache.vision_len), pick(cache.vision_indices),
                      pick(cache.text_k), pick(cache.text_v), pick(cache.answer_k), pick(cache.answer_v),
                      pick(cache.k_lazy), pick(cache.k_act), cache.n_q_heads, cache.preserve_first_head,
                      n_answer=cache.n_answer, fetch=cache.fetch, budgets=[cache.budgets[s] for s in keep])
    if cache.ragged:
        _set_lens(out, [lens[s][0] for s in keep], [lens[s][1] for s in keep])
    return out


def _grow_answer(cache: SlimKVCache, need: int) -> None:
    cap = cache.answer_k.shape[2]
    new_cap = max(need, 2 * cap, 16)
    cache.answer_k = _pad_rows(cache.answer_k, new_cap).contiguous()
    cache.answer_v = _pad_rows(cache.answer_v, new_cap).contiguous()


def append_answer(cache: SlimKVCache, k_rows: torch.Tensor, v_rows: torch.Tensor, grow: bool = True) -> None:
    """decode.py:111-121: grow every sequence's answer segment by one token
    (k_rows / v_rows: [B, Hkv, d]). With ``grow`` the capacity doubles when
    exhausted (the reference's lists are unbounded); otherwise a full
    segment raises."""
    if k_rows.shape != (cache.batch, cache.n_kv_heads, cache.head_dim) or v_rows.shape != k_rows.shape:
        raise ShapeError("append needs one k and one v row per (sequence, KV head)")
    if cache.n_answer >= cache.answer_k.shape[2]:
        if not grow:
            raise ShapeError("answer capacity exhausted")
        _grow_answer(cache, cache.n_answer + 1)
    if cache.ragged:  # per-sequence rows answer_len[s], advanced on the device
        ops.append_answer(k_rows, v_rows, cache.answer_k, cache.answer_v, 0, cache.answer_len_dev)
        cache.answer_lens = [a + 1 for a in cache.answer_lens]
        cache.n_answer = max(cache.answer_lens)
        return
    ops.append_answer(k_rows, v_rows, cache.answer_k, cache.answer_v, cache.n_answer)
    cache.n_answer += 1


def classify_decode_query(q: torch.Tensor, cache: SlimKVCache, tau: float) -> torch.Tensor:
    """decode.py:124-140 for a batch: u8 [B, Hq] active flags of one decode
    token per sequence (the classification decode_attention also runs)."""
    if q.shape != (cache.batch, cache.n_q_heads, cache.head_dim):
        raise ShapeError(f"decode query must be [B, Hq, d], got {tuple(q.shape)}")
    qb = (q if q.dtype == torch.bfloat16 else q.to(torch.bfloat16)).contiguous()
    flags = torch.empty(cache.batch, cache.n_q_heads, device=q.device, dtype=torch.uint8)
    ops.call_decode_flags(qb, cache.k_lazy, cache.k_act, cache.n_kv_heads, float(tau), cache.preserve_first_head, flags)
    return flags


def decode_attention(q: torch.Tensor, cache: SlimKVCache, tau: float, flags: torch.Tensor | None = None,
                     log: bool = True):
    """decode.py:157-194 for a batch: returns (out f32 [B, Hq, d], flags u8
    [B, Hq]); ``flags`` overrides classification (decode.py:170-173)."""
    if q.shape != (cache.batch, cache.n_q_heads, cache.head_dim):
        raise ShapeError(f"decode query must be [B, Hq, d], got {tuple(q.shape)}")
    qb = q if q.dtype == torch.bfloat16 else q.to(torch.bfloat16)
    fo = None if flags is None else flags.to(device=q.device, dtype=torch.uint8).contiguous()
    if cache.ragged:
        out, fl = ops.decode_step_varlen(qb.contiguous(), cache.vision_k, cache.vision_v, cache.vision_len,
                                         cache.text_k, cache.text_v, cache.text_len_dev, cache.answer_k,
                                         cache.answer_v, cache.answer_len_dev, cache.k_lazy, cache.k_act, tau,
                                         cache.preserve_first_head, cache.status, fo)
        if any(t + a == 0 for t, a in cache.seq_text_answer()) and int(cache.status[0]):
            raise DegenerateContextError("lazy head with no text and no answer KV (decode.py:152-153)")
        if log:
            account(cache, fl)
        return out, fl
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
    ta = sum(t + a for t, a in cache.seq_text_answer()) * cache.n_kv_heads * row
    return vt, vt * row, ta


def account(cache: SlimKVCache, flags: torch.Tensor) -> None:
    vt, vb, tb = step_bytes(cache, flags)
    f = cache.fetch
    f.vision_tokens += vt
    f.vision_bytes += vb
    f.text_answer_bytes += tb
    f.step_vision_tokens.append(vt)
    f.step_active_heads.append(int(flags.sum()))
