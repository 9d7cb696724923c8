"""Slimmed decode: slim KV cache (K6) and decode attention (K7).

Two call forms over one device cache:

* the reference's own signatures (drop-in for ``slimattn.decode``):
  ``build_cache(w, sel, preserve_first_head=True)`` (:82-108),
  ``append_answer(cache, k_heads, v_heads)`` (:111-121),
  ``classify_decode_query(q_heads, cache, tau, counter=None)`` (:124-140) and
  ``decode_attention(q_heads, cache, tau, counter=None, flags=None)`` ->
  ``(list of [d] outputs, flags)`` (:157-194), NumPy in / NumPy out, float64
  classification, fetches metered per head under the reference's flat
  8-byte model (``FetchLog``, :45-61);
* batched device forms for serving (``build_cache_device``,
  ``append_answer_batch``, ``classify_decode_batch``,
  ``decode_attention_batch``): torch tensors [B, H, d] on the GPU, no host
  round trip, bytes metered at the cache's bf16 storage width.

Both run K7 under GQA rule B: one pruned vision segment of exactly ``b`` rows
per (sequence, KV group), the group's vision rows are fetched iff any of its
Q heads is active, lazy Q heads attend over text + answer only (exclusion
semantics).

Serving lifecycle (beyond the reference's one growable list per head,
decode.py:111-121, and its batch-of-one scope): the cache is
PAGED. A ``PagePool`` holds one layer's K / V in 64-row pages; each
(sequence, KV group) owns a page list — its vision pages, then text pages,
then answer pages — in the batch's device page table, and every sequence has
its own budget, prompt-text and answer length. ``admit`` writes only the new
sequence's pages and concatenates small per-sequence tables, ``evict``
returns a finished sequence's pages to the pool, and answer growth takes one
page per group every 64 tokens: no operation copies another sequence's KV.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

import numpy as np

from . import ops
from .attention import AttentionWorkload
from .errors import DegenerateContextError, IntegrityError, ShapeError

VALUE_BYTES_BF16 = 2
VALUE_BYTES_REFERENCE = 8  # metrics.py VALUE_BYTES: the reference's flat float64 memory model


@dataclass
class FetchLog:
    """``decode.py:45-61``. Reference-signature caches meter per head at the
    reference's 8-byte value width; batched device caches meter the bytes K7
    reads (a KV group's rows once, bf16 = 2 bytes)."""

    vision_tokens: int = 0
    vision_bytes: int = 0
    text_answer_bytes: int = 0
    step_vision_tokens: list = field(default_factory=list)
    step_active_heads: list = field(default_factory=list)

    @property
    def steps(self) -> int:
        return len(self.step_active_heads)

    @property
    def active_head_steps(self) -> int:
        return int(sum(self.step_active_heads))


PAGE = 64  # rows per page (= K7's TMA box)


class PagePool:
    """One layer's KV pages on one device: K and V [n_pages, 64, 128] bf16,
    zero-initialised (rows past a segment's end inside its last page stay
    finite, so masked keys contribute exactly 0), and a free list. Growing
    reallocates both tensors geometrically (rare; page ids stay valid)."""

    def __init__(self, n_pages: int = 1024, device="cuda", width: int = 128):
        self.width = width
        self.k = torch.zeros(n_pages, PAGE, width, device=device, dtype=torch.bfloat16)
        self.v = torch.zeros_like(self.k)
        self.free = list(range(n_pages - 1, -1, -1))  # pop() hands out low ids first

    @property
    def n_pages(self) -> int:
        return self.k.shape[0]

    @property
    def used(self) -> int:
        return self.n_pages - len(self.free)

    def reserve(self, n: int) -> None:
        """Make at least n pages free (one reallocation instead of many)."""
        if len(self.free) >= n:
            return
        old = self.n_pages
        new = max(2 * old, old + n - len(self.free))
        grow = lambda t: torch.cat([t, torch.zeros(new - old, PAGE, self.width, device=t.device, dtype=t.dtype)])
        self.k, self.v = grow(self.k), grow(self.v)
        self.free = list(range(new - 1, old - 1, -1)) + self.free

    def alloc(self, n: int) -> np.ndarray:
        self.reserve(n)
        return np.array([self.free.pop() for _ in range(n)], dtype=np.int32)

    def release(self, pages) -> None:
        self.free.extend(int(p) for p in np.asarray(pages).ravel())


_POOLS: dict = {}


def default_pool(device) -> PagePool:
    """The per-device pool caches are built in unless one is passed."""
    device = torch.device(device)
    if device.index is None:
        device = torch.device(device.type, torch.cuda.current_device())
    key = str(device)
    if key not in _POOLS:
        _POOLS[key] = PagePool(1024, device)
    return _POOLS[key]


def _pages(rows: int) -> int:
    return -(-rows // PAGE)


@dataclass
class SlimKVCache:
    """A batch of sequences' slim caches in one PagePool. Per sequence s and
    KV group g the page list pages[s][g] = vision pages (budget rows), text
    pages, answer pages (allocated ahead up to ``answer_capacity`` and then
    64 rows at a time); the device table [B, Hkv, max_pages] mirrors it."""

    pool: PagePool
    table: torch.Tensor           # i32 [B, Hkv, max_pages]
    pages: list                   # per sequence: host i32 [Hkv, n] page ids
    vision_len: torch.Tensor      # i32 [B] = b per sequence
    text_len: torch.Tensor        # i32 [B]
    answer_len: torch.Tensor      # i32 [B], advanced on the device by each append
    vision_indices: list          # per sequence: i32 [Hkv, b] original positions
    k_lazy: torch.Tensor          # f64 [B, Hkv, 128]
    k_act: torch.Tensor
    n_q_heads: int
    preserve_first_head: bool
    budgets: list                 # host copies of the lengths
    text_lens: list
    answer_lens: list
    fetch: FetchLog = field(default_factory=FetchLog)
    status: torch.Tensor | None = None  # i32 [1] degenerate-context flag of the last step
    # reference-signature caches (build_cache(w, sel)): logical head dim of
    # rows zero-padded to the 128-column storage, and the reference's
    # per-head fetch accounting at its 8-byte value width
    dim: int = 0
    value_bytes: int = VALUE_BYTES_BF16
    per_head_log: bool = False

    @property
    def batch(self) -> int:
        return self.table.shape[0]

    @property
    def n_kv_heads(self) -> int:
        return self.table.shape[1]

    @property
    def store_dim(self) -> int:
        """Row width in device memory (128)."""
        return self.pool.width

    @property
    def head_dim(self) -> int:
        """Logical head dim (the reference's; rows are zero-padded past it)."""
        return self.dim or self.store_dim

    @property
    def num_heads(self) -> int:
        """Q heads (decode.py:74-76: one head list per attention head)."""
        return self.n_q_heads

    @property
    def budget(self) -> int:
        """The shared vision budget (decode.py:66); one per sequence."""
        if len(set(self.budgets)) != 1:
            raise ShapeError("sequences of this batch hold different budgets; see .budgets")
        return self.budgets[0]

    @property
    def n_text(self) -> int:
        return max(self.text_lens)

    @property
    def n_answer(self) -> int:
        return max(self.answer_lens)

    @property
    def ragged(self) -> bool:
        return len(set(zip(self.text_lens, self.answer_lens))) > 1

    def seq_text_answer(self) -> list:
        """Per sequence (text rows, answer rows)."""
        return list(zip(self.text_lens, self.answer_lens))

    def answer_capacity(self, s: int) -> int:
        """Answer rows sequence s can take before its next page is needed."""
        return (self.pages[s].shape[1] - _pages(self.budgets[s]) - _pages(self.text_lens[s])) * PAGE

    def n_chunks(self) -> int:
        """K7 work items per (sequence, group): 32 pages each."""
        most = max(_pages(b) + _pages(t) + _pages(a) for b, t, a in
                   zip(self.budgets, self.text_lens, self.answer_lens))
        return max(1, -(-most // 32))

    def rows(self, s: int, g: int, segment: str, which: str = "k") -> torch.Tensor:
        """The rows of one segment ("vision" / "text" / "answer") of sequence
        s, group g, gathered from its pages (inspection and tests)."""
        tv, tt = _pages(self.budgets[s]), _pages(self.text_lens[s])
        n, first = {"vision": (self.budgets[s], 0), "text": (self.text_lens[s], tv),
                    "answer": (self.answer_lens[s], tv + tt)}[segment]
        ids = torch.from_numpy(self.pages[s][g, first:first + _pages(n)].astype(np.int64)).to(self.table.device)
        src = self.pool.k if which == "k" else self.pool.v
        return src.index_select(0, ids).reshape(-1, self.store_dim)[:n]

    def resident_bytes(self) -> int:
        """Bytes a step would read with every group active (slimmed cache)."""
        ta = sum(t + a for t, a in self.seq_text_answer())
        return (sum(self.budgets) + ta) * self.n_kv_heads * 2 * self.store_dim * VALUE_BYTES_BF16

    def release(self) -> None:
        """Return every page of this batch to the pool."""
        for p in self.pages:
            self.pool.release(p)
        self.pages = [np.zeros((self.n_kv_heads, 0), np.int32) for _ in self.pages]


def build_cache_device(K: torch.Tensor, V: torch.Tensor, vision_selected: torch.Tensor, budget: int, n_vision: int,
                       n_text: int, k_lazy: torch.Tensor, k_act: torch.Tensor, n_q_heads: int,
                       preserve_first_head: bool = True, answer_capacity: int = 64,
                       pool: PagePool | None = None) -> SlimKVCache:
    """One sequence's slim cache (decode.py:82-108) written straight into the
    page pool: the ``budget`` selected vision rows of every KV group (K6
    gather into pages), the text span, answer pages reserved for
    ``answer_capacity`` rows; probe keys frozen from the unpruned K.
    K / V [Hkv, N, 128] bf16 (or castable)."""
    hkv, n, d = K.shape
    if vision_selected.shape[0] != hkv:
        raise IntegrityError("one selection per KV group required")
    if not 1 <= budget <= n_vision:
        raise IntegrityError(f"budget {budget} outside the vision span")
    if vision_selected.shape[-1] < budget:
        raise IntegrityError("the selection holds fewer indices than the budget")
    pool = pool or default_pool(K.device)
    if d != pool.width:
        raise ShapeError(f"cache rows are {pool.width} columns; zero-pad K / V first")
    Kb = (K if K.dtype == torch.bfloat16 else K.to(torch.bfloat16)).contiguous()
    Vb = (V if V.dtype == torch.bfloat16 else V.to(torch.bfloat16)).contiguous()
    tv, tt, ta = _pages(budget), _pages(n_text), _pages(answer_capacity)
    pages = pool.alloc(hkv * (tv + tt + ta)).reshape(hkv, tv + tt + ta)
    table = torch.from_numpy(pages).to(K.device)[None].contiguous()
    vsel = vision_selected.to(device=K.device, dtype=torch.int32).contiguous()
    ops.page_write(Kb, vsel, budget, table[0], 0, pool.k)
    ops.page_write(Vb, vsel, budget, table[0], 0, pool.v)
    if n_text:
        tk = Kb[:, n_vision:n_vision + n_text].contiguous()
        tvv = Vb[:, n_vision:n_vision + n_text].contiguous()
        ops.page_write(tk, None, n_text, table[0], tv, pool.k)
        ops.page_write(tvv, None, n_text, table[0], tv, pool.v)
    i32 = dict(dtype=torch.int32, device=K.device)
    return SlimKVCache(pool, table, [pages], torch.tensor([budget], **i32), torch.tensor([n_text], **i32),
                       torch.zeros(1, **i32), [vsel[:, :budget].clone()], k_lazy.unsqueeze(0).contiguous(),
                       k_act.unsqueeze(0).contiguous(), n_q_heads, preserve_first_head, [budget], [n_text], [0],
                       status=torch.zeros(1, **i32))


def cache_from_prompt(Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, n_vision: int, n_text: int, cfg,
                      answer_capacity: int = 64, pool: PagePool | None = None) -> SlimKVCache:
    """The prefill -> decode hand-off of one sequence: the
    prompt's selection (K1-K3), its budget restricted to the vision span
    (select_vision_keys, kv_select.py:179-195) and the slim cache built from
    it (K6 into pages). Q [Hq, N, d], K / V [Hkv, N, d] on the device."""
    from .pipeline import select_device

    hq, hkv, n = Q.shape[0], K.shape[0], K.shape[1]
    k_lazy, k_act, _, _, _, _, _, _, mass, sel = select_device(Q, K, n_vision, cfg)
    b = min(int(sel.info[0]), n_vision)
    vsel = ops.select(mass, hkv, n, cfg.block_size, cfg.p, "token", vision_limit=n_vision, budget_override=b)
    return build_cache_device(K, V, vsel.selected, b, n_vision, n_text, k_lazy, k_act, hq,
                              cfg.preserve_first_head, answer_capacity=answer_capacity, pool=pool)


def _table(pages: list, device) -> torch.Tensor:
    width = max(1, max(p.shape[1] for p in pages))
    t = np.zeros((len(pages), pages[0].shape[0], width), dtype=np.int32)
    for s, p in enumerate(pages):
        t[s, :, : p.shape[1]] = p
    return torch.from_numpy(t).to(device)


def stack_caches(caches: list[SlimKVCache]) -> SlimKVCache:
    """Batch sequences of one pool into one cache: the page tables, lengths
    and probe keys are concatenated (O(table), no KV copy). The inputs are
    consumed (their pages now belong to the batch)."""
    c0 = caches[0]
    for c in caches[1:]:
        if c.pool is not c0.pool:
            raise ShapeError("caches of one batch must live in the same PagePool")
        if (c.n_q_heads, c.n_kv_heads, c.head_dim, c.preserve_first_head, c.per_head_log) != \
                (c0.n_q_heads, c0.n_kv_heads, c0.head_dim, c0.preserve_first_head, c0.per_head_log):
            raise ShapeError("caches of one batch must share head layout and preserve_first_head")
    pages = [p for c in caches for p in c.pages]
    cat = lambda name: torch.cat([getattr(c, name) for c in caches]).contiguous()
    return SlimKVCache(c0.pool, _table(pages, c0.table.device), pages, cat("vision_len"), cat("text_len"),
                       cat("answer_len"), [v for c in caches for v in c.vision_indices], cat("k_lazy"),
                       cat("k_act"), c0.n_q_heads, c0.preserve_first_head, [b for c in caches for b in c.budgets],
                       [t for c in caches for t in c.text_lens], [a for c in caches for a in c.answer_lens],
                       status=torch.zeros(1, dtype=torch.int32, device=c0.table.device), dim=c0.dim,
                       value_bytes=c0.value_bytes, per_head_log=c0.per_head_log)


def admit(cache: SlimKVCache, new: SlimKVCache | list) -> SlimKVCache:
    """Add sequences (built with ``build_cache_device`` in the same pool) to
    a running batch; only their own pages were written. Fetch accounting
    continues on the returned cache."""
    out = stack_caches([cache] + (list(new) if isinstance(new, list) else [new]))
    out.fetch = cache.fetch
    return out


def evict(cache: SlimKVCache, keep: list) -> SlimKVCache:
    """Drop finished sequences: their pages go back to the pool; the batch
    keeps the rows ``keep`` (in that order). Fetch accounting continues."""
    if not keep:
        raise ShapeError("evict would leave an empty batch")
    if any(not 0 <= s < cache.batch for s in keep):
        raise ShapeError("evict: sequence index outside the batch")
    for s in range(cache.batch):
        if s not in keep:
            cache.pool.release(cache.pages[s])
    idx = torch.tensor(keep, dtype=torch.long, device=cache.table.device)
    pick = lambda t: t.index_select(0, idx).contiguous()
    pages = [cache.pages[s] for s in keep]
    return SlimKVCache(cache.pool, _table(pages, cache.table.device), pages, pick(cache.vision_len),
                       pick(cache.text_len), pick(cache.answer_len), [cache.vision_indices[s] for s in keep],
                       pick(cache.k_lazy), pick(cache.k_act), cache.n_q_heads, cache.preserve_first_head,
                       [cache.budgets[s] for s in keep], [cache.text_lens[s] for s in keep],
                       [cache.answer_lens[s] for s in keep], fetch=cache.fetch, status=cache.status,
                       dim=cache.dim, value_bytes=cache.value_bytes, per_head_log=cache.per_head_log)


def append_answer_batch(cache: SlimKVCache, k_rows: torch.Tensor, v_rows: torch.Tensor, grow: bool = True) -> None:
    """decode.py:111-121: grow every sequence's answer segment by one token
    (k_rows / v_rows: [B, Hkv, 128]). A sequence whose answer pages are full
    takes one new page per group (the reference's lists are unbounded);
    with ``grow=False`` that raises instead."""
    if k_rows.shape != (cache.batch, cache.n_kv_heads, cache.store_dim) or v_rows.shape != k_rows.shape:
        raise ShapeError("append needs one k and one v row per (sequence, KV head)")
    need = [s for s in range(cache.batch) if cache.answer_lens[s] >= cache.answer_capacity(s)]
    if need:
        if not grow:
            raise ShapeError("answer capacity exhausted")
        for s in need:
            cache.pages[s] = np.concatenate([cache.pages[s], cache.pool.alloc(cache.n_kv_heads)[:, None]], axis=1)
        width = max(p.shape[1] for p in cache.pages)
        if width > cache.table.shape[2]:
            cache.table = torch.nn.functional.pad(cache.table, (0, max(width, 2 * cache.table.shape[2])
                                                                - cache.table.shape[2])).contiguous()
        for s in need:
            col = cache.pages[s].shape[1] - 1
            cache.table[s, :, col] = torch.from_numpy(cache.pages[s][:, col]).to(cache.table.device)
    ops.append_answer_paged(k_rows, v_rows, cache.pool.k, cache.pool.v, cache.table, cache.vision_len,
                            cache.text_len, cache.answer_len)
    cache.answer_lens = [a + 1 for a in cache.answer_lens]


def classify_decode_batch(q: torch.Tensor, cache: SlimKVCache, tau: float) -> torch.Tensor:
    """decode.py:124-140 for a batch: u8 [B, Hq] active flags of one decode
    token per sequence (the classification decode_attention also runs)."""
    if q.shape != (cache.batch, cache.n_q_heads, cache.store_dim):
        raise ShapeError(f"decode query must be [B, Hq, d], got {tuple(q.shape)}")
    qb = (q if q.dtype == torch.bfloat16 else q.to(torch.bfloat16)).contiguous()
    flags = torch.empty(cache.batch, cache.n_q_heads, device=q.device, dtype=torch.uint8)
    ops.call_decode_flags(qb, cache.k_lazy, cache.k_act, cache.n_kv_heads, float(tau), cache.preserve_first_head, flags,
                          head_dim=cache.head_dim)
    return flags


def decode_attention_batch(q: torch.Tensor, cache: SlimKVCache, tau: float, flags: torch.Tensor | None = None,
                           log: bool = True):
    """decode.py:157-194 for a batch: returns (out f32 [B, Hq, 128], flags u8
    [B, Hq]); ``flags`` overrides classification (decode.py:170-173). A lazy
    head with neither text nor answer rows raises DegenerateContextError
    (decode.py:152-153; read back only when such a sequence exists)."""
    if q.shape != (cache.batch, cache.n_q_heads, cache.store_dim):
        raise ShapeError(f"decode query must be [B, Hq, d], got {tuple(q.shape)}")
    qb = (q if q.dtype == torch.bfloat16 else q.to(torch.bfloat16)).contiguous()
    fo = None if flags is None else flags.to(device=q.device, dtype=torch.uint8).contiguous()
    out, fl = ops.decode_paged(qb, cache.pool.k, cache.pool.v, cache.table, cache.vision_len, cache.text_len,
                               cache.answer_len, cache.n_chunks(), cache.k_lazy, cache.k_act, tau,
                               cache.preserve_first_head, cache.status, head_dim=cache.head_dim, flags_override=fo)
    if any(t + a == 0 for t, a in cache.seq_text_answer()) and int(cache.status[0]):
        raise DegenerateContextError("lazy head with no text and no answer KV (decode.py:152-153)")
    if log:
        account(cache, fl)
    return out, fl


def step_bytes(cache: SlimKVCache, flags: torch.Tensor) -> tuple[int, int, int]:
    """(vision tokens, vision bytes, text+answer bytes) one step reads."""
    rep = cache.n_q_heads // cache.n_kv_heads
    fetched = flags.view(cache.batch, cache.n_kv_heads, rep).any(dim=2).cpu()
    row = 2 * cache.store_dim * VALUE_BYTES_BF16
    vt = int(sum(int(fetched[s].sum()) * cache.budgets[s] for s in range(cache.batch)))
    ta = sum(t + a for t, a in cache.seq_text_answer()) * cache.n_kv_heads * row
    return vt, vt * row, ta


def account(cache: SlimKVCache, flags: torch.Tensor) -> None:
    if cache.per_head_log:
        _account_per_head(cache, flags)
        return
    vt, vb, tb = step_bytes(cache, flags)
    f = cache.fetch
    f.vision_tokens += vt
    f.vision_bytes += vb
    f.text_answer_bytes += tb
    f.step_vision_tokens.append(vt)
    f.step_active_heads.append(int(flags.sum()))


def _account_per_head(cache: SlimKVCache, flags: torch.Tensor) -> None:
    """decode.py:176-193: per Q head, ``budget`` vision tokens and
    budget * 2 * d * VALUE_BYTES bytes when active, the text + answer rows it
    attended over otherwise too (the reference's flat model)."""
    f = cache.fetch
    fl = flags.cpu().numpy().astype(bool)
    row = 2 * cache.head_dim * cache.value_bytes
    step_vision = 0
    for s, ((t, a), b) in enumerate(zip(cache.seq_text_answer(), cache.budgets)):
        for h in range(cache.n_q_heads):
            if fl[s, h]:
                step_vision += b
                f.vision_bytes += b * row
            f.text_answer_bytes += (t + a) * row
    f.vision_tokens += step_vision
    f.step_vision_tokens.append(step_vision)
    f.step_active_heads.append(int(fl.sum()))


# ------------------------------------------------ reference-signature operators
def _rows(x, count: int, dim: int, what: str) -> np.ndarray:
    """Per-head rows (list of [d] / [1, d] arrays or an [H, d] array) as a
    float64 [H, d] array, with the reference's shape errors."""
    if isinstance(x, torch.Tensor):
        x = x.detach().cpu().numpy()
    if len(x) != count:
        raise ShapeError(f"{what} needs one row per head")
    arr = np.stack([np.asarray(r, dtype=np.float64).reshape(-1) for r in x])
    if arr.shape[1] != dim:
        raise ShapeError(f"{what} rows must have length {dim}")
    return arr


def _pad(t: torch.Tensor, width: int) -> torch.Tensor:
    return torch.nn.functional.pad(t, (0, width - t.shape[-1])) if t.shape[-1] < width else t


def build_cache(w: AttentionWorkload, sel, preserve_first_head: bool = True) -> SlimKVCache:
    """decode.py:82-108: prune each KV head's vision K/V to its selected
    indices (exactly ``sel.budget`` of them, inside the vision span), copy the
    text K/V, freeze the probe keys built from the UNPRUNED keys (float64),
    answer empty. ``sel`` is a SelectionResult (``select_vision_keys``); rows
    are stored bf16, zero-padded to 128 columns; a batch of one sequence."""
    nv, nt = w.layout.n_vision, w.layout.n_text
    hkv, d = w.num_kv_heads, w.head_dim
    if d > 128:
        raise ShapeError("head_dim must be <= 128")
    if len(sel.selected) != hkv:
        raise IntegrityError(f"selection covers {len(sel.selected)} heads, the cache {hkv}")
    for i, idx in enumerate(sel.selected):
        idx = np.asarray(idx, dtype=np.int64)
        if idx.shape[0] != sel.budget:
            raise IntegrityError(f"head {i} selection has {idx.shape[0]} keys, budget {sel.budget}")
        if idx.size and (idx.min() < 0 or idx.max() >= nv):
            raise IntegrityError(f"head {i} selection indices fall outside the vision span")
    if sel.budget < 1:
        raise IntegrityError("the vision budget must be positive")
    _, K, V = w.device_tensors(torch.float64)
    K, V = _pad(K, 128).contiguous(), _pad(V, 128).contiguous()
    k_lazy, k_act, _ = ops.kv_probe(K, nv, w.layout.sink_index, max(1, K.shape[1]))  # float64, unpruned K
    vidx = torch.from_numpy(np.stack([np.asarray(i, dtype=np.int32) for i in sel.selected])).to(K.device)
    cache = build_cache_device(K.to(torch.bfloat16), V.to(torch.bfloat16), vidx, int(sel.budget), nv, nt, k_lazy, k_act,
                               w.num_heads, preserve_first_head, answer_capacity=PAGE)
    cache.dim, cache.value_bytes, cache.per_head_log = d, VALUE_BYTES_REFERENCE, True
    return cache


def append_answer(cache: SlimKVCache, k_heads, v_heads) -> None:
    """decode.py:111-121: grow every KV head's answer segment by one token."""
    if cache.batch != 1:
        raise ShapeError("the reference-signature append takes a one-sequence cache; use append_answer_batch")
    k = _rows(k_heads, cache.n_kv_heads, cache.head_dim, "append")
    v = _rows(v_heads, cache.n_kv_heads, cache.head_dim, "append")
    dev = cache.table.device
    to = lambda a: _pad(torch.from_numpy(a).to(dev), cache.store_dim).to(torch.bfloat16)[None].contiguous()
    append_answer_batch(cache, to(k), to(v))


def classify_decode_query(q_heads, cache: SlimKVCache, tau: float, counter=None) -> np.ndarray:
    """decode.py:124-140: per-head active flags of one decoding token,
    classified in float64 against the frozen probe keys; head 0 forced
    active under first-head preservation. ``counter`` (OpCounter) is
    accepted for signature compatibility; op counting is out of scope."""
    if cache.batch != 1:
        raise ShapeError("the reference-signature classification takes a one-sequence cache")
    if not 0.0 <= tau < 1.0:
        raise ValueError(f"tau must be in [0, 1), got {tau}")
    q = _rows(q_heads, cache.n_q_heads, cache.head_dim, "decode query")
    qd = torch.from_numpy(q).to(cache.table.device)[None].contiguous()
    flags = torch.empty(1, cache.n_q_heads, device=qd.device, dtype=torch.uint8)
    ops.decode_flags_f64(qd, cache.k_lazy, cache.k_act, cache.n_kv_heads, float(tau), cache.preserve_first_head, flags)
    return flags[0].cpu().numpy().astype(bool)


def decode_attention(q_heads, cache: SlimKVCache, tau: float, counter=None, flags=None):
    """decode.py:157-194: one decode step over all heads with the conditional
    vision fetch. ``flags`` overrides the classification (decode.py:170-173).
    Returns (list of float64 [d] outputs, bool flags); the fetch log gains one
    entry. Lazy heads with neither text nor answer rows raise
    DegenerateContextError (decode.py:152-153)."""
    if cache.batch != 1:
        raise ShapeError("the reference-signature decode takes a one-sequence cache; use decode_attention_batch")
    q = _rows(q_heads, cache.n_q_heads, cache.head_dim, "decode query")
    if flags is None:
        fl = classify_decode_query(q, cache, tau, counter)
    else:
        fl = np.asarray(flags, dtype=bool).reshape(-1)
        if fl.shape[0] != cache.n_q_heads:
            raise ShapeError("flags needs one entry per head")
    dev = cache.table.device
    if not fl.all() and cache.n_text + cache.n_answer == 0:
        raise DegenerateContextError("lazy head with no text and no answer KV")
    qb = _pad(torch.from_numpy(q).to(dev), cache.store_dim).to(torch.bfloat16)[None].contiguous()
    out, _ = decode_attention_batch(qb, cache, tau, flags=torch.from_numpy(fl[None].astype(np.uint8)).to(dev))
    o = out[0, :, : cache.head_dim].double().cpu().numpy()
    return [o[h] for h in range(cache.n_q_heads)], fl
