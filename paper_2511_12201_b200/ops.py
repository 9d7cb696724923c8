"""Device-level operators over the C ABI (torch tensors on ``cuda``).

Every function here is one (or two) ``omni_*`` calls on the current torch CUDA
stream; outputs are allocated with the torch caching allocator and passed
down as plain pointers. No host synchronisation happens on the prefill path:
budget, counts and tile bounds stay on the device and grids are sized by
upper bounds.

Layouts: Q [Hq, N, d], K/V [Hkv, N, d] (bf16 for attention; bf16 or fp32 for
selection, the reference's "fp32 validation mode"). GQA rule B: Q head h
belongs to KV group h // (Hq // Hkv).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import torch

from . import _lib
from .errors import ParameterError, ShapeError

GRAN = {"token": 0, "block": 1}
DTYPE = {torch.bfloat16: 0, torch.float32: 1, torch.float64: 2}
TILE = 128  # attention tile rows / key tile (K_sel padding)


def _p(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dtype(t: torch.Tensor) -> int:
    if t.dtype not in DTYPE:
        raise ShapeError(f"unsupported dtype {t.dtype}; use bfloat16, float32 or float64")
    return DTYPE[t.dtype]


def _cuda3(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda:
        raise ShapeError(f"{name} must be a CUDA tensor")
    if t.dim() != 3 or not t.is_contiguous():
        raise ShapeError(f"{name} must be a contiguous [heads, tokens, dim] tensor, got {tuple(t.shape)}")


def n_blocks(n: int, block: int) -> int:
    return math.ceil(n / block)


def round_up(x: int, m: int) -> int:
    return ((x + m - 1) // m) * m


# ----------------------------------------------------------------------- K1
def kv_probe(K: torch.Tensor, n_vision: int, sink_index: int, block_size: int):
    """Probe keys (k_lazy = K[sink], k_act = vision mean) and pooled keys, f64.
    query_select.py:41-47 + block_probe.py:58."""
    _cuda3(K, "K")
    hkv, n, d = K.shape
    nb = n_blocks(n, block_size)
    f64 = dict(device=K.device, dtype=torch.float64)
    k_lazy, k_act = torch.empty(hkv, d, **f64), torch.empty(hkv, d, **f64)
    pooled = torch.empty(hkv, nb, d, **f64)
    ws = torch.empty(max(1, _lib.size("omni_kv_probe_workspace", hkv, n, d, block_size)), device=K.device, dtype=torch.uint8)
    _lib.call("omni_kv_probe", _p(K), _dtype(K), hkv, n, d, n_vision, sink_index, block_size,
              _p(k_lazy), _p(k_act), _p(pooled), _p(ws), _stream())
    return k_lazy, k_act, pooled


# ----------------------------------------------------------------------- K2
def q_score(Q: torch.Tensor, k_lazy, k_act, n_vision: int, tau: float, preserve_first_head: bool, block_size: int,
            want_prob: bool = False, O_zero: torch.Tensor | None = None):
    """Lazy/active flags, optional p_act, pooled queries and per-block active
    counts. query_select.py:50-92 + block_probe.py:57."""
    _cuda3(Q, "Q")
    hq, n, d = Q.shape
    hkv = k_lazy.shape[0]
    nb = n_blocks(n, block_size)
    active = torch.empty(hq, n, device=Q.device, dtype=torch.uint8)
    p_act = torch.empty(hq, max(n_vision, 1), device=Q.device, dtype=torch.float64) if want_prob else None
    pooled = torch.empty(hq, nb, d, device=Q.device, dtype=torch.float64)
    bact = torch.empty(hq, nb, device=Q.device, dtype=torch.int32)
    if O_zero is not None:
        _cuda3(O_zero, "O")
        if O_zero.dtype != torch.bfloat16 or O_zero.shape != Q.shape:
            raise ShapeError("O must be bf16 with Q's shape")
    _lib.call("omni_q_score", _p(Q), _dtype(Q), hq, hkv, n, d, n_vision, float(tau), int(bool(preserve_first_head)),
              block_size, _p(k_lazy), _p(k_act), _p(active), _p(p_act), _p(pooled), _p(bact), _p(O_zero), _stream())
    return active, p_act, pooled, bact


def compact_rows(active: torch.Tensor, block_active: torch.Tensor, block_size: int):
    """Ascending active row positions per head (prefill.py:106) + counts."""
    hq, n = active.shape
    rows = torch.empty(hq, n, device=active.device, dtype=torch.int32)
    counts = torch.empty(hq, device=active.device, dtype=torch.int32)
    _lib.call("omni_compact_rows", _p(active), _p(block_active), hq, n, block_size, _p(rows), _p(counts), _stream())
    return rows, counts


# ----------------------------------------------------------------------- K3
def probe_mass(pooled_q: torch.Tensor, pooled_k: torch.Tensor, return_workspace: bool = False):
    """Column mass of the block-causal pooled probe per Q head, f64 [Hq, nb].
    block_probe.py:44-64,76."""
    hq, nb, d = pooled_q.shape
    hkv = pooled_k.shape[0]
    mass = torch.empty(hq, nb, device=pooled_q.device, dtype=torch.float64)
    ws = torch.empty(_lib.size("omni_probe_mass_workspace", hq, nb) // 8, device=pooled_q.device, dtype=torch.float64)
    _lib.call("omni_probe_mass_map" if return_workspace else "omni_probe_mass", _p(pooled_q), _p(pooled_k), hq, hkv,
              nb, d, _p(mass), _p(ws), _stream())
    if return_workspace:
        return mass, ws
    return mass


def exact_mass(Q: torch.Tensor, K: torch.Tensor) -> torch.Tensor:
    """Column mass of the full causal map per Q head, f64 [Hq, N]
    (kv_select.py:56-73 without the N^2 map)."""
    _cuda3(Q, "Q")
    _cuda3(K, "K")
    if Q.dtype != K.dtype:
        raise ShapeError("Q and K must share a dtype")
    hq, n, d = Q.shape
    mass = torch.empty(hq, n, device=Q.device, dtype=torch.float64)
    ws = torch.empty(_lib.size("omni_exact_mass_workspace", hq, n), device=Q.device, dtype=torch.uint8)
    _lib.call("omni_exact_mass", _p(Q), _p(K), _dtype(Q), hq, K.shape[0], n, d, _p(mass), _p(ws), _stream())
    return mass


@dataclass
class Selection:
    """Device-resident selection (kv_select.SelectionResult + scores)."""

    selected: torch.Tensor      # i32 [Hkv, N]; first `counts[g]` entries valid, ascending
    info: torch.Tensor          # i32 [4 + Hkv] = budget, flattest, Hkv, nb, counts...
    stats: torch.Tensor         # f64 [Hkv + 4] = kurtoses..., retained, total, margin, replayed
    group_scores: torch.Tensor  # f64 [Hkv, nb] per-token score of each block

    @property
    def counts(self) -> torch.Tensor:
        return self.info[4:]


def select(mass: torch.Tensor, n_kv_heads: int, seq_len: int, block_size: int, p: float,
           granularity: str = "token", vision_limit: int = -1, budget_override: int = 0) -> Selection:
    """Flattest-head budget + per-group top-b (kv_select.py:49-195)."""
    if granularity not in GRAN:
        raise ParameterError(f"granularity must be one of {tuple(GRAN)}")
    hq, nb = mass.shape
    dev = mass.device
    selected = torch.empty(n_kv_heads, seq_len, device=dev, dtype=torch.int32)
    info = torch.empty(4 + n_kv_heads, device=dev, dtype=torch.int32)
    stats = torch.empty(n_kv_heads + 4, device=dev, dtype=torch.float64)
    gs = torch.empty(n_kv_heads, nb, device=dev, dtype=torch.float64)
    wsb = _lib.size("omni_select_workspace", n_kv_heads, seq_len, block_size)
    ws = torch.empty(wsb, device=dev, dtype=torch.uint8) if wsb else None
    _lib.call("omni_select_ex", _p(mass.contiguous()), hq, n_kv_heads, seq_len, block_size, float(p),
              GRAN[granularity], int(vision_limit), int(budget_override), _p(selected), _p(info), _p(stats), _p(gs),
              _p(ws), _stream())
    return Selection(selected, info, stats, gs)


def block_sums(x: torch.Tensor, block_size: int) -> torch.Tensor:
    """np.add.reduceat(x[r], arange(0, n, block_size)) per row, in NumPy's
    order (omni_block_sums; kv_select.py:160)."""
    if x.dtype != torch.float64 or not x.is_cuda or x.dim() != 2:
        raise ShapeError("block_sums takes a CUDA float64 [rows, n] tensor")
    x = x.contiguous()
    rows, n = x.shape
    out = torch.empty(rows, n_blocks(n, block_size), device=x.device, dtype=torch.float64)
    _lib.call("omni_block_sums", _p(x), rows, n, int(block_size), _p(out), _stream())
    return out


def top_blocks(block_mass: torch.Tensor, seq_len: int, block_size: int, budget: int):
    """select_top_blocks' table from block masses [G, nb] (omni_top_blocks):
    returns (selected i32 [G, seq_len], counts i32 [G])."""
    if block_mass.dtype != torch.float64 or not block_mass.is_cuda or block_mass.dim() != 2:
        raise ShapeError("top_blocks takes CUDA float64 block masses [groups, blocks]")
    bm = block_mass.contiguous()
    g = bm.shape[0]
    selected = torch.empty(g, seq_len, device=bm.device, dtype=torch.int32)
    info = torch.zeros(4 + g, device=bm.device, dtype=torch.int32)
    ws = torch.empty(_lib.size("omni_top_blocks_workspace", g, seq_len, block_size), device=bm.device,
                     dtype=torch.uint8)
    _lib.call("omni_top_blocks", _p(bm), g, seq_len, int(block_size), int(budget), _p(selected), _p(info), _p(ws),
              _stream())
    return selected, info[4:]


def probe_map(ws: torch.Tensor, n_q_heads: int, nb: int) -> torch.Tensor:
    """The normalised block-causal probe map [Hq, nb, nb] from the workspace
    of ``probe_mass(..., return_workspace=True)`` (omni_probe_map)."""
    out = torch.empty(n_q_heads, nb, nb, device=ws.device, dtype=torch.float64)
    _lib.call("omni_probe_map", _p(ws), n_q_heads, nb, _p(out), _stream())
    return out


# ----------------------------------------------------------------------- K6
def gather_rows(src: torch.Tensor, idx: torch.Tensor, counts: torch.Tensor | int, dst_rows: int,
                pad_rows: int = 1, out: torch.Tensor | None = None) -> torch.Tensor:
    """dst[g, r] = src[g, idx[g, r]] for r < count_g; zero rows up to the next
    multiple of pad_rows (prefill.py:109-110, decode.py:92-107)."""
    _cuda3(src, "src")
    g, rows, d = src.shape
    if out is None:
        out = torch.empty(g, dst_rows, d, device=src.device, dtype=src.dtype)
    cnt_t = counts if isinstance(counts, torch.Tensor) else None
    cnt_c = 0 if cnt_t is not None else int(counts)
    _lib.call("omni_gather_rows", _p(src), _dtype(src), g, rows, d, _p(idx), idx.shape[-1], _p(cnt_t), cnt_c,
              _p(out), dst_rows, pad_rows, _stream())
    return out


def slim_cache(K: torch.Tensor, V: torch.Tensor, vision_selected: torch.Tensor, budget: int, vcap: int):
    """build_cache's pruning + regrouping (decode.py:92-107): the budget
    selected vision rows of every KV group, [Hkv, vcap, d], rows past the
    budget zero (omni_slim_cache)."""
    _cuda3(K, "K")
    _cuda3(V, "V")
    hkv, n, d = K.shape
    vk = torch.empty(hkv, vcap, d, device=K.device, dtype=K.dtype)
    vv = torch.empty_like(vk)
    _lib.call("omni_slim_cache", _p(K), _p(V), _dtype(K), hkv, n, d, _p(vision_selected), vision_selected.shape[-1],
              int(budget), int(vcap), _p(vk), _p(vv), _stream())
    return vk, vv


def scatter_rows(src: torch.Tensor, idx: torch.Tensor, counts: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """out[g, idx[g, r]] = src[g, r] for r < counts[g] (inverse of gather_rows)."""
    _cuda3(src, "src")
    _cuda3(out, "out")
    g, rows, d = src.shape
    if out.dtype != src.dtype or out.shape[0] != g or out.shape[2] != d:
        raise ShapeError("scatter target must match the source dtype, groups and row width")
    _lib.call("omni_scatter_rows", _p(src), _dtype(src), g, rows, d, _p(idx), idx.shape[-1], _p(counts), _p(out),
              out.shape[1], _stream())
    return out


def scatter_key_grads(src: torch.Tensor, idx: torch.Tensor, counts: torch.Tensor, out: torch.Tensor,
                      sink_index: int = -1, sink_add: torch.Tensor | None = None) -> torch.Tensor:
    """out[g, idx[g, r]] = cast(src[g, r] (+ sink_add[g] at sink_index)) for
    r < counts[g]; out (fp32 or bf16, zero-initialised) gets sink_add alone at
    sink_index when the sink is not selected (the training backward's key
    gradient epilogue: scatter, sink add and dtype cast in one pass)."""
    _cuda3(src, "src")
    _cuda3(out, "out")
    g, rows, d = src.shape
    if src.dtype != torch.float32 or out.shape[0] != g or out.shape[2] != d:
        raise ShapeError("key gradient scatter takes fp32 [G, rows, d] into [G, N, d]")
    if out.dtype not in (torch.float32, torch.bfloat16):
        raise ShapeError("key gradients must be float32 or bfloat16")
    sa = None if sink_add is None else sink_add.to(torch.float32).contiguous()
    _lib.call("omni_scatter_key_grads", _p(src), g, rows, d, _p(idx), idx.shape[-1], _p(counts), int(sink_index),
              _p(sa), _p(out), _dtype(out), out.shape[1], _stream())
    return out


# ----------------------------------------------------------------------- K4
last_fwd_status: torch.Tensor | None = None


def sparse_attn_fwd(Q, K_sel, V_sel, V, rows, counts, selected, sel_counts, sink_index: int,
                    O: torch.Tensor, lse: torch.Tensor | None = None):
    """tcgen05 sparse flash-attention forward into O (lazy rows untouched)."""
    hq, n, d = Q.shape
    hkv, cap, _ = K_sel.shape
    if Q.dtype != torch.bfloat16 or K_sel.dtype != torch.bfloat16 or V.dtype != torch.bfloat16:
        raise ShapeError("sparse attention consumes bf16 Q/K/V")
    if selected.shape[-1] != n:
        raise ShapeError("selected must be [Hkv, N]")
    # the fast kernel's overflow status word (caller-owned workspace, zeroed
    # by the call itself): one per call from the stream-ordered caching
    # allocator, so concurrent forwards on different streams never share it
    global last_fwd_status
    status = torch.empty(1, device=Q.device, dtype=torch.int32)
    last_fwd_status = status  # diagnostics only (tests read whether the safe re-run fired)
    _lib.call("omni_sparse_attn_fwd_ex", _p(Q), _p(K_sel), _p(V_sel), _p(V), _p(rows), _p(counts), _p(selected),
              _p(sel_counts), hq, hkv, n, d, cap, sink_index, _p(O), _p(lse), _p(status), _stream())
    return O, lse


def sparse_attn_bwd(Q, K_sel, V_sel, O, dO, lse, rows, counts, selected, sel_counts, dq_dtype=torch.float32):
    """Backward of K4 over the compacted keys; returns (dQ, dK_sel, dV_sel,
    dV_sink): dK / dV in fp32 (reduced over the group's Q heads), dQ in
    ``dq_dtype`` (fp32 or bf16, written directly by the dq kernel)."""
    hq, n, d = Q.shape
    hkv, cap, _ = K_sel.shape
    f32 = dict(device=Q.device, dtype=torch.float32)
    if dq_dtype not in (torch.float32, torch.bfloat16):
        raise ParameterError("dQ dtype must be float32 or bfloat16")
    dQ = torch.empty(hq, n, d, device=Q.device, dtype=dq_dtype)
    dK = torch.empty(hkv, cap, d, **f32)
    dV = torch.empty(hkv, cap, d, **f32)
    dVs = torch.empty(hkv, d, **f32)
    ws = torch.empty(max(1, _lib.size("omni_sparse_attn_bwd_workspace", hq, n)), device=Q.device, dtype=torch.uint8)
    _lib.call("omni_sparse_attn_bwd_ex", _p(Q), _p(K_sel), _p(V_sel), _p(O), _p(dO), _p(lse), _p(rows), _p(counts),
              _p(selected), _p(sel_counts), hq, hkv, n, d, cap, _dtype(dQ), _p(dQ), _p(dK), _p(dV), _p(dVs), _p(ws),
              _stream())
    return dQ, dK, dV, dVs


# ----------------------------------------------------------------------- K7
def decode_paged(q, pool_k, pool_v, table, vision_len, text_len, answer_len, n_chunks: int, k_lazy, k_act,
                 tau: float, preserve_first_head: bool, status, head_dim: int | None = None, flags_override=None,
                 out=None, flags=None):
    """One batched decode step over the paged slim cache (omni_decode;
    decode.py:124-194, rule B). ``head_dim``: logical width of rows
    zero-padded to the 128-column storage (softmax scale 1/sqrt(head_dim))."""
    b, hq, d = q.shape
    hkv = table.shape[1]
    dev = q.device
    if out is None:
        out = torch.empty(b, hq, d, device=dev, dtype=torch.float32)
    if flags is None:
        flags = torch.empty(b, hq, device=dev, dtype=torch.uint8)
    ws = torch.empty(_lib.size("omni_decode_workspace", b, hq, n_chunks), device=dev, dtype=torch.uint8)
    _lib.call("omni_decode", _p(q), _p(pool_k), _p(pool_v), pool_k.shape[0], _p(table), table.shape[2],
              _p(vision_len), _p(text_len), _p(answer_len), int(n_chunks), _p(k_lazy), _p(k_act), b, hq, hkv,
              head_dim or d, float(tau), int(bool(preserve_first_head)), _p(flags_override), _p(flags), _p(out),
              _p(ws), _p(status), _stream())
    return out, flags


def append_answer_paged(k_rows, v_rows, pool_k, pool_v, table, vision_len, text_len, answer_len) -> None:
    """One launch for the batch's new answer K / V rows (omni_append_answer):
    row answer_len[s] of every (sequence, group), answer_len advanced on the
    device. The rows' pages must be in the table already."""
    b, hkv, d = k_rows.shape
    for name, t in (("k_rows", k_rows), ("v_rows", v_rows)):
        if not t.is_cuda or t.device != pool_k.device:
            raise ShapeError(f"{name} must be a CUDA tensor on the cache's device")
    # bind the converted rows to locals: they must outlive the (asynchronous)
    # append kernel, or the allocator could hand K's temporary to V's copy
    kb = k_rows.to(torch.bfloat16).contiguous()
    vb = v_rows.to(torch.bfloat16).contiguous()
    _lib.call("omni_append_answer", _p(kb), _p(vb), _p(pool_k), _p(pool_v), _p(table), table.shape[2],
              _p(vision_len), _p(text_len), _p(answer_len), b, hkv, d, _stream())


def page_write(src: torch.Tensor, idx, count: int, table_rows: torch.Tensor, first_slot: int,
               pool: torch.Tensor) -> None:
    """Rows of src [G, rows, 128] bf16 (gathered by idx [G, >= count] when
    given) into the pages table_rows[g, first_slot + r / 64] of ``pool``
    (omni_page_write); the last page's tail is zero-filled."""
    _cuda3(src, "src")
    g, rows, d = src.shape
    if src.dtype != torch.bfloat16 or pool.dtype != torch.bfloat16:
        raise ShapeError("pages hold bf16 rows")
    tr = table_rows.contiguous()
    _lib.call("omni_page_write", _p(src), g, rows, d, _p(idx), idx.shape[-1] if idx is not None else 0, int(count),
              _p(tr), tr.shape[-1], int(first_slot), _p(pool), _stream())


def call_decode_flags(q, k_lazy, k_act, n_kv_heads: int, tau: float, preserve_first_head: bool, flags,
                      head_dim: int | None = None) -> None:
    b, hq, d = q.shape
    _lib.call("omni_decode_flags", _p(q), _p(k_lazy), _p(k_act), b, hq, n_kv_heads, head_dim or d, float(tau),
              int(bool(preserve_first_head)), _p(flags), _stream())


def decode_flags_f64(q, k_lazy, k_act, n_kv_heads: int, tau: float, preserve_first_head: bool, flags) -> None:
    """classify_decode_query on float64 queries [B, Hq, d] (omni_decode_flags_f64)."""
    if q.dtype != torch.float64 or not q.is_cuda:
        raise ShapeError("decode_flags_f64 takes CUDA float64 queries")
    b, hq, d = q.shape
    _lib.call("omni_decode_flags_f64", _p(q.contiguous()), _p(k_lazy), _p(k_act), b, hq, n_kv_heads, d,
              k_lazy.shape[-1], float(tau), int(bool(preserve_first_head)), _p(flags), _stream())


def device_check() -> None:
    _lib.call("omni_device_check")
