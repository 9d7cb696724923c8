"""Reference-named prefill operators on the GPU (reference ``prefill.py``).

``sparse_prefill`` and ``sparse_head_attention`` keep the reference's names,
argument meaning and return shapes (per-head NumPy lists when called with
NumPy inputs) and run the B200 kernels: K1-K3 selection, K6 regroup, K4
tcgen05 attention. The always-on dense oracle and recall instrumentation of
the reference (prefill.py:160, :176-179) are not part of the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .attention import AttentionWorkload
from .errors import ParameterError, ShapeError
from .kv_select import KeyScores
from .pipeline import DevicePrefill, SparsityConfig, sparse_prefill_device  # noqa: F401  (re-export)

SCORE_SOURCES = ("exact", "probe")
GRANULARITIES = ("token", "block")


@dataclass
class SelectionResult:
    """Shared budget + per-group ascending index lists (kv_select.py:39-46)."""

    budget: int
    selected: list
    flattest_head: int


@dataclass
class PrefillOutput:
    """reference prefill.py:68-86 without the op counters; ``recall_per_head``
    (metrics.py:26-39, GPU LSE identity) is filled when requested."""

    outputs: list
    query_masks: list
    selection: SelectionResult
    kurtoses: list
    flattest_retained_mass: float
    flattest_total_mass: float
    score_source: str
    device: DevicePrefill | None = field(default=None, repr=False)
    key_scores: KeyScores | None = None
    recall_per_head: list | None = None

    @property
    def active_per_head(self) -> list:
        return [int(m.sum()) for m in self.query_masks]


def sparse_prefill(w: AttentionWorkload, cfg: SparsityConfig = SparsityConfig(),
                   score_source: str = "exact", with_recall: bool = False) -> PrefillOutput:
    """Query masks -> probe key scores -> flattest-group budget -> per-group
    top-b -> sparse attention (reference prefill.py:142-192 under rule B).
    The block-probe score source is the hot path; "exact" computes the
    dense causal maps' column masses on the GPU (K3x, O(N^2 d) float64)
    without materialising them."""
    if score_source not in SCORE_SOURCES:
        raise ParameterError(f"score source must be one of {SCORE_SOURCES}")
    # selection in the caller's precision (float64 for the reference's own
    # arrays), attention on bf16 copies (sparse_prefill_device converts)
    Q, K, V = w.device_tensors(w.source_dtype())
    res = sparse_prefill_device(Q, K, V, w.layout.n_vision, SparsityConfig(
        tau=cfg.tau, p=cfg.p, block_size=cfg.block_size, granularity=cfg.granularity,
        preserve_first_head=cfg.preserve_first_head, sink_index=w.layout.sink_index), score_source=score_source)
    info = res.selection.info.cpu().numpy()
    stats = res.selection.stats.cpu().numpy()
    b, flat, hkv = int(info[0]), int(info[1]), K.shape[0]
    sel = res.selection.selected.cpu().numpy()
    selected = [sel[g, :b].astype(np.int64) for g in range(hkv)]
    outs = list(res.outputs.float().cpu().numpy().astype(np.float64))
    masks = list(res.active.cpu().numpy().astype(bool))
    n = Q.shape[1]
    gs = res.selection.group_scores.cpu().numpy()
    blk = 1 if gs.shape[1] == n else cfg.block_size
    scores = [np.repeat(gs[g], blk)[:n] for g in range(hkv)]  # block-constant per-token scores
    recall = None
    if with_recall:
        from .metrics import attention_recall_device

        bf = lambda t: t.to(torch.bfloat16).contiguous()
        recall = attention_recall_device(res, bf(Q), bf(K), bf(V), w.layout.sink_index).cpu().tolist()
    return PrefillOutput(outs, masks, SelectionResult(b, selected, flat), list(stats[:hkv]), float(stats[hkv]),
                         float(stats[hkv + 1]), score_source, res, KeyScores(scores, list(stats[:hkv])), recall)


def sparse_head_attention(q, k, v, selected, active, sink_index: int):
    """One head's sparse attention (reference prefill.py:89-122): active rows
    attend causally (original positions) to ``selected`` keys, rows with no
    visible key copy ``v[sink_index]``, lazy rows are zero. Accepts NumPy or
    torch inputs ([N, d], d = 128); returns the same kind."""
    as_np = not isinstance(q, torch.Tensor)
    t = lambda x: torch.as_tensor(np.asarray(x) if as_np else x).to("cuda", torch.bfloat16).contiguous()
    Q, K, V = t(q)[None], t(k)[None], t(v)[None]
    n, d = Q.shape[1], Q.shape[2]
    if K.shape[1:] != (n, d) or V.shape[1:] != (n, d):
        raise ShapeError("q, k, v must share [N, d]")
    act = torch.as_tensor(np.asarray(active, dtype=np.uint8) if as_np else active.to(torch.uint8)).to("cuda")[None]
    sel_np = np.asarray(selected if as_np else selected.cpu(), dtype=np.int32)
    O = torch.zeros_like(Q)
    if sel_np.size == 0 or int(act.sum()) == 0:
        return O[0].float().cpu().numpy().astype(np.float64) if as_np else O[0]
    if np.any(np.diff(sel_np) <= 0) or sel_np.min() < 0 or sel_np.max() >= n:
        raise ShapeError("selected must be ascending, unique indices into the sequence")
    bact = act.sum(dim=1, dtype=torch.int32)[:, None]
    rows, counts = ops.compact_rows(act, bact, n)
    selected_t = torch.zeros(1, n, dtype=torch.int32, device="cuda")
    selected_t[0, : sel_np.size] = torch.from_numpy(sel_np).cuda()
    cnt = torch.tensor([sel_np.size], dtype=torch.int32, device="cuda")
    cap = ops.round_up(n, ops.TILE)
    Ks = ops.gather_rows(K, selected_t, cnt, cap, ops.TILE)
    Vs = ops.gather_rows(V, selected_t, cnt, cap, ops.TILE)
    ops.sparse_attn_fwd(Q, Ks, Vs, V, rows, counts, selected_t, cnt, sink_index, O, None)
    return O[0].float().cpu().numpy().astype(np.float64) if as_np else O[0]
