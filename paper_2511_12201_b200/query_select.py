"""Reference-named query-selection operators on the GPU (reference
``query_select.py:22-92``) over K1 ``omni_kv_probe`` and K2 ``omni_q_score``.
NumPy in -> NumPy out, like the reference; float64 inputs stay float64 and
all arithmetic is float64 on the device."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .attention import AttentionWorkload, TokenLayout
from .errors import LayoutError


@dataclass(frozen=True)
class ProbeKeys:
    """Sink key and vision-key mean (query_select.py:22-27)."""

    lazy_key: np.ndarray
    active_key: np.ndarray


@dataclass
class QueryMask:
    """query_select.py:30-38."""

    active: np.ndarray

    @property
    def count_active(self) -> int:
        return int(self.active.sum())


def _dev(x) -> torch.Tensor:
    """Device copy in the caller's precision (float64 NumPy arrays stay
    float64, as the reference computes; fp32 / bf16 tensors keep theirs)."""
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(x)))
    if t.dtype not in (torch.float64, torch.float32, torch.bfloat16):
        t = t.to(torch.float64)
    return t.to(device="cuda").contiguous()


def build_probe_keys(k, layout: TokenLayout) -> ProbeKeys:
    """k_lazy = K[sink], k_act = mean(K[:nv]) in float64 (query_select.py:41-47)."""
    if layout.n_vision == 0:
        raise LayoutError("probe keys need at least one vision token")
    K = _dev(k)[None]
    kl, ka, _ = ops.kv_probe(K, layout.n_vision, layout.sink_index, max(1, K.shape[1]))
    return ProbeKeys(kl[0].cpu().numpy(), ka[0].cpu().numpy())


def classify_queries(q, probes: ProbeKeys, tau: float):
    """Two-logit softmax per query row; active iff p_act > tau (strict).
    Returns (active_prob, active) (query_select.py:50-68)."""
    if not 0.0 <= tau < 1.0:
        raise ValueError(f"tau must be in [0, 1), got {tau}")
    Q = _dev(q)[None]
    n = Q.shape[1]
    kl = torch.from_numpy(np.asarray(probes.lazy_key, dtype=np.float64)).cuda()[None]
    ka = torch.from_numpy(np.asarray(probes.active_key, dtype=np.float64)).cuda()[None]
    active, p, _, _ = ops.q_score(Q, kl, ka, n, tau, False, max(1, n), want_prob=True)
    return p[0].cpu().numpy(), active[0].cpu().numpy().astype(bool)


def build_query_masks(w: AttentionWorkload, tau: float, preserve_first_head: bool = True) -> list:
    """Vision rows classified per Q head against its KV group's probe keys,
    text/answer rows active, head 0 forced active (query_select.py:71-92)."""
    if not 0.0 <= tau < 1.0:
        raise ValueError(f"tau must be in [0, 1), got {tau}")
    Q, K, _ = w.device_tensors(w.source_dtype())
    nv = w.layout.n_vision
    kl, ka, _ = ops.kv_probe(K, nv, w.layout.sink_index, 256)
    active, _, _, _ = ops.q_score(Q, kl, ka, nv, tau, preserve_first_head, 256)
    return [QueryMask(a) for a in active.cpu().numpy().astype(bool)]
