"""Rule-B composition of the reference functions (oracle; tests only).

The reference is MHA-only (``SPEC.md:145``). GQA rule B,
glue restated from ``prefill.py:160-175`` and nothing else:

* query laziness per Q head, probe keys from its KV head (group) K;
* probe block scores per Q head (Q_h against its group's K), token scores
  summed over the group's Q heads in ascending head order;
* kurtosis / flattest / budget over the Hkv group vectors;
* one top-b index set per group; every Q head of the group attends over it.

With heads_q == heads_kv every step is the reference's ``sparse_prefill``
(minus the always-on dense oracle and recall instrumentation).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2511_12201_b200.errors import ParameterError

from . import selection as sel
from .attention import causal_attention, sparse_head_attention
from .numerics import f64


@dataclass
class PrefillResult:
    active: np.ndarray            # [Hq, N] bool
    p_act: np.ndarray             # [Hq, nv] f64 active probabilities
    probes: list                  # per group (k_lazy, k_act)
    block_mass: np.ndarray | None  # [Hq, nb] probe column mass (probe path)
    group_scores: list            # per group token scores [N]
    kurtoses: list
    flattest: int
    budget: int
    retained: float
    total: float
    selected: list                # per group int64 [b]
    outputs: np.ndarray | None    # [Hq, N, d] f64


def select(Q, K, n_vision: int, sink_index: int, tau: float, p: float, block_size: int = 256,
           granularity: str = "token", preserve_first_head: bool = True, score_source: str = "probe",
           block_mass_override: np.ndarray | None = None) -> PrefillResult:
    """Masks + scores + flattest + budget + top-b under rule B."""
    hq, hkv = len(Q), len(K)
    if hq % hkv:
        raise ParameterError("heads_q must be a multiple of heads_kv")
    rep = hq // hkv
    n = np.asarray(Q[0]).shape[0]
    probes = [sel.probe_keys(K[g], n_vision, sink_index) for g in range(hkv)]
    active = np.zeros((hq, n), dtype=bool)
    p_act = np.zeros((hq, n_vision))
    for h in range(hq):
        kl, ka = probes[h // rep]
        p_act[h], verdict = sel.classify(Q[h][:n_vision], kl, ka, tau)
        active[h] = True
        active[h, :n_vision] = verdict
        if preserve_first_head and h == 0:
            active[h] = True

    mass = None
    if score_source == "probe":
        if block_mass_override is not None:
            mass = np.asarray(block_mass_override, dtype=np.float64)
        else:
            mass = np.stack([sel.block_mass(sel.probe_map(Q[h], K[h // rep], block_size)) for h in range(hq)])
        per_head = [sel.token_scores_from_blocks(mass[h], n, block_size) for h in range(hq)]
    elif score_source == "exact":
        per_head = [sel.exact_scores(causal_attention(Q[h], K[h // rep], K[h // rep])[0]) for h in range(hq)]
    else:
        raise ParameterError("score source must be one of ('exact', 'probe')")

    groups = []
    for g in range(hkv):
        acc = per_head[g * rep].copy()
        for r in range(1, rep):
            acc += per_head[g * rep + r]
        groups.append(acc)
    kurt = sel.kurtoses(groups)
    flat = sel.flattest(kurt)
    b, retained, total = sel.budget(groups[flat], p)
    if granularity == "token":
        chosen = sel.key_masks(groups, b)
    elif granularity == "block":
        chosen = sel.top_blocks(groups, b, block_size)
    else:
        raise ParameterError("granularity must be one of ('token', 'block')")
    return PrefillResult(active, p_act, probes, mass, groups, kurt, flat, b, retained, total, chosen, None)


def prefill(Q, K, V, n_vision: int, sink_index: int, tau: float, p: float, block_size: int = 256,
            granularity: str = "token", preserve_first_head: bool = True, score_source: str = "probe",
            heads: list | None = None) -> PrefillResult:
    """Full rule-B sparse prefill; ``heads`` limits which Q heads' outputs are
    computed (others stay zero) for bounded CPU samples."""
    res = select(Q, K, n_vision, sink_index, tau, p, block_size, granularity, preserve_first_head, score_source)
    hq, hkv = len(Q), len(K)
    rep = hq // hkv
    n, d = np.asarray(Q[0]).shape
    out = np.zeros((hq, n, d))
    for h in (range(hq) if heads is None else heads):
        g = h // rep
        out[h] = sparse_head_attention(Q[h], K[g], V[g], res.selected[g], res.active[h], sink_index)
    res.outputs = out
    return res


def vision_selection(res: PrefillResult, n_vision: int):
    """``kv_select.py:179-195`` on the group scores (decode hand-off)."""
    return sel.vision_keys(res.group_scores, res.budget, n_vision)


def to_f64_heads(x) -> list:
    return [f64(t) for t in x]
