"""Generate golden fixtures by running the REFERENCE package itself.

Runs only in the build container, where ``/root/reference`` exists (it never
travels to the GPU box). Imports the reference ``slimattn`` package read-only
(``PYTHONDONTWRITEBYTECODE``; NumPy kernel core, which the survey measured to
give bit-identical selections to the Cython core) and writes
``tests/golden/*.npz``. The fixtures pin the NumPy restatement in ``oracle/``:

* ``c1_seed{0,1,2}.npz`` — config C1 (4 MHA heads, d=128, nv=1984, nt=64,
  fp32-rounded inputs, tau=0.08, p=0.82, B=256, probe scores): input digests,
  active masks, probe block masses, kurtoses, flattest head, budget, selected
  index sets, per-head output checksums and sampled output rows.
* ``tiny_paths.npz`` — small MHA workload through the exact score path (token
  and block granularity) and the probe path with B=16, full outputs.
* ``decode_trace.npz`` — select_vision_keys -> build_cache -> 8 decode steps
  with appends, flags, outputs and fetch-log totals.
* ``gqa_seed{0,1}.npz`` — rule-B composition of reference functions on the
  restated GQA generator (Hq=8, Hkv=2, d=64, N=4096): masks, block masses,
  group kurtoses, flattest, budget, selections, output checksums/samples.

Usage: ``python tests/golden/make_golden.py`` from the repo root.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ["SLIMATTN_KERNELS"] = "py"
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from slimattn import attention as r_att  # noqa: E402
from slimattn import block_probe as r_bp  # noqa: E402
from slimattn import decode as r_dec  # noqa: E402
from slimattn import kv_select as r_kv  # noqa: E402
from slimattn import prefill as r_pf  # noqa: E402
from slimattn import query_select as r_qs  # noqa: E402
from slimattn import workload as r_wl  # noqa: E402

from oracle.workload import Spec, generate  # noqa: E402  (GQA generator; its MHA reduction is pinned below)


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def sample_rows(n: int, count: int = 16) -> np.ndarray:
    return np.unique(np.linspace(0, n - 1, count).astype(np.int64))


def to_workload(Q, K, V, nv, nt, sink=0):
    layout = r_att.TokenLayout(nv, nt, 0, sink)
    return r_att.AttentionWorkload([np.array(q) for q in Q], [np.array(k) for k in K], [np.array(v) for v in V], layout)


def c1(seed: int) -> None:
    spec = r_wl.WorkloadSpec(heads=4, head_dim=128, n_vision=1984, n_text=64, seed=seed)
    w = r_wl.generate_workload(spec)
    raw_digest = digest(*w.queries, *w.keys, *w.values)
    Q = np.stack(w.queries).astype(np.float32).astype(np.float64)
    K = np.stack(w.keys).astype(np.float32).astype(np.float64)
    V = np.stack(w.values).astype(np.float32).astype(np.float64)
    wf = to_workload(Q, K, V, 1984, 64)
    cfg = r_pf.SparsityConfig()
    masks = r_qs.build_query_masks(wf, cfg.tau, cfg.preserve_first_head)
    p_act = np.stack([r_qs.classify_queries(q[:1984], r_qs.build_probe_keys(k, wf.layout), cfg.tau)[0]
                      for q, k in zip(wf.queries, wf.keys)])
    pmaps = [r_bp.probe_attention(q, k, cfg.block_size) for q, k in zip(wf.queries, wf.keys)]
    mass = np.stack([r_kv.colsum(pm.attention) for pm in pmaps])
    scores = r_pf.compute_key_scores(wf, cfg, "probe", [], r_pf.OpCounter())
    flat = r_kv.flattest_head(scores)
    b, retained, total = r_kv.budget_with_retained_mass(scores.scores[flat], cfg.p)
    selection = r_kv.build_key_masks(scores, b)
    outs = np.stack([r_pf.sparse_head_attention(q, k, v, s, m.active, 0)
                     for q, k, v, s, m in zip(wf.queries, wf.keys, wf.values, selection.selected, masks)])
    rows = sample_rows(2048, 24)
    np.savez_compressed(
        os.path.join(HERE, f"c1_seed{seed}.npz"),
        seed=seed, raw_digest=raw_digest, f32_digest=digest(Q.astype(np.float32), K.astype(np.float32), V.astype(np.float32)),
        active=np.packbits(np.stack([m.active for m in masks]), axis=1), n=2048,
        p_act=p_act, block_mass=mass, kurtoses=np.array(scores.kurtoses), flattest=flat,
        budget=b, retained=retained, total=total,
        selected=np.stack(selection.selected).astype(np.int32),
        out_sum=outs.sum(axis=(1, 2)), out_sq=(outs * outs).sum(axis=(1, 2)),
        rows=rows, out_rows=outs[:, rows, :],
    )


def tiny_paths() -> None:
    spec = r_wl.WorkloadSpec(heads=4, head_dim=32, n_vision=120, n_text=8, seed=11)
    w = r_wl.generate_workload(spec)
    res = {}
    for tag, source, gran, block in (("exact_token", "exact", "token", 16), ("exact_block", "exact", "block", 16),
                                     ("probe_token", "probe", "token", 16), ("probe_b1", "probe", "token", 1)):
        cfg = r_pf.SparsityConfig(block_size=block, granularity=gran)
        out = r_pf.sparse_prefill(w, cfg, source)
        res[f"{tag}_outputs"] = np.stack(out.outputs)
        res[f"{tag}_selected"] = np.stack(out.selection.selected).astype(np.int32)
        res[f"{tag}_budget"] = out.selection.budget
        res[f"{tag}_flattest"] = out.selection.flattest_head
        res[f"{tag}_kurtoses"] = np.array(out.key_scores.kurtoses)
        res[f"{tag}_scores"] = np.stack(out.key_scores.scores)
        res[f"{tag}_active"] = np.stack([m.active for m in out.query_masks])
        res[f"{tag}_recall"] = np.array(out.recall_per_head)
        res[f"{tag}_retained"] = out.flattest_retained_mass
    # AC1: tau=0, p=1 -> sparse == dense oracle
    cfg = r_pf.SparsityConfig(tau=0.0, p=1.0, block_size=16)
    out = r_pf.sparse_prefill(w, cfg, "exact")
    res["ac1_outputs"] = np.stack(out.outputs)
    res["dense_outputs"] = np.stack(r_att.full_multihead(w, causal=True).head_outputs)
    np.savez_compressed(os.path.join(HERE, "tiny_paths.npz"), digest=digest(*w.queries, *w.keys, *w.values), **res)


def decode_trace() -> None:
    spec = r_wl.WorkloadSpec(heads=4, head_dim=32, n_vision=256, n_text=16, seed=5)
    w = r_wl.generate_workload(spec)
    cfg = r_pf.SparsityConfig(block_size=16)
    pre = r_pf.sparse_prefill(w, cfg, "probe")
    vsel = r_kv.select_vision_keys(pre.key_scores, pre.selection.budget, 256)
    cache = r_dec.build_cache(w, vsel, True)
    rng = np.random.default_rng(123)
    steps = r_wl.generate_decode_inputs(spec, w, 8, rng)
    flags, outs = [], []
    for q, k, v in steps:
        o, f = r_dec.decode_attention(q, cache, cfg.tau)
        flags.append(f)
        outs.append(np.stack(o))
        r_dec.append_answer(cache, k, v)
    log = cache.fetch
    totals = (log.vision_tokens, log.vision_bytes, log.text_answer_bytes,
              np.array(log.step_vision_tokens), np.array(log.step_active_heads))
    forced = np.array([True, False, True, False])
    o_forced, _ = r_dec.decode_attention(steps[0][0], cache, cfg.tau, flags=forced)
    o_dense = r_dec.decode_attention_dense(steps[0][0], cache, forced)
    o_zero = r_dec.decode_attention_dense(steps[0][0], cache, forced, zero_masked_vision=True)
    np.savez_compressed(
        os.path.join(HERE, "decode_trace.npz"),
        budget=vsel.budget, vision_selected=np.stack(vsel.selected).astype(np.int32),
        flags=np.stack(flags), outputs=np.stack(outs),
        queries=np.stack([np.stack(s[0]) for s in steps]),
        vision_tokens=totals[0], vision_bytes=totals[1], text_answer_bytes=totals[2],
        step_vision_tokens=totals[3], step_active_heads=totals[4],
        forced_outputs=np.stack(o_forced), forced_dense=np.stack(o_dense), forced_zeroed=np.stack(o_zero),
    )


def gqa(seed: int) -> None:
    hq, hkv, d, nv, nt, B = 8, 2, 64, 4032, 64, 256
    Q, K, V = generate(Spec(heads=hq, heads_kv=hkv, head_dim=d, n_vision=nv, n_text=nt, seed=seed))
    n, rep = nv + nt, hq // hkv
    layout = r_att.TokenLayout(nv, nt, 0, 0)
    tau, p = 0.08, 0.82
    probes = [r_qs.build_probe_keys(K[g], layout) for g in range(hkv)]
    active, pacts, per_head, mass = [], [], [], []
    for h in range(hq):
        pa, verdict = r_qs.classify_queries(Q[h][:nv], probes[h // rep], tau)
        a = np.ones(n, dtype=bool)
        a[:nv] = verdict
        if h == 0:
            a[:] = True
        active.append(a)
        pacts.append(pa)
        pm = r_bp.probe_attention(Q[h], K[h // rep], B)
        mass.append(r_kv.colsum(pm.attention))
        per_head.append(r_bp.block_scores_to_token_scores(pm, n))
    groups = []
    for g in range(hkv):
        acc = per_head[g * rep].copy()
        for r in range(1, rep):
            acc += per_head[g * rep + r]
        groups.append(acc)
    ks = r_kv.key_scores_from_vectors(groups)
    flat = r_kv.flattest_head(ks)
    b, retained, total = r_kv.budget_with_retained_mass(ks.scores[flat], p)
    selection = r_kv.build_key_masks(ks, b)
    outs = np.stack([r_pf.sparse_head_attention(Q[h], K[h // rep], V[h // rep], selection.selected[h // rep], active[h], 0)
                     for h in range(hq)])
    vsel = r_kv.select_vision_keys(ks, b, nv)
    rows = sample_rows(n, 24)
    np.savez_compressed(
        os.path.join(HERE, f"gqa_seed{seed}.npz"),
        seed=seed, digest=digest(Q, K, V), active=np.packbits(np.stack(active), axis=1), n=n,
        p_act=np.stack(pacts), block_mass=np.stack(mass), kurtoses=np.array(ks.kurtoses), flattest=flat,
        budget=b, retained=retained, total=total, selected=np.stack(selection.selected).astype(np.int32),
        vision_budget=vsel.budget, vision_selected=np.stack(vsel.selected).astype(np.int32),
        out_sum=outs.sum(axis=(1, 2)), out_sq=(outs * outs).sum(axis=(1, 2)), rows=rows, out_rows=outs[:, rows, :],
    )


if __name__ == "__main__":
    for s in (0, 1, 2):
        c1(s)
    tiny_paths()
    decode_trace()
    for s in (0, 1):
        gqa(s)
    print("golden fixtures written to", HERE)
