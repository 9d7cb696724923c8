"""Parity report (north_star: "max-abs and relative errors reported"): one run
that measures, against the oracle (pinned to the reference), the error of every
floating-point output of the path and the decision margins of every discrete
choice, asserts the stated tolerances, and writes the numbers as JSON
(``OMNI_PARITY_OUT=<path>``; the committed copy is ``profiles/r02_parity.json``,
which bench.py quotes as its ``parity`` key).

Error definitions per tensor: ``max_abs`` = max |gpu - ref|; ``max_rel`` =
max_abs / max |ref| (normwise); ``p99_elem_rel`` = 99th percentile of
|gpu - ref| / (|ref| + 0.02) elementwise. References are float64 on the same
(bf16-rounded where the GPU consumes bf16) inputs.
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle import attention as oatt
from oracle import pipeline as opipe
from oracle.grad import sparse_attention_grads
from oracle.workload import Spec, generate, round_bf16

pytestmark = pytest.mark.gpu


def dev(x, dtype=torch.bfloat16):
    return torch.tensor(np.asarray(x), dtype=dtype, device="cuda")


def err(got, ref):
    got, ref = np.asarray(got, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    d = np.abs(got - ref)
    return {"max_abs": float(d.max()), "max_rel": float(d.max() / max(np.abs(ref).max(), 1e-30)),
            "p99_elem_rel": float(np.quantile(d / (np.abs(ref) + 0.02), 0.99))}


def test_parity_report(golden):
    from paper_2511_12201_b200 import decode as gdec
    from paper_2511_12201_b200.attention import AttentionWorkload, TokenLayout
    from paper_2511_12201_b200.autograd import SparseAttentionFn, plan_from_selection
    from paper_2511_12201_b200.kv_select import SelectionResult
    from paper_2511_12201_b200.pipeline import SparsityConfig, select_device, sparse_prefill_device

    rep = {"tolerances": {"attention_outputs": "|err| <= 0.02 + 0.02 |ref| elementwise (bf16 operands, fp32 accum)",
                          "gradients": "max_rel <= 2e-2 per tensor", "decode": "|err| <= 5e-3 + 2e-2 |ref|",
                          "selections": "bit-exact (active masks, flattest group, budget, index sets)"}}

    # ---- C1 (fp32 validation mode, MHA 4 heads, N = 2048), three seeds: outputs + LSE
    c1 = {}
    for seed in range(3):
        Q, K, V = generate(Spec(heads=4, head_dim=128, n_vision=1984, n_text=64, seed=seed))
        Q, K, V = (x.astype(np.float32).astype(np.float64) for x in (Q, K, V))
        res = sparse_prefill_device(dev(Q, torch.float32), dev(K, torch.float32), dev(V, torch.float32), 1984,
                                    SparsityConfig())
        ref = opipe.select(Q, K, 1984, 0, 0.08, 0.82, 256)
        assert int(res.selection.info[0]) == ref.budget
        Qb, Kb, Vb = round_bf16(Q), round_bf16(K), round_bf16(V)
        out = res.outputs.float().cpu().numpy()
        lse = res.lse.cpu().numpy()
        exp = np.stack([oatt.sparse_head_attention(Qb[h], Kb[h], Vb[h], ref.selected[h], ref.active[h], 0)
                        for h in range(4)])
        e = err(out, exp)
        assert e["max_abs"] <= 0.02 + 0.02 * np.abs(exp).max()
        el = np.concatenate([oatt.sparse_head_lse(Qb[h], Kb[h], ref.selected[h], ref.active[h])[ref.active[h]]
                             for h in range(4)])
        gl = np.concatenate([lse[h][ref.active[h]] for h in range(4)])
        fin = np.isfinite(el)
        c1[f"seed{seed}"] = {"outputs": e, "lse": err(gl[fin], el[fin]),
                             "budget_margin_rel": float(res.selection.stats.cpu().numpy()[6])}
    rep["c1_fp32_validation"] = c1

    # ---- C3 64K (28 / 4 heads): sampled rows of three heads + decision margins
    from paper_2511_12201_b200.synthetic import generate_device

    n, nv = 65536, 65536 - 64
    Qd, Kd, Vd = generate_device(28, 4, 128, nv, 64, seed=0)
    res = sparse_prefill_device(Qd, Kd, Vd, nv, SparsityConfig(), want_prob=True)
    host = lambda t: list(t.float().cpu().numpy().astype(np.float64))
    Qh, Kh, Vh = host(Qd), host(Kd), host(Vd)
    ref = opipe.select(Qh, Kh, nv, 0, 0.08, 0.82, 256)
    assert int(res.selection.info[0]) == ref.budget and int(res.selection.info[1]) == ref.flattest
    np.testing.assert_array_equal(res.active.cpu().numpy().astype(bool), ref.active)
    out = res.outputs.float().cpu().numpy()
    rng = np.random.default_rng(0)
    errs, stats = [], res.selection.stats.cpu().numpy()
    for h in (0, 13, 27):
        g = h // 7
        sample = np.sort(rng.choice(np.flatnonzero(ref.active[h]), 256, replace=False))
        exp = oatt.sparse_head_attention(Qh[h], Kh[g], Vh[g], ref.selected[g], ref.active[h], 0, rows_subset=sample)
        errs.append(err(out[h][sample], exp[sample]))
    p = res.p_act.cpu().numpy()
    kurt = np.sort(stats[:4])
    rep["c3_64k"] = {
        "outputs_sampled_rows": {k: max(e[k] for e in errs) for k in errs[0]},
        "p_act_vs_oracle_max_abs": float(np.abs(p - ref.p_act).max()),
        "decision_margins": {
            "budget_margin_rel_to_total": float(stats[6]), "budget_replayed": bool(stats[7]),
            "kurtosis_gap_rel": float((kurt[1] - kurt[0]) / abs(kurt[0])),
            "min_abs_p_act_minus_tau": float(np.abs(p - 0.08).min()),
        },
    }

    # ---- C4-style backward (GQA 8 / 2 heads, N = 2048) vs the float64 autograd oracle
    Q, K, V = (round_bf16(x) for x in generate(Spec(heads=8, heads_kv=2, head_dim=128, n_vision=2000, n_text=48,
                                                        seed=0)))
    dO = round_bf16(np.random.default_rng(0).normal(size=Q.shape))
    Qg, Kg, Vg = (dev(x).requires_grad_(True) for x in (Q, K, V))
    with torch.no_grad():
        _, _, _, active, _, _, rows, counts, _, sel = select_device(Qg.detach(), Kg.detach(), 2000, SparsityConfig())
    O = SparseAttentionFn.apply(Qg, Kg, Vg, plan_from_selection(rows, counts, sel, 0))
    O.backward(dev(dO))
    ref = opipe.select(Q, K, 2000, 0, 0.08, 0.82, 256)
    o_ref, dq, dk, dv = sparse_attention_grads(Q, K, V, ref.selected, ref.active, 0, dO)
    g = {"outputs": err(O.detach().float().cpu().numpy(), o_ref)}
    for name, t, r in (("dQ", Qg, dq), ("dK", Kg, dk), ("dV", Vg, dv)):
        g[name] = err(t.grad.float().cpu().numpy(), r)
        assert g[name]["max_rel"] <= 2e-2, (name, g[name])
    rep["backward_gqa_8_2_n2048"] = g

    # ---- decode: the reference's own trace through the reference-signature operators
    gt = golden("decode_trace.npz")
    spec = Spec(heads=4, head_dim=32, n_vision=256, n_text=16, seed=5)
    Q, K, V = generate(spec)
    w = AttentionWorkload(list(Q), list(K), list(V), TokenLayout(256, 16))
    b = int(gt["budget"])
    cache = gdec.build_cache(w, SelectionResult(b, [np.asarray(s, dtype=np.int64) for s in gt["vision_selected"]], 0))
    from oracle.workload import decode_inputs

    outs, flags_ok = [], True
    for i, (q, k, v) in enumerate(decode_inputs(spec, K, 8, np.random.default_rng(123))):
        o, f = gdec.decode_attention(list(q), cache, 0.08)
        flags_ok &= bool(np.array_equal(f, gt["flags"][i]))
        outs.append(np.stack(o))
        gdec.append_answer(cache, list(k), list(v))
    assert flags_ok
    rep["decode_reference_trace"] = {"outputs": err(np.stack(outs), gt["outputs"]), "flags_bit_exact": flags_ok,
                                     "fetch_log_equal": cache.fetch.vision_bytes == int(gt["vision_bytes"])
                                     and cache.fetch.text_answer_bytes == int(gt["text_answer_bytes"])}
    assert rep["decode_reference_trace"]["fetch_log_equal"]

    path = os.environ.get("OMNI_PARITY_OUT")
    if path:
        with open(path, "w") as fh:
            json.dump(rep, fh, indent=1)
