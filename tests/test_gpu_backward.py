"""Gradient parity of the sparse attention backward (K5) against the float64
torch-autograd oracle (oracle/grad.py), whose forward is pinned to the
reference's sparse_head_attention.

Tolerance: bf16 operands (Q, K, V, O, dO, P, dS) with fp32 accumulation —
max |g - g_ref| <= 2e-2 * max |g_ref| per tensor (reported in the message).
"""

import numpy as np
import pytest
import torch

from oracle import pipeline as opipe
from oracle.grad import sparse_attention_grads
from oracle.workload import Spec, generate, round_bf16

pytestmark = pytest.mark.gpu

REL = 2e-2


def dev(x, dtype=torch.bfloat16):
    return torch.tensor(np.asarray(x), dtype=dtype, device="cuda")


def rel_err(got, ref):
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


def run_case(hq, hkv, nv, nt, seed, row_sample=None, tau=0.08, p=0.82):
    from paper_2511_12201_b200.autograd import SparseAttentionFn, plan_from_selection
    from paper_2511_12201_b200.pipeline import SparsityConfig, select_device

    Q, K, V = (round_bf16(x) for x in generate(Spec(heads=hq, heads_kv=hkv, head_dim=128, n_vision=nv,
                                                        n_text=nt, seed=seed)))
    n = nv + nt
    rng = np.random.default_rng(seed)
    dO = round_bf16(rng.normal(size=Q.shape))
    if row_sample is not None:
        keep = np.zeros(n, dtype=bool)
        keep[rng.choice(n, row_sample, replace=False)] = True
        dO[:, ~keep] = 0.0
    Qd, Kd, Vd = (dev(x).requires_grad_(True) for x in (Q, K, V))
    cfg = SparsityConfig(tau=tau, p=p)
    with torch.no_grad():
        _, _, _, active, _, _, rows, counts, _, sel = select_device(Qd.detach(), Kd.detach(), nv, cfg)
    O = SparseAttentionFn.apply(Qd, Kd, Vd, plan_from_selection(rows, counts, sel, 0))
    O.backward(dev(dO))
    torch.cuda.synchronize()
    ref = opipe.select(Q, K, nv, 0, tau, p, 256)
    b = int(sel.info[0])
    assert b == ref.budget
    subset = None if row_sample is None else np.flatnonzero(keep)
    out_ref, dq_ref, dk_ref, dv_ref = sparse_attention_grads(Q, K, V, ref.selected, ref.active, 0, dO,
                                                             rows_subset=subset)
    got = [x.grad.float().cpu().numpy() for x in (Qd, Kd, Vd)]
    errs = {name: rel_err(g, r) for name, g, r in zip(("dQ", "dK", "dV"), got, (dq_ref, dk_ref, dv_ref))}
    assert all(e <= REL for e in errs.values()), errs
    assert np.all(got[0][~ref.active] == 0.0)
    if row_sample is None:
        np.testing.assert_allclose(O.detach().float().cpu().numpy(), out_ref, atol=2e-2, rtol=2e-2)
    return errs


def test_backward_gqa_small():
    run_case(8, 2, 2000, 48, seed=0)


def test_backward_mha_ragged():
    run_case(4, 4, 1500, 37, seed=3)


def test_backward_32k_row_sample():
    """C4 shapes (28 Q / 4 KV heads, 32K tokens): dO restricted to a random
    sample of rows so the float64 oracle stays tractable; dK / dV then only
    receive those rows' contributions on both sides."""
    run_case(28, 4, 32768 - 64, 64, seed=1, row_sample=192)
