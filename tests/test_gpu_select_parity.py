"""K3b parity by construction (csrc/select.cu): on identical score vectors the
GPU's kurtoses, flattest group, budget (with retained / total mass) and index
sets equal the reference's bit for bit — kurtosis in NumPy's pairwise order,
the budget replayed in the reference's sequential cumsum order whenever the
parallel scan's decision margin is inside its rounding bound — including
constructed near-ties (p * total a few ulps from a cumulative-mass step,
groups whose kurtoses differ only by summation order, tied scores), the
general (CUB-sorted) path beyond 8 groups / 1024 blocks, and the full C2/C3
shapes (32K and 128K tokens, 28/4 heads) against the oracle's selection.

The oracle (``oracle/selection.py``) is pinned to the reference's own outputs
by ``tests/test_oracle_golden.py``; its arithmetic order is the reference's
NumPy backend's (the one the golden fixtures were generated with)."""

import numpy as np
import pytest
import torch

from oracle import attention as oatt
from oracle import pipeline as opipe
from oracle import selection as osel
from oracle.numerics import kurtosis as okurt

pytestmark = pytest.mark.gpu


def rvec(rng, n):
    return np.abs(rng.standard_normal(n)) * np.exp(rng.standard_normal(n))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).cuda()


@pytest.mark.parametrize("n", [2, 7, 129, 1000, 1024, 1025, 8192, 8193, 65553])
def test_kurtosis_bit_exact(n):
    """key_scores_from_vectors: kurtoses == the reference's, bit for bit
    (cluster kernel up to 1024 tokens, general path above)."""
    from paper_2511_12201_b200.kv_select import flattest_head, key_scores_from_vectors

    rng = np.random.default_rng(n)
    vecs = [rvec(rng, n) for _ in range(3)]
    ks = key_scores_from_vectors(vecs)
    assert ks.kurtoses == [okurt(v) for v in vecs]
    assert flattest_head(ks) == osel.flattest([okurt(v) for v in vecs])


def test_flattest_among_permutations_and_copies():
    """Groups holding permutations of one vector have kurtoses that differ only
    in summation-order rounding: the GPU must pick the reference's argmin.
    Identical copies tie exactly: lowest index."""
    from paper_2511_12201_b200 import ops

    rng = np.random.default_rng(5)
    base = rvec(rng, 3000)
    vecs = [rng.permutation(base) for _ in range(6)]
    ref = [okurt(v) for v in vecs]
    assert len(set(ref)) > 1  # the orders really round differently
    sel = ops.select(dev(np.stack(vecs)), 6, 3000, 1, 0.8, "token")
    stats = sel.stats.cpu().numpy()
    assert list(stats[:6]) == ref
    assert int(sel.info[1]) == osel.flattest(ref)
    sel = ops.select(dev(np.stack([base] * 4)), 4, 3000, 1, 0.8, "token")
    assert int(sel.info[1]) == 0


def near_tie_ps(a, ks):
    """p values whose threshold p * total lands on, or one ulp either side
    of, the descending cumulative mass at the given indices."""
    cum = np.cumsum(np.sort(a)[::-1])
    total = cum[-1]
    out = []
    for k in ks:
        p0 = cum[k] / total
        out += [p0, np.nextafter(p0, 0.0), np.nextafter(p0, 1.0), cum[k - 1] / total]
    return [float(p) for p in out if 0.0 < p <= 1.0]


@pytest.mark.parametrize("n", [500, 5000, 70001])
def test_budget_near_ties_replayed_bit_exact(n):
    """budget_with_retained_mass at p values placing the threshold exactly on
    (or an ulp beside) a cumulative-mass step: b, retained and total equal the
    reference's (the margin gate fires and the sequential replay decides)."""
    from paper_2511_12201_b200 import ops

    rng = np.random.default_rng(n)
    a = rvec(rng, n)
    ps = near_tie_ps(a, [n // 3, n // 2, (9 * n) // 10]) + [1.0]
    replays = 0
    for p in ps:
        sel = ops.select(dev(a[None]), 1, n, 1, p, "token")
        stats = sel.stats.cpu().numpy()
        b, retained, total = osel.budget(a, p)
        assert int(sel.info[0]) == b, p
        if stats[4] == 1.0:
            replays += 1
            assert (stats[1], stats[2]) == (retained, total), p
        else:  # decided by the fast scan: the margin exceeded the rounding bound
            assert stats[3] > (4 * n + 16) * 2.0 ** -53
            np.testing.assert_allclose(stats[1:3], [retained, total], rtol=1e-12)
        np.testing.assert_array_equal(sel.selected[0, :b].cpu().numpy(), osel.top_b(a, b))
    assert replays >= len(ps) // 2  # the constructed ties really exercise the replay


def test_budget_random_p_fast_path_matches():
    from paper_2511_12201_b200.kv_select import budget_with_retained_mass

    rng = np.random.default_rng(9)
    for _ in range(10):
        n = int(rng.integers(10, 20000))
        a = rvec(rng, n)
        p = float(rng.uniform(0.05, 0.99))
        b, retained, total = budget_with_retained_mass(a, p)
        rb, rr, rt = osel.budget(a, p)
        assert b == rb
        np.testing.assert_allclose([retained, total], [rr, rt], rtol=1e-12)


@pytest.mark.parametrize("hq,hkv,nb,B", [(8, 2, 64, 256), (28, 4, 256, 256), (6, 6, 300, 7), (12, 12, 40, 16)])
def test_probe_path_selection_bit_exact_on_identical_masses(hq, hkv, nb, B):
    """ops.select on given per-Q-head block masses (the probe path's K3b input)
    vs the rule-B composition of the reference functions on the same masses:
    kurtoses bit-exact, flattest / budget / index sets identical, including p
    at near-tie points of the flattest group (cluster kernel for <= 8 groups,
    general path for 12 groups)."""
    from paper_2511_12201_b200 import ops

    rng = np.random.default_rng(hq * 1000 + nb)
    n = nb * B - (B // 3)  # short last block
    mass = np.abs(rng.standard_normal((hq, nb))) * np.exp(rng.standard_normal((hq, nb)))
    rep = hq // hkv
    per_head = [osel.token_scores_from_blocks(mass[h], n, B) for h in range(hq)]
    groups = []
    for g in range(hkv):
        acc = per_head[g * rep].copy()
        for r in range(1, rep):
            acc += per_head[g * rep + r]
        groups.append(acc)
    kurt = osel.kurtoses(groups)
    flat = osel.flattest(kurt)
    ps = [0.82, 0.5] + near_tie_ps(groups[flat], [n // 4, n // 2])
    for p in ps:
        for gran in ("token", "block"):
            sel = ops.select(dev(mass), hkv, n, B, p, gran)
            info, stats = sel.info.cpu().numpy(), sel.stats.cpu().numpy()
            assert list(stats[:hkv]) == kurt
            assert int(info[1]) == flat
            b = osel.budget(groups[flat], p)[0]
            assert int(info[0]) == b, (p, gran)
            exp = osel.key_masks(groups, b) if gran == "token" else osel.top_blocks(groups, b, B)
            got = sel.selected.cpu().numpy()
            for g in range(hkv):
                np.testing.assert_array_equal(got[g, :b], exp[g], err_msg=f"p={p} {gran} group {g}")


def test_ties_top_b_blocks_vision_and_long_token_path():
    """Tied scores (integers), select_top_blocks with a short last block, the
    vision-limited selection and a 40K-token token-level selection (general
    path; the exact score source's selection at C2 sizes)."""
    from paper_2511_12201_b200.kv_select import (KeyScores, build_key_masks, select_top_blocks, select_vision_keys,
                                                 top_b_indices)

    rng = np.random.default_rng(3)
    a = rng.integers(0, 5, 777).astype(np.float64)
    for b in (1, 100, 500, 777):
        np.testing.assert_array_equal(top_b_indices(a, b), osel.top_b(a, b))
    vecs = [rng.integers(0, 4, 1003).astype(np.float64) for _ in range(3)]
    ks = KeyScores(vecs, [okurt(v) for v in vecs])
    for b in (5, 333, 1003):
        got = select_top_blocks(ks, b, 7)
        for g, e in zip(got.selected, osel.top_blocks(vecs, b, 7)):
            np.testing.assert_array_equal(g, e)
    long = [rvec(rng, 40000) for _ in range(4)]
    ks = KeyScores(long, [okurt(v) for v in long])
    got = build_key_masks(ks, 17000)
    for g, e in zip(got.selected, osel.key_masks(long, 17000)):
        np.testing.assert_array_equal(g, e)
    got = select_vision_keys(ks, 30000, 25000)
    bb, exp = osel.vision_keys(long, 30000, 25000)
    assert got.budget == bb
    for g, e in zip(got.selected, exp):
        np.testing.assert_array_equal(g, e)


@pytest.mark.parametrize("n", [32768, 131072])
def test_full_size_selection_and_outputs_vs_oracle(n):
    """C2 (32K) and C3 upper (128K), 28/4 heads, reference defaults: active
    masks, flattest group, budget and all index sets bit-exact vs the oracle's
    selection on the same bf16 tensors (float64 on both sides); masses and
    kurtoses within 1e-10; sampled output rows of three heads within the bf16
    tolerance; the budget decision's margin is reported in stats."""
    from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device
    from paper_2511_12201_b200.synthetic import generate_device

    nt = 64
    nv = n - nt
    Q, K, V = generate_device(28, 4, 128, nv, nt, seed=0)
    res = sparse_prefill_device(Q, K, V, nv, SparsityConfig())
    torch.cuda.synchronize()
    host = lambda t: list(t.float().cpu().numpy().astype(np.float64))
    Qh, Kh, Vh = host(Q), host(K), host(V)
    del Q, K, V
    ref = opipe.select(Qh, Kh, nv, 0, 0.08, 0.82, 256)
    np.testing.assert_array_equal(res.active.cpu().numpy().astype(bool), ref.active)
    info = res.selection.info.cpu().numpy()
    assert int(info[1]) == ref.flattest and int(info[0]) == ref.budget
    sel = res.selection.selected.cpu().numpy()
    for g in range(4):
        np.testing.assert_array_equal(sel[g, : ref.budget], ref.selected[g])
    stats = res.selection.stats.cpu().numpy()
    np.testing.assert_allclose(stats[:4], ref.kurtoses, rtol=1e-10)
    np.testing.assert_allclose(res.block_mass.cpu().numpy(), ref.block_mass, rtol=1e-10, atol=1e-13)
    assert stats[6] > 0.0  # decision margin (relative to the total mass)
    out = res.outputs.float().cpu().numpy()
    rng = np.random.default_rng(n)
    for h in (0, 13, 27):
        g = h // 7
        rows = np.flatnonzero(ref.active[h])
        sample = np.sort(rng.choice(rows, 256, replace=False))
        exp = oatt.sparse_head_attention(Qh[h], Kh[g], Vh[g], ref.selected[g], ref.active[h], 0, rows_subset=sample)
        np.testing.assert_allclose(out[h][sample], exp[sample], atol=2e-2, rtol=2e-2)
        lazy = ~ref.active[h]
        assert not out[h][lazy].any()


def test_float64_workload_selects_in_float64():
    """A float64 workload (the reference's own arrays, unrounded) selects in
    float64 on the device: masks, budget and index sets equal the oracle's on
    the unrounded inputs (no silent fp32 / bf16 rounding before
    the decisions)."""
    from oracle.workload import Spec, generate
    from paper_2511_12201_b200.attention import AttentionWorkload, TokenLayout
    from paper_2511_12201_b200.pipeline import SparsityConfig
    from paper_2511_12201_b200.prefill import sparse_prefill

    Q, K, V = generate(Spec(heads=4, head_dim=128, n_vision=1984, n_text=64, seed=7))
    w = AttentionWorkload(list(Q), list(K), list(V), TokenLayout(1984, 64))
    out = sparse_prefill(w, SparsityConfig(), score_source="probe")
    ref = opipe.select(Q, K, 1984, 0, 0.08, 0.82, 256)
    np.testing.assert_array_equal(np.stack(out.query_masks), ref.active)
    assert out.selection.budget == ref.budget and out.selection.flattest_head == ref.flattest
    for g in range(4):
        np.testing.assert_array_equal(out.selection.selected[g], ref.selected[g])
    np.testing.assert_allclose(out.kurtoses, ref.kurtoses, rtol=1e-12)
