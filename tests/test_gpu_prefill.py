"""GPU parity of the sparse prefill path (K1-K4) against the CPU oracle.

Selections (active masks, flattest group, budget, index sets) must be
bit-exact; probabilities / masses / kurtoses within 1e-10 relative (float64
on both sides, different summation order); attention outputs within the bf16
tolerance ATOL/RTOL below (bf16 operands, fp32 accumulation, bf16 output vs a
float64 oracle on the same bf16-rounded inputs).
"""

import numpy as np
import pytest
import torch

from oracle import attention as oatt
from oracle import pipeline as opipe
from oracle.workload import Spec, generate, round_bf16

pytestmark = pytest.mark.gpu

ATOL, RTOL = 2e-2, 2e-2


def to_dev(x, dtype=torch.bfloat16):
    return torch.tensor(np.asarray(x), dtype=dtype, device="cuda")


def check_selection(res, ref, hkv):
    np.testing.assert_array_equal(res.active.cpu().numpy().astype(bool), ref.active)
    info = res.selection.info.cpu().numpy()
    assert int(info[1]) == ref.flattest
    assert int(info[0]) == ref.budget
    np.testing.assert_array_equal(info[4:], ref.budget)
    sel = res.selection.selected.cpu().numpy()
    for g in range(hkv):
        np.testing.assert_array_equal(sel[g, : ref.budget], ref.selected[g])
    stats = res.selection.stats.cpu().numpy()
    np.testing.assert_allclose(stats[:hkv], ref.kurtoses, rtol=1e-10)
    np.testing.assert_allclose(res.block_mass.cpu().numpy(), ref.block_mass, rtol=1e-10, atol=1e-13)


def check_outputs(res, Q, K, V, ref, heads, sink=0):
    out = res.outputs.float().cpu().numpy()
    hq, hkv = len(Q), len(K)
    rep = hq // hkv
    for h in heads:
        g = h // rep
        exp = oatt.sparse_head_attention(Q[h], K[g], V[g], ref.selected[g], ref.active[h], sink)
        np.testing.assert_allclose(out[h], exp, atol=ATOL, rtol=RTOL, err_msg=f"head {h}")
        lazy = ~ref.active[h]
        assert np.all(out[h][lazy] == 0.0)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_c1_fp32_validation_mode(golden, seed):
    """C1: 4 MHA heads, d=128, N=2048, fp32 inputs -> bit-exact selections vs
    the reference fixtures; outputs within bf16 tolerance."""
    from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device

    g = golden(f"c1_seed{seed}.npz")
    Q, K, V = generate(Spec(heads=4, head_dim=128, n_vision=1984, n_text=64, seed=seed))
    Q, K, V = (x.astype(np.float32).astype(np.float64) for x in (Q, K, V))
    res = sparse_prefill_device(to_dev(Q, torch.float32), to_dev(K, torch.float32), to_dev(V, torch.float32), 1984,
                                SparsityConfig(), want_prob=True)
    torch.cuda.synchronize()
    act = np.unpackbits(g["active"], axis=1)[:, :2048].astype(bool)
    np.testing.assert_array_equal(res.active.cpu().numpy().astype(bool), act)
    np.testing.assert_allclose(res.p_act.cpu().numpy(), g["p_act"], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(res.block_mass.cpu().numpy(), g["block_mass"], rtol=1e-10)
    info = res.selection.info.cpu().numpy()
    assert int(info[0]) == int(g["budget"]) and int(info[1]) == int(g["flattest"])
    np.testing.assert_allclose(res.selection.stats.cpu().numpy()[:4], g["kurtoses"], rtol=1e-10)
    np.testing.assert_allclose(res.selection.stats.cpu().numpy()[4], float(g["retained"]), rtol=1e-9)
    sel = res.selection.selected.cpu().numpy()[:, : int(g["budget"])]
    np.testing.assert_array_equal(sel, g["selected"])
    # attention consumes the bf16-rounded tensors: compare against the oracle on those
    Qb, Kb, Vb = round_bf16(Q), round_bf16(K), round_bf16(V)
    out = res.outputs.float().cpu().numpy()
    for h in range(4):
        exp = oatt.sparse_head_attention(Qb[h], Kb[h], Vb[h], g["selected"][h], act[h], 0)
        np.testing.assert_allclose(out[h], exp, atol=ATOL, rtol=RTOL)
    # and the fixture's float64 reference outputs (fp32 inputs) sit within the same band
    np.testing.assert_allclose(out[:, g["rows"], :], g["out_rows"], atol=ATOL, rtol=RTOL)


@pytest.mark.parametrize("n_vision,n_text,seed", [(8128, 64, 0), (8000, 77, 3), (3001, 50, 1)])
def test_gqa_rule_b_bf16(n_vision, n_text, seed):
    """Qwen2-7B head layout (28 Q / 4 KV, d=128), bf16; ragged N exercises
    short probe blocks and partial 128-row tiles."""
    from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device

    Q, K, V = generate(Spec(heads=28, heads_kv=4, head_dim=128, n_vision=n_vision, n_text=n_text, seed=seed))
    Q, K, V = round_bf16(Q), round_bf16(K), round_bf16(V)
    res = sparse_prefill_device(to_dev(Q), to_dev(K), to_dev(V), n_vision, SparsityConfig())
    torch.cuda.synchronize()
    ref = opipe.select(Q, K, n_vision, 0, 0.08, 0.82, 256)
    check_selection(res, ref, 4)
    check_outputs(res, Q, K, V, ref, heads=[0, 6, 7, 27])


def test_block_granularity_and_second_operating_point():
    from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device

    Q, K, V = generate(Spec(heads=8, heads_kv=2, head_dim=128, n_vision=4000, n_text=96, seed=7, lazy_fraction=0.7))
    Q, K, V = round_bf16(Q), round_bf16(K), round_bf16(V)
    for cfg in (SparsityConfig(tau=0.12, p=0.75), SparsityConfig(granularity="block"),
                SparsityConfig(block_size=64), SparsityConfig(preserve_first_head=False)):
        res = sparse_prefill_device(to_dev(Q), to_dev(K), to_dev(V), 4000, cfg)
        torch.cuda.synchronize()
        ref = opipe.select(Q, K, 4000, 0, cfg.tau, cfg.p, cfg.block_size, cfg.granularity, cfg.preserve_first_head)
        check_selection(res, ref, 2)
        check_outputs(res, Q, K, V, ref, heads=[1, 4])


def test_sparsity_disabled_equals_dense_causal():
    """AC1 on the GPU: tau=0, p=1 -> dense causal attention."""
    from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device

    Q, K, V = generate(Spec(heads=4, heads_kv=2, head_dim=128, n_vision=1000, n_text=24, seed=2))
    Q, K, V = round_bf16(Q), round_bf16(K), round_bf16(V)
    res = sparse_prefill_device(to_dev(Q), to_dev(K), to_dev(V), 1000, SparsityConfig(tau=0.0, p=1.0))
    torch.cuda.synchronize()
    assert int(res.selection.info[0]) == 1024
    assert bool(res.active.all())
    out = res.outputs.float().cpu().numpy()
    for h in range(4):
        _, dense = oatt.causal_attention(Q[h], K[h // 2], V[h // 2])
        np.testing.assert_allclose(out[h], dense, atol=ATOL, rtol=RTOL)


def test_sink_fallback_rows_and_tiny_budget():
    """Rows whose causal range holds no selected key copy V[sink]
    (prefill.py:119-120); exercised with a hand-made selection."""
    from paper_2511_12201_b200 import ops

    rng = np.random.default_rng(0)
    hq, hkv, n, d = 4, 2, 700, 128
    Q, K, V = (round_bf16(rng.normal(size=s)) for s in ((hq, n, d), (hkv, n, d), (hkv, n, d)))
    active = rng.random((hq, n)) < 0.6
    sel = [np.array([130, 131, 400, 555], dtype=np.int64), np.arange(300, 560, dtype=np.int64)]
    sink = 3
    Qd, Kd, Vd = to_dev(Q), to_dev(K), to_dev(V)
    a = torch.tensor(active.astype(np.uint8), device="cuda")
    bact = torch.tensor(active.reshape(hq, -1).sum(axis=1, keepdims=True).astype(np.int32), device="cuda")
    rows, counts = ops.compact_rows(a, bact, n)
    selected = torch.zeros(hkv, n, dtype=torch.int32, device="cuda")
    cnts = torch.tensor([len(s) for s in sel], dtype=torch.int32, device="cuda")
    for g in range(hkv):
        selected[g, : len(sel[g])] = torch.tensor(sel[g], dtype=torch.int32)
    cap = ops.round_up(n, 128)
    Ks = ops.gather_rows(Kd, selected, cnts, cap, 128)
    Vs = ops.gather_rows(Vd, selected, cnts, cap, 128)
    O = torch.zeros_like(Qd)
    lse = torch.empty(hq, n, device="cuda", dtype=torch.float32)
    ops.sparse_attn_fwd(Qd, Ks, Vs, Vd, rows, counts, selected, cnts, sink, O, lse)
    torch.cuda.synchronize()
    out = O.float().cpu().numpy()
    for h in range(hq):
        exp = oatt.sparse_head_attention(Q[h], K[h // 2], V[h // 2], sel[h // 2], active[h], sink)
        np.testing.assert_allclose(out[h], exp, atol=ATOL, rtol=RTOL)
        ref_lse = oatt.sparse_head_lse(Q[h], K[h // 2], sel[h // 2], active[h])
        got = lse.cpu().numpy()[h]
        fin = np.isfinite(ref_lse)
        np.testing.assert_allclose(got[fin], ref_lse[fin], atol=2e-3, rtol=1e-3)
        fallback = active[h] & ~fin
        assert np.all(np.isneginf(got[fallback]))


def test_64k_qwen2_selection_bit_exact():
    """Full-size C3 shapes (28/4 heads, 64K tokens): selections bit-exact vs the
    oracle's selection path; attention checked on a row sample of two heads."""
    from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device

    nv, nt = 65536 - 64, 64
    Q, K, V = generate(Spec(heads=28, heads_kv=4, head_dim=128, n_vision=nv, n_text=nt, seed=0))
    Q, K, V = round_bf16(Q), round_bf16(K), round_bf16(V)
    res = sparse_prefill_device(to_dev(Q), to_dev(K), to_dev(V), nv, SparsityConfig())
    torch.cuda.synchronize()
    ref = opipe.select(Q, K, nv, 0, 0.08, 0.82, 256)
    check_selection(res, ref, 4)
    out = res.outputs.float().cpu().numpy()
    sample = np.sort(np.random.default_rng(1).choice(65536, 512, replace=False))
    for h in (0, 13):
        g = h // 7
        exp = oatt.sparse_head_attention(Q[h], K[g], V[g], ref.selected[g], ref.active[h], 0, rows_subset=sample)
        np.testing.assert_allclose(out[h][sample], exp[sample], atol=ATOL, rtol=RTOL)


@pytest.mark.parametrize("tag,gran", [("exact_token", "token"), ("exact_block", "block")])
def test_exact_score_source_matches_reference_fixture(golden, tag, gran):
    """score_source='exact' (K3x two-pass column mass, f64) reproduces the
    reference's exact-path selections bit for bit (tests/golden/tiny_paths)."""
    from paper_2511_12201_b200.pipeline import SparsityConfig, select_device

    g = golden("tiny_paths.npz")
    Q, K, V = generate(Spec(heads=4, head_dim=32, n_vision=120, n_text=8, seed=11))
    cfg = SparsityConfig(block_size=16, granularity=gran)
    out = select_device(to_dev(Q, torch.float32), to_dev(K, torch.float32), 120, cfg, score_source="exact")
    active, mass, sel = out[3], out[8], out[9]
    torch.cuda.synchronize()
    np.testing.assert_array_equal(active.cpu().numpy().astype(bool), g[f"{tag}_active"])
    # The fixture ran on the unrounded float64 workload; the GPU consumes the
    # fp32-rounded copy, so the masses agree to fp32 input rounding (~1e-7)
    # with the fixture and to 1e-10 with the oracle on the rounded inputs.
    np.testing.assert_allclose(mass.cpu().numpy(), g[f"{tag}_scores"], rtol=1e-6, atol=1e-12)
    Qr, Kr = [x.astype(np.float32).astype(np.float64) for x in (Q, K)]
    ref = opipe.select(Qr, Kr, 120, 0, 0.08, 0.82, 16, granularity=gran, score_source="exact")
    np.testing.assert_allclose(mass.cpu().numpy(), np.stack(ref.group_scores), rtol=1e-10, atol=1e-13)
    b = int(sel.info[0])
    assert b == int(g[f"{tag}_budget"]) and int(sel.info[1]) == int(g[f"{tag}_flattest"])
    np.testing.assert_array_equal(sel.selected[:, :b].cpu().numpy(), g[f"{tag}_selected"])


def test_exact_score_source_c1_end_to_end():
    """C1 shape through sparse_prefill(score_source='exact') vs the oracle."""
    from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device

    Q, K, V = generate(Spec(heads=4, head_dim=128, n_vision=1984, n_text=64, seed=1))
    Q, K, V = round_bf16(Q), round_bf16(K), round_bf16(V)
    res = sparse_prefill_device(to_dev(Q), to_dev(K), to_dev(V), 1984, SparsityConfig(), score_source="exact")
    torch.cuda.synchronize()
    ref = opipe.select(Q, K, 1984, 0, 0.08, 0.82, 256, score_source="exact")
    assert int(res.selection.info[0]) == ref.budget and int(res.selection.info[1]) == ref.flattest
    sel = res.selection.selected.cpu().numpy()
    for g in range(4):
        np.testing.assert_array_equal(sel[g, : ref.budget], ref.selected[g])
    check_outputs(res, Q, K, V, ref, heads=[0, 3])


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_q_score_decision_at_the_boundary(dtype):
    """K2 decides far from the boundary on l1 - l0 vs ln(tau/(1-tau)) and
    evaluates the reference expression (query_select.py:63-68) near it. tau
    is set to the ORACLE's p_act of sample rows (the hardest ties). Every row
    whose oracle p is farther from tau than the measured GPU-vs-oracle p
    difference gets the oracle's verdict; the only rows allowed to differ are
    those within that arithmetic difference of tau (the tie rows themselves)."""
    from paper_2511_12201_b200 import ops

    Q, K, V = generate(Spec(heads=4, heads_kv=2, head_dim=128, n_vision=3000, n_text=40, seed=11))
    Qr, Kr = round_bf16(Q), round_bf16(K)
    Qd, Kd = to_dev(Qr, dtype), to_dev(Kr, dtype)
    kl, ka, _ = ops.kv_probe(Kd, 3000, 0, 256)
    _, p, _, _ = ops.q_score(Qd, kl, ka, 3000, 0.08, False, 256, want_prob=True)
    p = p.cpu().numpy()
    ref = opipe.select(Qr, Kr, 3000, 0, 0.08, 0.82, 256, preserve_first_head=False)
    p_ref = ref.p_act
    diff = float(np.max(np.abs(p - p_ref)))
    assert diff < 1e-12
    for r in (5, 777, 2999):
        tau = float(p_ref[1, r])
        if not 0.0 < tau < 1.0:
            continue
        act, _, _, _ = ops.q_score(Qd, kl, ka, 3000, tau, False, 256)
        got = act.cpu().numpy()[:, :3000].astype(bool)
        exp = p_ref > tau
        clear = np.abs(p_ref - tau) > 2 * diff
        np.testing.assert_array_equal(got[clear], exp[clear])
        # rows in the ambiguous band: the GPU's verdict is its own p > tau
        np.testing.assert_array_equal(got[~clear], p[~clear] > tau)
        assert int((~clear).sum()) <= 4


@pytest.mark.parametrize("seed", [0, 5])
def test_q_score_fast_kernel_equals_float64_verdicts(seed):
    """The hot-path K2 (fp32 dot product with a rigorous error bound, float64
    re-evaluation inside it) gives exactly the verdicts p_act > tau of the
    float64 kernel (want_prob path, query_select.py:63-68) on every row —
    including taus placed ON rows' p (exact ties: the bound must route them to
    the float64 evaluation) and the lazy-row zeroing of O."""
    from paper_2511_12201_b200 import ops
    from paper_2511_12201_b200.synthetic import generate_device

    n, nv = 16384, 16384 - 64
    Q, K, _ = generate_device(28, 4, 128, nv, 64, seed=seed, lazy_fraction=0.5)
    kl, ka, pk = ops.kv_probe(K, nv, 0, 256)
    _, p, pooled_ref, bact_ref = ops.q_score(Q, kl, ka, nv, 0.08, True, 256, want_prob=True)
    pc = p.cpu().numpy()
    taus = [0.08, 0.5, float(pc[3, 100]), float(pc[17, 9000]), float(pc[27, nv - 1])]
    for tau in taus:
        if not 0.0 < tau < 1.0:
            continue
        O = torch.full_like(Q, 1.0)
        act, _, pooled, bact = ops.q_score(Q, kl, ka, nv, tau, True, 256, O_zero=O)
        got = act.cpu().numpy().astype(bool)
        exp = np.ones_like(got)
        exp[:, :nv] = pc > tau
        exp[0, :] = True  # preserve_first_head
        np.testing.assert_array_equal(got, exp)
        assert torch.equal(pooled, pooled_ref) or torch.allclose(pooled, pooled_ref, rtol=1e-13, atol=1e-15)
        assert torch.equal(bact.sum(dim=1), act.sum(dim=1, dtype=torch.int32))
        lazy = ~act.bool()
        assert bool((O[lazy] == 0).all()) and bool((O[~lazy] == 1).all())
