"""The reference-named operator API running on the GPU, checked with the
reference's own known-answer examples and against the oracle —
these read like the reference's tests, but every number comes from the
CUDA kernels."""

import numpy as np
import pytest

from oracle import selection as osel
from oracle.workload import Spec, generate

pytestmark = pytest.mark.gpu


def test_spec_budget_kats():
    """a=[3,1,.5,.5]: p=.6 -> b=1; p=.82 -> b=3."""
    from paper_2511_12201_b200 import kv_select as ks

    a = np.array([3.0, 1.0, 0.5, 0.5])
    assert ks.determine_budget(a, 0.6) == 1
    assert ks.determine_budget(a, 0.82) == 3
    b, retained, total = ks.budget_with_retained_mass(a, 0.82)
    assert (b, retained, total) == (3, 4.5, 5.0)
    assert ks.determine_budget(a, 1.0) == 4


def test_spec_top_b_ties_and_flattest():
    """exactly b keys, ties to the lower index."""
    from paper_2511_12201_b200 import kv_select as ks

    a = np.array([0.1, 0.5, 0.5, 0.5, 0.2, 0.0])
    np.testing.assert_array_equal(ks.top_b_indices(a, 2), [1, 2])
    np.testing.assert_array_equal(ks.top_b_indices(a, 6), np.arange(6))
    one_hot = np.zeros(10)
    one_hot[5] = 1.0
    np.testing.assert_array_equal(ks.top_b_indices(one_hot, 1), [5])
    scores = ks.key_scores_from_vectors([np.full(64, 2.0) + np.linspace(0, 1e-3, 64), np.eye(64)[3] * 64.0])
    assert ks.flattest_head(scores) == 0
    np.testing.assert_allclose(scores.kurtoses, [osel.kurtosis(v) for v in scores.scores], rtol=1e-12)
    two_point = ks.key_scores_from_vectors([np.array([-1.0, 1.0]), np.array([-1.0, 1.0])])
    assert two_point.kurtoses[0] == pytest.approx(1.0, abs=1e-15)
    assert ks.flattest_head(two_point) == 0  # tie -> lowest index


def test_spec_probe_keys_and_classification():
    """SPEC.md:173-176, 182-185."""
    from paper_2511_12201_b200.attention import TokenLayout
    from paper_2511_12201_b200.query_select import ProbeKeys, build_probe_keys, classify_queries

    k = np.zeros((3, 32))
    k[0, 0] = 1.0
    k[1, 1] = 1.0
    pk = build_probe_keys(k, TokenLayout(2, 1))
    np.testing.assert_allclose(pk.active_key[:2], [0.5, 0.5])
    np.testing.assert_allclose(pk.lazy_key, k[0])
    probes = ProbeKeys(np.eye(32)[0], np.eye(32)[1])
    q = np.zeros((2, 32))
    q[0, :2] = 1.0        # equal logits -> p = 0.5 -> active at tau = 0.08
    q[1, 0] = 50.0        # aligned with the lazy key -> p -> 0 -> lazy
    p, act = classify_queries(q, probes, 0.08)
    assert p[0] == pytest.approx(0.5, abs=1e-15) and act[0]
    assert p[1] < 1e-3 and not act[1]
    with pytest.raises(ValueError):
        classify_queries(q, probes, 1.0)


def test_query_masks_and_probe_match_oracle():
    from paper_2511_12201_b200.attention import AttentionWorkload, TokenLayout
    from paper_2511_12201_b200.block_probe import block_scores_to_token_scores, probe_attention
    from paper_2511_12201_b200.query_select import build_query_masks

    Q, K, V = generate(Spec(heads=4, head_dim=32, n_vision=500, n_text=12, seed=9))
    Q, K = Q.astype(np.float32).astype(np.float64), K.astype(np.float32).astype(np.float64)
    w = AttentionWorkload(list(Q), list(K), list(V), TokenLayout(500, 12))
    masks = build_query_masks(w, 0.08)
    for h in range(4):
        kl, ka = osel.probe_keys(K[h], 500, 0)
        np.testing.assert_array_equal(masks[h].active, osel.query_mask(Q[h], kl, ka, 500, 0.08, h == 0))
    pm = probe_attention(Q[1], K[1], 64)
    ref = osel.probe_map(Q[1], K[1], 64)
    np.testing.assert_allclose(pm.attention, ref, rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(block_scores_to_token_scores(pm, 512),
                               osel.token_scores_from_blocks(osel.block_mass(ref), 512, 64), rtol=1e-10)
    one = probe_attention(Q[1], K[1], 512)  # B = N -> [[1]]
    np.testing.assert_allclose(one.attention, [[1.0]])


def test_sparse_prefill_and_head_attention_api():
    from oracle import attention as oatt
    from oracle import pipeline as opipe
    from paper_2511_12201_b200.attention import AttentionWorkload, TokenLayout
    from paper_2511_12201_b200.prefill import SparsityConfig, sparse_head_attention, sparse_prefill

    Q, K, V = generate(Spec(heads=4, heads_kv=2, head_dim=128, n_vision=1500, n_text=36, seed=4))
    w = AttentionWorkload(list(Q), list(K), list(V), TokenLayout(1500, 36))
    out = sparse_prefill(w, SparsityConfig(), "probe")
    from oracle.workload import round_bf16
    Qb, Kb, Vb = round_bf16(Q), round_bf16(K), round_bf16(V)
    ref = opipe.select(Qb, Kb, 1500, 0, 0.08, 0.82, 256)
    assert out.selection.budget == ref.budget and out.selection.flattest_head == ref.flattest
    for g in range(2):
        np.testing.assert_array_equal(out.selection.selected[g], ref.selected[g])
    for h in range(4):
        np.testing.assert_array_equal(out.query_masks[h], ref.active[h])
        exp = oatt.sparse_head_attention(Qb[h], Kb[h // 2], Vb[h // 2], ref.selected[h // 2], ref.active[h], 0)
        np.testing.assert_allclose(out.outputs[h], exp, atol=2e-2, rtol=2e-2)
    single = sparse_head_attention(Qb[1], Kb[0], Vb[0], ref.selected[0], ref.active[1], 0)
    np.testing.assert_allclose(single, oatt.sparse_head_attention(Qb[1], Kb[0], Vb[0], ref.selected[0],
                                                                  ref.active[1], 0), atol=2e-2, rtol=2e-2)
    empty = sparse_head_attention(Qb[1], Kb[0], Vb[0], np.array([], dtype=np.int64), ref.active[1], 0)
    assert not empty.any()  # prefill.py:107-108


def test_prefill_output_key_scores_and_recall():
    """PrefillOutput.key_scores (kv_select.py:23-36, rule B: per KV group) and
    recall_per_head (metrics.py:26-39) vs the oracle on the same inputs."""
    from oracle import metrics as om
    from oracle import pipeline as opipe
    from oracle.workload import round_bf16
    from paper_2511_12201_b200.attention import AttentionWorkload, TokenLayout
    from paper_2511_12201_b200.prefill import SparsityConfig, sparse_prefill

    Q, K, V = generate(Spec(heads=4, heads_kv=2, head_dim=128, n_vision=1500, n_text=36, seed=8))
    Qb, Kb, Vb = round_bf16(Q), round_bf16(K), round_bf16(V)
    w = AttentionWorkload(list(Qb), list(Kb), list(Vb), TokenLayout(1500, 36))
    out = sparse_prefill(w, SparsityConfig(), "probe", with_recall=True)
    ref = opipe.select(Qb, Kb, 1500, 0, 0.08, 0.82, 256)
    assert out.key_scores.num_heads == 2 and out.key_scores.num_keys == 1536
    for g in range(2):
        np.testing.assert_allclose(out.key_scores.scores[g], ref.group_scores[g], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(out.key_scores.kurtoses, ref.kurtoses, rtol=1e-10)
    for h in range(4):
        exp = om.head_recall(Qb[h], Kb[h // 2], ref.selected[h // 2], ref.active[h])
        assert abs(out.recall_per_head[h] - exp) < 2e-3


def test_select_top_blocks_sparsity_gap_and_decode_classification():
    """kv_select.select_top_blocks / sparsity_gap (kv_select.py:147-210) and
    decode.classify_decode_query (decode.py:124-140) vs the oracle."""
    import torch

    from paper_2511_12201_b200 import decode as gdec
    from paper_2511_12201_b200 import kv_select as ks

    rng = np.random.default_rng(3)
    vecs = [rng.gamma(0.5 + i, size=1000) for i in range(3)]
    scores = ks.key_scores_from_vectors(vecs)
    for b, blk in ((1, 64), (300, 64), (257, 100), (1000, 128)):
        got = ks.select_top_blocks(scores, b, blk)
        exp = osel.top_blocks(vecs, b, blk)
        for g in range(3):
            np.testing.assert_array_equal(got.selected[g], exp[g])
    for p in (0.2, 0.82):
        assert ks.sparsity_gap(scores, p) == osel.sparsity_gap(vecs, p)
    # decode classification: flags of decode_attention and the standalone call agree with the oracle rule
    hq, hkv, d = 8, 2, 128
    q = torch.randn(3, hq, d, device="cuda").to(torch.bfloat16)
    k_lazy = torch.randn(3, hkv, d, device="cuda", dtype=torch.float64)
    k_act = torch.randn(3, hkv, d, device="cuda", dtype=torch.float64)
    K = torch.randn(hkv, 200, d, device="cuda").to(torch.bfloat16)
    sel = torch.arange(64, device="cuda", dtype=torch.int32).repeat(hkv, 1)
    caches = [gdec.build_cache_device(K, K, sel, 64, 184, 16, k_lazy[s], k_act[s], hq) for s in range(3)]
    cache = gdec.stack_caches(caches)
    fl = gdec.classify_decode_batch(q, cache, 0.3).cpu().numpy().astype(bool)
    _, fl2 = gdec.decode_attention_batch(q, cache, 0.3, log=False)
    np.testing.assert_array_equal(fl, fl2.cpu().numpy().astype(bool))
    for s in range(3):
        for h in range(hq):
            g = h // (hq // hkv)
            _, verdict = osel.classify(q[s, h].double().cpu().numpy()[None], k_lazy[s, g].cpu().numpy(),
                                       k_act[s, g].cpu().numpy(), 0.3)
            assert fl[s, h] == (bool(verdict[0]) or h == 0)
