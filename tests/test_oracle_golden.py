"""Pin the NumPy oracle to outputs of the reference itself (tests/golden/*.npz,
produced by tests/golden/make_golden.py from /root/reference)."""

import hashlib

import numpy as np
import pytest

from oracle import attention as oatt
from oracle import pipeline, selection
from oracle.workload import Spec, decode_inputs, generate


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_c1_matches_reference(golden, seed):
    g = golden(f"c1_seed{seed}.npz")
    Q, K, V = generate(Spec(heads=4, head_dim=128, n_vision=1984, n_text=64, seed=seed))
    assert digest(*Q, *K, *V) == str(g["raw_digest"]), "generator restatement drifted from workload.py"
    Q, K, V = (x.astype(np.float32).astype(np.float64) for x in (Q, K, V))
    res = pipeline.prefill(Q, K, V, 1984, 0, 0.08, 0.82, 256)
    act = np.unpackbits(g["active"], axis=1)[:, : int(g["n"])].astype(bool)
    np.testing.assert_array_equal(res.active, act)
    np.testing.assert_allclose(res.p_act, g["p_act"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(res.block_mass, g["block_mass"], rtol=1e-12)
    np.testing.assert_allclose(res.kurtoses, g["kurtoses"], rtol=1e-12)
    assert res.flattest == int(g["flattest"])
    assert res.budget == int(g["budget"])
    assert res.retained == pytest.approx(float(g["retained"]), rel=1e-12)
    np.testing.assert_array_equal(np.stack(res.selected), g["selected"])
    np.testing.assert_allclose(res.outputs.sum(axis=(1, 2)), g["out_sum"], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose((res.outputs ** 2).sum(axis=(1, 2)), g["out_sq"], rtol=1e-11)
    np.testing.assert_allclose(res.outputs[:, g["rows"], :], g["out_rows"], rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("tag,source,gran,block", [
    ("exact_token", "exact", "token", 16), ("exact_block", "exact", "block", 16),
    ("probe_token", "probe", "token", 16), ("probe_b1", "probe", "token", 1)])
def test_tiny_paths_match_reference(golden, tag, source, gran, block):
    g = golden("tiny_paths.npz")
    Q, K, V = generate(Spec(heads=4, head_dim=32, n_vision=120, n_text=8, seed=11))
    assert digest(*Q, *K, *V) == str(g["digest"])
    res = pipeline.prefill(Q, K, V, 120, 0, 0.08, 0.82, block, gran, True, source)
    np.testing.assert_array_equal(res.active, g[f"{tag}_active"])
    assert res.budget == int(g[f"{tag}_budget"])
    assert res.flattest == int(g[f"{tag}_flattest"])
    np.testing.assert_allclose(res.kurtoses, g[f"{tag}_kurtoses"], rtol=1e-12)
    np.testing.assert_allclose(np.stack(res.group_scores), g[f"{tag}_scores"], rtol=1e-12, atol=1e-14)
    np.testing.assert_array_equal(np.stack(res.selected), g[f"{tag}_selected"])
    np.testing.assert_allclose(res.outputs, g[f"{tag}_outputs"], rtol=1e-11, atol=1e-12)
    assert res.retained == pytest.approx(float(g[f"{tag}_retained"]), rel=1e-12)


def test_ac8_probe_b1_equals_exact(golden):
    """SPEC.md:597 AC8 — B=1 probe selection == exact selection (fixture and oracle)."""
    g = golden("tiny_paths.npz")
    np.testing.assert_array_equal(g["probe_b1_selected"], g["exact_token_selected"])
    Q, K, V = generate(Spec(heads=4, head_dim=32, n_vision=120, n_text=8, seed=11))
    a = pipeline.select(Q, K, 120, 0, 0.08, 0.82, 1, score_source="probe")
    b = pipeline.select(Q, K, 120, 0, 0.08, 0.82, 1, score_source="exact")
    for x, y in zip(a.selected, b.selected):
        np.testing.assert_array_equal(x, y)


def test_ac1_sparsity_disabled_equals_dense(golden):
    """SPEC.md:590 AC1 — tau=0, p=1 sparse prefill == dense oracle."""
    g = golden("tiny_paths.npz")
    Q, K, V = generate(Spec(heads=4, head_dim=32, n_vision=120, n_text=8, seed=11))
    res = pipeline.prefill(Q, K, V, 120, 0, 0.0, 1.0, 16, "token", True, "exact")
    np.testing.assert_allclose(res.outputs, g["ac1_outputs"], rtol=1e-11, atol=1e-12)
    dense = np.stack([oatt.causal_attention(Q[h], K[h], V[h])[1] for h in range(4)])
    np.testing.assert_allclose(dense, g["dense_outputs"], rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(res.outputs, dense, rtol=1e-6, atol=1e-9)


def test_decode_trace_matches_reference(golden):
    g = golden("decode_trace.npz")
    spec = Spec(heads=4, head_dim=32, n_vision=256, n_text=16, seed=5)
    Q, K, V = generate(spec)
    res = pipeline.select(Q, K, 256, 0, 0.08, 0.82, 16)
    b, vsel = pipeline.vision_selection(res, 256)
    assert b == int(g["budget"])
    np.testing.assert_array_equal(np.stack(vsel), g["vision_selected"])
    cache = oatt.build_cache(K, V, vsel, b, 256, 16, 0)
    log = oatt.FetchLog()
    steps = decode_inputs(spec, K, 8, np.random.default_rng(123))
    np.testing.assert_array_equal(np.stack([s[0] for s in steps]), g["queries"])
    for i, (q, k, v) in enumerate(steps):
        o, f = oatt.decode_step(q, cache, 0.08, 1, True, log)
        np.testing.assert_array_equal(f, g["flags"][i])
        np.testing.assert_allclose(np.stack(o), g["outputs"][i], rtol=1e-11, atol=1e-12)
        oatt.append_answer(cache, k, v, 32)
    assert log.vision_tokens == int(g["vision_tokens"])
    assert log.vision_bytes == int(g["vision_bytes"])
    assert log.text_answer_bytes == int(g["text_answer_bytes"])
    np.testing.assert_array_equal(log.step_active_heads, g["step_active_heads"])
    forced = np.array([True, False, True, False])
    o, _ = oatt.decode_step(steps[0][0], cache, 0.08, 1, True, oatt.FetchLog(), flags=forced)
    np.testing.assert_allclose(np.stack(o), g["forced_outputs"], rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(np.stack(oatt.decode_dense(steps[0][0], cache, forced, 1)), g["forced_dense"], rtol=1e-10)
    z = np.stack(oatt.decode_dense(steps[0][0], cache, forced, 1, zero_masked_vision=True))
    np.testing.assert_allclose(z, g["forced_zeroed"], rtol=1e-10)
    assert np.abs(z[1] - np.stack(o)[1]).max() > 1e-6  # SPEC.md:462 exclusion != literal zeroing


@pytest.mark.parametrize("seed", [0, 1])
def test_gqa_rule_b_matches_reference_composition(golden, seed):
    g = golden(f"gqa_seed{seed}.npz")
    Q, K, V = generate(Spec(heads=8, heads_kv=2, head_dim=64, n_vision=4032, n_text=64, seed=seed))
    assert digest(Q, K, V) == str(g["digest"])
    res = pipeline.prefill(Q, K, V, 4032, 0, 0.08, 0.82, 256)
    act = np.unpackbits(g["active"], axis=1)[:, : int(g["n"])].astype(bool)
    np.testing.assert_array_equal(res.active, act)
    np.testing.assert_allclose(res.p_act, g["p_act"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(res.block_mass, g["block_mass"], rtol=1e-12)
    np.testing.assert_allclose(res.kurtoses, g["kurtoses"], rtol=1e-12)
    assert res.flattest == int(g["flattest"]) and res.budget == int(g["budget"])
    np.testing.assert_array_equal(np.stack(res.selected), g["selected"])
    vb, vs = pipeline.vision_selection(res, 4032)
    assert vb == int(g["vision_budget"])
    np.testing.assert_array_equal(np.stack(vs), g["vision_selected"])
    np.testing.assert_allclose(res.outputs[:, g["rows"], :], g["out_rows"], rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(res.outputs.sum(axis=(1, 2)), g["out_sum"], rtol=1e-9, atol=1e-9)


def test_grad_oracle_forward_pinned_to_sparse_head_attention():
    from oracle.grad import sparse_attention_grads
    Q, K, V = generate(Spec(heads=4, heads_kv=2, head_dim=16, n_vision=60, n_text=4, seed=3))
    res = pipeline.select(Q, K, 60, 0, 0.08, 0.82, 8)
    dO = np.random.default_rng(0).normal(size=Q.shape)
    out, dq, dk, dv = sparse_attention_grads(Q, K, V, res.selected, res.active, 0, dO)
    for h in range(4):
        ref = oatt.sparse_head_attention(Q[h], K[h // 2], V[h // 2], res.selected[h // 2], res.active[h], 0)
        np.testing.assert_allclose(out[h], ref, rtol=1e-12, atol=1e-13)
    assert np.all(dq[~res.active] == 0.0)


def _pairwise(a, lo, n):
    """NumPy's pairwise summation (loops_utils.h.src pairwise_sum) restated
    in pure Python: the order csrc/select.cu emulates for kurtosis."""
    if n < 8:
        r = 0.0
        for i in range(n):
            r = r + a[lo + i]
        return r
    if n <= 128:
        r = [a[lo + j] for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] = r[j] + a[lo + i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res = res + a[lo + i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return _pairwise(a, lo, n2) + _pairwise(a, lo + n2, n - n2)


def test_numpy_summation_orders_the_gpu_emulates():
    """Pins the arithmetic order K3b reproduces: np.sum is the pairwise sum
    above for every length, np.add.reduceat sums a segment as its first
    element plus the pairwise sum of the rest, and the oracle's kurtosis
    (_core_py.kurtosis) is three pairwise means. Values spread over many
    binades so that any other order rounds differently."""
    from oracle.numerics import kurtosis

    rng = np.random.default_rng(0)
    for n in list(range(1, 260)) + [1000, 1023, 4097, 8193, 65536, 65553, 131072]:
        a = rng.standard_normal(n) * np.exp(rng.standard_normal(n) * 8)
        lst = a.tolist()
        assert np.sum(a) == _pairwise(lst, 0, n), n
        if n >= 20:
            starts = np.arange(0, n, 13)
            r = np.add.reduceat(a, starts)
            for k in (0, len(starts) // 2, len(starts) - 1):
                s0 = int(starts[k])
                m = min(13, n - s0)
                want = lst[s0] + _pairwise(lst, s0 + 1, m - 1) if m > 1 else lst[s0]
                assert r[k] == want
        if n in (1000, 4097, 65553):
            v = np.abs(a)
            mu = _pairwise(v.tolist(), 0, n) / n
            d = [x - mu for x in v.tolist()]
            m2 = _pairwise([x * x for x in d], 0, n) / n
            m4 = _pairwise([((x * x) * x) * x for x in d], 0, n) / n
            assert kurtosis(v) == m4 / (m2 * m2)
