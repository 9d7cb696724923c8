"""GPU parity of cache slimming (K6) and slimmed decode (K7) vs the oracle.

Flags are bit-exact (float64 classification on both sides); outputs within
atol 5e-3 / rtol 2e-2: cache values are the same bf16 numbers on both sides,
the kernel accumulates in fp32 with P rounded to bf16 for the PV tensor-core
product (the same class of rounding as the prefill kernel)."""

import numpy as np
import pytest
import torch

from oracle import attention as oatt
from oracle import pipeline as opipe
from oracle.workload import Spec, decode_inputs, generate, round_bf16

pytestmark = pytest.mark.gpu


def dev(x, dtype=torch.bfloat16):
    return torch.tensor(np.asarray(x), dtype=dtype, device="cuda")


def build_pair(seed, hq=8, hkv=2, nv=2000, nt=48, steps=6, tau=0.08, lazy=0.5, answer_capacity=16):
    from paper_2511_12201_b200 import decode as gdec
    from paper_2511_12201_b200 import ops
    from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device

    spec = Spec(heads=hq, heads_kv=hkv, head_dim=128, n_vision=nv, n_text=nt, seed=seed, lazy_fraction=lazy)
    Q, K, V = (round_bf16(x) for x in generate(spec))
    n = nv + nt
    res = sparse_prefill_device(dev(Q), dev(K), dev(V), nv, SparsityConfig(tau=tau))
    b = int(res.selection.info[0])
    vsel = ops.select(res.block_mass, hkv, n, 256, 0.82, "token", vision_limit=nv, budget_override=b)
    bv = int(vsel.info[0])
    cache = gdec.build_cache_device(dev(K), dev(V), vsel.selected, bv, nv, nt, res.k_lazy, res.k_act, hq,
                             answer_capacity=answer_capacity)
    ref = opipe.select(Q, K, nv, 0, tau, 0.82, 256)
    rb, rsel = opipe.vision_selection(ref, nv)
    assert rb == bv
    for g in range(hkv):
        np.testing.assert_array_equal(vsel.selected[g, :bv].cpu().numpy(), rsel[g])
    ocache = oatt.build_cache(K, V, rsel, rb, nv, nt, 0)
    trace = decode_inputs(spec, K, steps, np.random.default_rng(100 + seed))
    trace = [(round_bf16(q), round_bf16(k), round_bf16(v)) for q, k, v in trace]
    return cache, ocache, trace, hq // hkv


def test_build_cache_gathers_selected_rows():
    cache, ocache, _, _ = build_pair(0)
    b = cache.budgets[0]
    for g in range(cache.n_kv_heads):
        np.testing.assert_array_equal(cache.rows(0, g, "vision", "k").float().cpu().numpy(), ocache[g].vision_k)
        np.testing.assert_array_equal(cache.rows(0, g, "vision", "v").float().cpu().numpy(), ocache[g].vision_v)
        np.testing.assert_array_equal(cache.rows(0, g, "text", "v").float().cpu().numpy(), ocache[g].text_v)
        np.testing.assert_array_equal(cache.vision_indices[0][g].cpu().numpy(), ocache[g].vision_indices)
        np.testing.assert_allclose(cache.k_act[0, g].cpu().numpy(), ocache[g].k_act, rtol=1e-13)
        np.testing.assert_array_equal(cache.k_lazy[0, g].cpu().numpy(), ocache[g].k_lazy)


def test_decode_trace_matches_oracle():
    from paper_2511_12201_b200 import decode as gdec

    cache, ocache, trace, rep = build_pair(1)
    log = oatt.FetchLog()
    for q, k, v in trace:
        out, flags = gdec.decode_attention_batch(dev(q).unsqueeze(0), cache, 0.08)
        o_ref, f_ref = oatt.decode_step(q, ocache, 0.08, rep, True, log)
        np.testing.assert_array_equal(flags[0].cpu().numpy().astype(bool), f_ref)
        np.testing.assert_allclose(out[0].cpu().numpy(), np.stack(o_ref), atol=5e-3, rtol=2e-2)
        gdec.append_answer_batch(cache, dev(k).unsqueeze(0), dev(v).unsqueeze(0))
        oatt.append_answer(ocache, k, v, 128)
    assert cache.fetch.vision_tokens == log.vision_tokens
    assert cache.fetch.step_active_heads == log.step_active_heads


def test_forced_flags_exclusion_semantics():
    from paper_2511_12201_b200 import decode as gdec

    cache, ocache, trace, rep = build_pair(2)
    q = trace[0][0]
    forced = np.zeros(cache.n_q_heads, dtype=bool)
    forced[[0, 3, 5]] = True
    out, fl = gdec.decode_attention_batch(dev(q).unsqueeze(0), cache, 0.08, flags=torch.tensor(forced[None]))
    np.testing.assert_array_equal(fl[0].cpu().numpy().astype(bool), forced)
    exp = np.stack(oatt.decode_dense(q, ocache, forced, rep))
    np.testing.assert_allclose(out[0].cpu().numpy(), exp, atol=5e-3, rtol=2e-2)


def test_batched_decode_ragged_budgets():
    """Batch of sequences with different budgets and lazy patterns (C5 shape
    logic at small N): every sequence matches its own oracle."""
    from paper_2511_12201_b200 import decode as gdec

    pairs = [build_pair(s, lazy=0.3 + 0.2 * s) for s in range(3)]
    assert len({p[0].pool.k.data_ptr() for p in pairs}) == 1  # one page pool for the device
    batch = gdec.stack_caches([p[0] for p in pairs])
    logs = [oatt.FetchLog() for _ in pairs]
    for step in range(4):
        q = np.stack([p[2][step][0] for p in pairs])
        out, flags = gdec.decode_attention_batch(dev(q), batch, 0.08)
        for s, (c, oc, tr, rep) in enumerate(pairs):
            o_ref, f_ref = oatt.decode_step(tr[step][0], oc, 0.08, rep, True, logs[s])
            np.testing.assert_array_equal(flags[s].cpu().numpy().astype(bool), f_ref)
            np.testing.assert_allclose(out[s].cpu().numpy(), np.stack(o_ref), atol=5e-3, rtol=2e-2)
            oatt.append_answer(oc, tr[step][1], tr[step][2], 128)
        ks = dev(np.stack([p[2][step][1] for p in pairs]))
        vs = dev(np.stack([p[2][step][2] for p in pairs]))
        gdec.append_answer_batch(batch, ks, vs)
    assert batch.fetch.vision_tokens == sum(l.vision_tokens for l in logs)


def test_serving_lifecycle_ragged_admit_evict_grow():
    """Serving batch: sequences with different vision spans, budgets, prompt
    text and answer lengths (ragged K7), answer capacity growth, eviction of a
    finished sequence and admission of a new one mid-stream; every live
    sequence matches its own oracle at every step."""
    from paper_2511_12201_b200 import decode as gdec

    specs = [dict(seed=0, nv=2000, nt=48), dict(seed=1, nv=1500, nt=20), dict(seed=2, nv=2300, nt=64)]
    live = [build_pair(steps=8, answer_capacity=2, **sp) for sp in specs]
    batch = gdec.stack_caches([p[0] for p in live])
    assert batch.ragged and batch.text_lens == [48, 20, 64]
    logs = [oatt.FetchLog() for _ in live]
    t = [0] * len(live)

    def step():
        q = np.stack([p[2][t[s]][0] for s, p in enumerate(live)])
        out, flags = gdec.decode_attention_batch(dev(q), batch, 0.08)
        for s, (c, oc, tr, rep) in enumerate(live):
            o_ref, f_ref = oatt.decode_step(tr[t[s]][0], oc, 0.08, rep, True, logs[s])
            np.testing.assert_array_equal(flags[s].cpu().numpy().astype(bool), f_ref)
            np.testing.assert_allclose(out[s].cpu().numpy(), np.stack(o_ref), atol=5e-3, rtol=2e-2)
            oatt.append_answer(oc, tr[t[s]][1], tr[t[s]][2], 128)
        ks = dev(np.stack([p[2][t[s]][1] for s, p in enumerate(live)]))
        vs = dev(np.stack([p[2][t[s]][2] for s, p in enumerate(live)]))
        gdec.append_answer_batch(batch, ks, vs)
        for s in range(len(live)):
            t[s] += 1

    for _ in range(3):
        step()
    assert batch.answer_lens == [3, 3, 3] and all(batch.answer_capacity(s) >= 3 for s in range(3))
    vt = batch.fetch.vision_tokens
    assert vt == sum(l.vision_tokens for l in logs)
    # sequence 1 finishes; its pages go back to the pool; a new one
    # (different spans) joins with no answer yet, writing only its own pages
    pool = batch.pool
    used = pool.used
    freed = batch.pages[1].size
    batch = gdec.evict(batch, [0, 2])
    assert pool.used == used - freed
    live, logs, t = [live[0], live[2]], [logs[0], logs[2]], [t[0], t[2]]
    new = build_pair(steps=8, seed=3, nv=1800, nt=33)
    ptr = pool.k.data_ptr()
    batch = gdec.admit(batch, new[0])
    assert pool.k.data_ptr() == ptr  # admission moved no KV
    live.append(new)
    logs.append(oatt.FetchLog())
    t.append(0)
    assert batch.answer_lens == [3, 3, 0] and batch.text_lens == [48, 64, 33]
    for _ in range(3):
        step()
    assert batch.answer_lens == [6, 6, 3]
    # answer growth takes one page per group every 64 tokens; grow=False refuses
    from paper_2511_12201_b200.errors import ShapeError

    u = build_pair(4, answer_capacity=1)[0]
    z = torch.zeros(1, 2, 128, device="cuda")
    for _ in range(3):
        gdec.append_answer_batch(u, z, z)
    assert not u.ragged and u.n_answer == 3 and u.answer_capacity(0) == 64
    while u.n_answer < u.answer_capacity(0):
        gdec.append_answer_batch(u, z, z)
    with pytest.raises(ShapeError):
        gdec.append_answer_batch(u, z, z, grow=False)
    pages = u.pages[0].shape[1]
    gdec.append_answer_batch(u, z, z)
    assert u.pages[0].shape[1] == pages + 1 and u.answer_capacity(0) == 128


def test_ragged_degenerate_context_flag():
    """A ragged batch member with no text and no answer rows and a lazy head
    raises DegenerateContextError (decode.py:152-153) via the device status."""
    from paper_2511_12201_b200 import decode as gdec
    from paper_2511_12201_b200.errors import DegenerateContextError

    a = build_pair(0)[0]
    b, _, trace, _ = build_pair(1, nt=0, lazy=0.9)
    batch = gdec.stack_caches([a, b])
    assert batch.ragged and batch.text_lens == [48, 0]
    q = np.stack([trace[0][0], trace[0][0]])
    forced = np.ones((2, 8), dtype=bool)
    forced[1, 3] = False  # a lazy head of the context-less sequence
    with pytest.raises(DegenerateContextError):
        gdec.decode_attention_batch(dev(q), batch, 0.08, flags=torch.tensor(forced))


def test_reference_signature_decode_replays_reference_trace(golden):
    """The reference's own decode trace (tests/golden/decode_trace.npz, made by
    slimattn: select_vision_keys -> build_cache(w, sel) -> 8 x
    decode_attention + append_answer, head_dim 32) replayed through the
    reference-signature operators on the GPU: flags bit-exact (float64
    classification of the unrounded queries), outputs within the bf16
    tolerance (the cache stores bf16 rows; the fixture is float64), FetchLog
    totals and per-step entries EQUAL under the reference's 8-byte model,
    forced flags (decode.py:170-173) with exclusion semantics."""
    from oracle.workload import Spec, decode_inputs, generate
    from paper_2511_12201_b200 import decode as gdec
    from paper_2511_12201_b200.attention import AttentionWorkload, TokenLayout
    from paper_2511_12201_b200.kv_select import SelectionResult

    g = golden("decode_trace.npz")
    spec = Spec(heads=4, head_dim=32, n_vision=256, n_text=16, seed=5)
    Q, K, V = generate(spec)
    w = AttentionWorkload(list(Q), list(K), list(V), TokenLayout(256, 16))
    b = int(g["budget"])
    sel = SelectionResult(b, [np.asarray(s, dtype=np.int64) for s in g["vision_selected"]], 0)
    cache = gdec.build_cache(w, sel, True)
    assert cache.budget == b and cache.num_heads == 4 and cache.head_dim == 32 and cache.n_answer == 0
    steps = decode_inputs(spec, K, 8, np.random.default_rng(123))
    np.testing.assert_array_equal(np.stack([s[0] for s in steps]), g["queries"])
    for i, (q, k, v) in enumerate(steps):
        fl = gdec.classify_decode_query(list(q), cache, 0.08)
        np.testing.assert_array_equal(fl, g["flags"][i])
        out, flags = gdec.decode_attention(list(q), cache, 0.08)
        np.testing.assert_array_equal(flags, g["flags"][i])
        assert isinstance(out, list) and len(out) == 4 and out[0].shape == (32,)
        np.testing.assert_allclose(np.stack(out), g["outputs"][i], atol=2e-2, rtol=2e-2)
        gdec.append_answer(cache, list(k), list(v))
    log = cache.fetch
    assert log.vision_tokens == int(g["vision_tokens"])
    assert log.vision_bytes == int(g["vision_bytes"])
    assert log.text_answer_bytes == int(g["text_answer_bytes"])
    np.testing.assert_array_equal(log.step_vision_tokens, g["step_vision_tokens"])
    np.testing.assert_array_equal(log.step_active_heads, g["step_active_heads"])
    assert cache.n_answer == 8 and log.steps == 8
    forced = np.array([True, False, True, False])
    out, fl = gdec.decode_attention(steps[0][0], cache, 0.08, flags=forced)
    np.testing.assert_array_equal(fl, forced)
    np.testing.assert_allclose(np.stack(out), g["forced_outputs"], atol=2e-2, rtol=2e-2)
    # exclusion (forced_outputs) vs literal zeroing (forced_zeroed) differ for the lazy heads
    assert np.abs(np.stack(out)[1] - g["forced_zeroed"][1]).max() > 1e-3


def test_reference_signature_errors():
    from oracle.workload import Spec, generate
    from paper_2511_12201_b200 import decode as gdec
    from paper_2511_12201_b200.attention import AttentionWorkload, TokenLayout
    from paper_2511_12201_b200.errors import DegenerateContextError, IntegrityError, ShapeError
    from paper_2511_12201_b200.kv_select import SelectionResult

    Q, K, V = generate(Spec(heads=2, head_dim=32, n_vision=64, n_text=0, seed=1))
    w = AttentionWorkload(list(Q), list(K), list(V), TokenLayout(64, 0))
    with pytest.raises(IntegrityError):
        gdec.build_cache(w, SelectionResult(4, [np.arange(3), np.arange(4)], 0))
    with pytest.raises(IntegrityError):
        gdec.build_cache(w, SelectionResult(2, [np.array([0, 64]), np.arange(2)], 0))
    cache = gdec.build_cache(w, SelectionResult(4, [np.arange(4), np.arange(4)], 0))
    with pytest.raises(ShapeError):
        gdec.append_answer(cache, [np.zeros(32)], [np.zeros(32)])
    with pytest.raises(ShapeError):
        gdec.append_answer(cache, [np.zeros(31)] * 2, [np.zeros(31)] * 2)
    with pytest.raises(DegenerateContextError):  # no text, no answer, a lazy head
        gdec.decode_attention(Q[:, 0], cache, 0.08, flags=np.array([True, False]))
    out, fl = gdec.decode_attention(Q[:, 0], cache, 0.08, flags=np.array([True, True]))
    assert len(out) == 2
