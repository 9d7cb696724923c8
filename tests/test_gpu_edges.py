"""Edge cases and error behaviour of the GPU path against the oracle:
all-lazy vision spans, no text span, tiny and ragged sequence lengths,
block sizes that do not divide N, and the reference's exceptions
(errors.py) for invalid knobs, layouts and shapes."""

import numpy as np
import pytest
import torch

from oracle import attention as oatt
from oracle import pipeline as opipe
from oracle.workload import Spec, generate, round_bf16

pytestmark = pytest.mark.gpu

ATOL, RTOL = 2e-2, 2e-2


def dev(x):
    return torch.tensor(np.asarray(x), dtype=torch.bfloat16, device="cuda")


def run_and_check(Q, K, V, nv, cfg, heads=None):
    from paper_2511_12201_b200.pipeline import sparse_prefill_device

    res = sparse_prefill_device(dev(Q), dev(K), dev(V), nv, cfg)
    torch.cuda.synchronize()
    ref = opipe.select(Q, K, nv, cfg.sink_index, cfg.tau, cfg.p, cfg.block_size, cfg.granularity,
                       cfg.preserve_first_head)
    np.testing.assert_array_equal(res.active.cpu().numpy().astype(bool), ref.active)
    assert int(res.selection.info[0]) == ref.budget and int(res.selection.info[1]) == ref.flattest
    sel = res.selection.selected.cpu().numpy()
    for g in range(len(K)):
        np.testing.assert_array_equal(sel[g, : ref.budget], ref.selected[g])
    out = res.outputs.float().cpu().numpy()
    rep = len(Q) // len(K)
    for h in heads if heads is not None else range(len(Q)):
        exp = oatt.sparse_head_attention(Q[h], K[h // rep], V[h // rep], ref.selected[h // rep], ref.active[h],
                                         cfg.sink_index)
        np.testing.assert_allclose(out[h], exp, atol=ATOL, rtol=RTOL, err_msg=f"head {h}")
    return res, ref


def test_all_vision_rows_lazy():
    """tau close to 1 without preserve_first_head: every vision query is lazy
    (zero output rows); text queries stay active and attend causally."""
    from paper_2511_12201_b200.pipeline import SparsityConfig

    Q, K, V = (round_bf16(x) for x in generate(Spec(heads=4, heads_kv=2, head_dim=128, n_vision=900, n_text=30,
                                                     seed=2)))
    res, ref = run_and_check(Q, K, V, 900, SparsityConfig(tau=0.999, preserve_first_head=False))
    assert not ref.active[:, :900].any() and ref.active[:, 900:].all()
    assert not res.outputs[:, :900].float().abs().sum().item()


def test_no_text_span_and_vision_only_prompt():
    from paper_2511_12201_b200.pipeline import SparsityConfig

    Q, K, V = (round_bf16(x) for x in generate(Spec(heads=4, heads_kv=1, head_dim=128, n_vision=777, n_text=0,
                                                     seed=9)))
    run_and_check(Q, K, V, 777, SparsityConfig())


@pytest.mark.parametrize("nv,nt,block", [(1, 1, 256), (5, 2, 4), (129, 1, 64), (257, 3, 256), (300, 41, 100)])
def test_tiny_and_ragged_lengths(nv, nt, block):
    """N of 2 .. 341 tokens: single-token probe blocks, blocks that do not
    divide N, partial 128-row tiles and a one-token vision span."""
    from paper_2511_12201_b200.pipeline import SparsityConfig

    rng = np.random.default_rng(nv + nt)
    n = nv + nt
    Q, K, V = (round_bf16(rng.normal(size=s)) for s in ((2, n, 128), (1, n, 128), (1, n, 128)))
    run_and_check(Q, K, V, nv, SparsityConfig(block_size=block))


def test_reference_exceptions():
    """Invalid knobs / layouts / shapes raise the reference's exception types."""
    from paper_2511_12201_b200 import ops
    from paper_2511_12201_b200.errors import LayoutError, ParameterError, ShapeError
    from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device

    with pytest.raises(ParameterError):
        SparsityConfig(tau=1.0)
    with pytest.raises(ParameterError):
        SparsityConfig(p=0.0)
    with pytest.raises(ParameterError):
        SparsityConfig(block_size=0)
    with pytest.raises(ParameterError):
        SparsityConfig(granularity="row")
    Q = torch.randn(4, 256, 128, device="cuda", dtype=torch.bfloat16)
    K = torch.randn(2, 256, 128, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(LayoutError):
        sparse_prefill_device(Q, K, K, 0, SparsityConfig())
    with pytest.raises(LayoutError):
        sparse_prefill_device(Q, K, K, 300, SparsityConfig())
    with pytest.raises(LayoutError):
        sparse_prefill_device(Q, K, K, 200, SparsityConfig(sink_index=256))
    with pytest.raises(ShapeError):
        sparse_prefill_device(Q[:3], K, K, 200, SparsityConfig())  # 3 Q heads over 2 KV groups
    with pytest.raises(ShapeError):
        sparse_prefill_device(Q, K[:, :200], K[:, :200], 100, SparsityConfig())
    with pytest.raises(ShapeError):
        sparse_prefill_device(Q.cpu(), K.cpu(), K.cpu(), 200, SparsityConfig())  # no CPU fallback
    with pytest.raises(ParameterError):
        kl, ka, _ = ops.kv_probe(K, 200, 0, 256)
        ops.q_score(Q, kl, ka, 200, 1.5, True, 256)
