"""Model-side drop-in: head concatenation + output
projection (attention.py:111-134) and the Qwen2-style OmniSparse attention
layer (projections, RoPE, packed sequences, forward + backward).

Tolerances: bf16 activations / weights, fp32 accumulation; the dense layer is
compared with an fp32 torch reference of the same layer at atol 3e-2 / rtol
3e-2 on outputs and a relative 3e-2 Frobenius error on gradients."""

import numpy as np
import pytest
import torch

from oracle import attention as oatt
from oracle.workload import Spec, generate, round_bf16

pytestmark = pytest.mark.gpu


def test_full_multihead_concat_and_output_projection():
    from paper_2511_12201_b200.attention import AttentionWorkload, TokenLayout, full_multihead

    Q, K, V = generate(Spec(heads=4, heads_kv=2, head_dim=128, n_vision=900, n_text=60, seed=4))
    Q, K, V = round_bf16(Q), round_bf16(K), round_bf16(V)
    W = np.random.default_rng(0).standard_normal((4 * 128, 96)) / 16
    w = AttentionWorkload(list(Q), list(K), list(V), TokenLayout(900, 60))
    res = full_multihead(w, output_proj=W, keep_attention=True)
    heads = []
    for h in range(4):
        a, o = oatt.causal_attention(Q[h], K[h // 2], V[h // 2])
        heads.append(o)
        np.testing.assert_allclose(res.attention[h].cpu().numpy(), a, atol=2e-5)
    exp = np.hstack(heads) @ W
    np.testing.assert_allclose(res.concatenated.cpu().numpy(), exp, atol=3e-2, rtol=3e-2)
    nc = full_multihead(w, causal=False)
    s = np.einsum("nd,md->nm", Q[1], K[0]) / np.sqrt(128)
    p = np.exp(s - s.max(axis=1, keepdims=True))
    exp_nc = (p / p.sum(axis=1, keepdims=True)) @ V[0]
    np.testing.assert_allclose(nc.head_outputs[1].float().cpu().numpy(), exp_nc, atol=2e-2, rtol=2e-2)


def _layer(cfg, hidden=512, hq=8, hkv=2, seed=0):
    from paper_2511_12201_b200.layer import OmniSparseAttention

    torch.manual_seed(seed)
    layer = OmniSparseAttention(hidden, hq, hkv, cfg=cfg, device="cuda")
    with torch.no_grad():
        for lin in (layer.q_proj, layer.k_proj, layer.v_proj, layer.o_proj):
            lin.weight.normal_(0, hidden ** -0.5)
    return layer


def _torch_reference(P, hq, hkv, theta, x):
    """fp32 dense causal layer from the parameter dict P (no sparsity)."""
    from paper_2511_12201_b200.layer import apply_rope, rope_cos_sin

    lin = torch.nn.functional.linear
    n = x.shape[0]
    q = lin(x, P["q_proj.weight"], P["q_proj.bias"]).view(n, hq, 128).transpose(0, 1)
    k = lin(x, P["k_proj.weight"], P["k_proj.bias"]).view(n, hkv, 128).transpose(0, 1)
    v = lin(x, P["v_proj.weight"], P["v_proj.bias"]).view(n, hkv, 128).transpose(0, 1)
    cos, sin = rope_cos_sin(n, 128, theta, x.device)
    q, k = apply_rope(q, cos, sin), apply_rope(k, cos, sin)
    rep = hq // hkv
    o = torch.nn.functional.scaled_dot_product_attention(q[None], k.repeat_interleave(rep, 0)[None],
                                                         v.repeat_interleave(rep, 0)[None], is_causal=True)[0]
    return lin(o.transpose(0, 1).reshape(n, -1), P["o_proj.weight"])


def test_layer_dense_mode_forward_backward_vs_torch():
    """tau = 0, p = 1: the layer is exact causal attention; outputs and the
    gradients of the input and every projection match an fp32 reference."""
    from paper_2511_12201_b200.pipeline import SparsityConfig

    layer = _layer(SparsityConfig(tau=0.0, p=1.0))
    torch.manual_seed(1)
    xb = torch.randn(1500, 512, device="cuda").to(torch.bfloat16).requires_grad_(True)
    y = layer(xb, n_vision=1400)
    g = torch.randn_like(y)
    y.backward(g)
    P = {n: p.detach().float().requires_grad_(True) for n, p in layer.named_parameters()}
    xr = xb.detach().float().requires_grad_(True)
    yr = _torch_reference(P, layer.hq, layer.hkv, layer.rope_theta, xr)
    yr.backward(g.float())
    np.testing.assert_allclose(y.float().detach().cpu().numpy(), yr.detach().cpu().numpy(), atol=3e-2, rtol=3e-2)
    rel = lambda a, b: float((a.float() - b).norm() / b.norm())
    assert rel(xb.grad, xr.grad) < 3e-2
    for name, p in layer.named_parameters():
        assert rel(p.grad, P[name].grad) < 3e-2, name


def test_layer_sparse_matches_pipeline_and_packing():
    """Default sparsity: the layer's attention core is the prefill pipeline's
    output bit for bit; packed sequences equal separate calls."""
    from paper_2511_12201_b200.attention import concat_heads
    from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device

    layer = _layer(SparsityConfig())
    torch.manual_seed(2)
    xa = torch.randn(2100, 512, device="cuda", dtype=torch.bfloat16)
    xb = torch.randn(1333, 512, device="cuda", dtype=torch.bfloat16)
    with torch.no_grad():
        q, k, v = layer.qkv(xa)
        core = layer.attend(q, k, v, 2000)
        res = sparse_prefill_device(q, k, v, 2000, layer.cfg)
        assert torch.equal(core.float(), concat_heads(res.outputs))
        ya, yb = layer(xa, 2000), layer(xb, 1300)
        packed = layer(torch.cat([xa, xb]), [2000, 1300], cu_seqlens=[0, 2100, 3433])
    # same attention cores; the o_proj GEMM may pick another cuBLAS kernel for another M
    torch.testing.assert_close(packed, torch.cat([ya, yb]), atol=1e-2, rtol=1e-2)
    assert bool(torch.isfinite(packed).all())
