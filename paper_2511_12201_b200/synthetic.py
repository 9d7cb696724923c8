"""Device-side synthetic workloads for benchmarking.

Same construction and constants as the reference generator
(``workload.py:31-37``, ``:88-129``; restated bit-exactly on the CPU in
``oracle/workload.py``) but drawn with torch's CUDA RNG, so 64K-128K token
layers are generated in milliseconds instead of minutes. Statistically the
same workload (lazy fraction, hot keys, sharpness profile over KV groups);
not bit-identical to the NumPy stream — parity tests use the oracle generator.
"""

from __future__ import annotations

import math

import torch

CONTENT_SCALE = 0.4
SINK_NORM = 0.2
ACTIVE_ALIGN = 3.0
LAZY_ANTI_ALIGN = 9.0
HOT_KEY_SCALE = 0.9
HOT_QUERY_MEAN = 3.0
HOT_FRACTION = 0.03


def _unit(gen, d, device):
    v = torch.randn(d, generator=gen, device=device)
    return v / v.norm()


def generate_device(hq: int, hkv: int, d: int, n_vision: int, n_text: int, seed: int = 0,
                    lazy_fraction: float = 0.5, sink_index: int = 0, device="cuda", dtype=torch.bfloat16,
                    make_q: bool = True):
    """Returns (Q [hq,N,d] | None, K [hkv,N,d], V [hkv,N,d]) in ``dtype``."""
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    n = n_vision + n_text
    sqd = math.sqrt(d)
    pool = torch.arange(n_vision, device=device)
    pool = pool[pool != sink_index]
    n_lazy = min(int(round(lazy_fraction * n_vision)), pool.numel())
    lazy_rows = pool[torch.randperm(pool.numel(), generator=gen, device=device)[:n_lazy]]
    lazy = torch.zeros(n, dtype=torch.bool, device=device)
    lazy[lazy_rows] = True
    act = ~lazy
    n_hot = max(2, int(round(HOT_FRACTION * n_vision)))
    prof = torch.zeros(1) if hkv == 1 else torch.linspace(0.0, 1.0, hkv)
    rep = hq // hkv
    Q = torch.empty(hq, n, d, device=device, dtype=dtype) if make_q else None
    K = torch.empty(hkv, n, d, device=device, dtype=dtype)
    V = torch.empty(hkv, n, d, device=device, dtype=dtype)
    for g in range(hkv):
        c = float(prof[g])
        u_content, u_sink, u_hot = (_unit(gen, d, device) for _ in range(3))
        k = torch.randn(n, d, generator=gen, device=device)
        k[:n_vision] += CONTENT_SCALE * sqd * u_content
        hot = pool[torch.randperm(pool.numel(), generator=gen, device=device)[:n_hot]]
        k[hot] += c * HOT_KEY_SCALE * sqd * u_hot
        k[sink_index] = SINK_NORM * sqd * u_sink
        K[g] = k.to(dtype)
        if make_q:
            for r in range(rep):
                q = torch.randn(n, d, generator=gen, device=device)
                q[lazy] -= LAZY_ANTI_ALIGN * u_content
                q[act] += ACTIVE_ALIGN * u_content
                mag = (torch.randn(int(act.sum()), 1, generator=gen, device=device) + HOT_QUERY_MEAN).abs()
                q[act] += c * mag * u_hot
                Q[g * rep + r] = q.to(dtype)
        V[g] = torch.randn(n, d, generator=gen, device=device).to(dtype)
    return Q, K, V


def decode_queries_device(hq: int, hkv: int, u_content: list, seeds, lazy_fraction: float, step: int,
                          dtype=torch.bfloat16):
    """``workload.py:132-157`` on the device: one decoding query per Q head,
    lazy with probability ``lazy_fraction``, aligned (+ACTIVE_ALIGN) or
    anti-aligned (-LAZY_ANTI_ALIGN) with its group's unit vision-key mean.
    u_content: per sequence [hkv, d] unit vectors. Returns [B, hq, d]."""
    rep = hq // hkv
    qs = []
    for u, seed in zip(u_content, seeds):
        gen = torch.Generator(device=u.device)
        gen.manual_seed(10_000 * int(seed) + step)
        q = torch.randn(hq, u.shape[1], generator=gen, device=u.device)
        lazy = torch.rand(hq, generator=gen, device=u.device) < lazy_fraction
        coef = torch.where(lazy, torch.full_like(q[:, 0], -LAZY_ANTI_ALIGN), torch.full_like(q[:, 0], ACTIVE_ALIGN))
        q += coef[:, None] * u.repeat_interleave(rep, dim=0)
        qs.append(q)
    return torch.stack(qs).to(dtype)


def unit_vision_mean(K: torch.Tensor, n_vision: int) -> torch.Tensor:
    m = K[:, :n_vision].float().mean(dim=1)
    return m / m.norm(dim=1, keepdim=True)
