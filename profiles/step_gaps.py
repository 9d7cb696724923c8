"""Prefill step time vs the sum of its kernels' standalone times (32K and
64K): the difference bounds what launch-gap removal (PDL / graphs) can win."""
import json, sys, torch
sys.path.insert(0, ".")
from paper_2511_12201_b200 import ops
from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device
from paper_2511_12201_b200.synthetic import generate_device


def t(fn, k=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(k):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / k


for n in (32768, 65536):
    nv = n - 64
    Q, K, V = generate_device(28, 4, 128, nv, 64, seed=0)
    O = torch.empty_like(Q)
    cfg = SparsityConfig()
    r = sparse_prefill_device(Q, K, V, nv, cfg, out=O)
    step = t(lambda: sparse_prefill_device(Q, K, V, nv, cfg, out=O))
    kl, ka, pk = ops.kv_probe(K, nv, 0, 256)
    act, _, pq, bact = ops.q_score(Q, kl, ka, nv, 0.08, True, 256, O_zero=O)
    mass = ops.probe_mass(pq, pk)
    cap = ops.round_up(n, 128)
    parts = {
        "K1": t(lambda: ops.kv_probe(K, nv, 0, 256)),
        "K2": t(lambda: ops.q_score(Q, kl, ka, nv, 0.08, True, 256, O_zero=O)),
        "K3a": t(lambda: ops.probe_mass(pq, pk)),
        "K3b": t(lambda: ops.select(mass, 4, n, 256, 0.82)),
        "gatherK": t(lambda: ops.gather_rows(K, r.selection.selected, r.selection.counts, cap, 128)),
        "K4": t(lambda: ops.sparse_attn_fwd(Q, r.K_sel, r.V_sel, V, r.rows, r.counts, r.selection.selected,
                                           r.selection.counts, 0, O, r.lse)),
    }
    print(json.dumps({"n": n, "step_ms": step, "sum_of_parts_ms": sum(parts.values()), "parts_ms": parts}))
