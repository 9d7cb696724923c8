"""Small-shape runs of the warp-specialised mbarrier / TMEM kernels for
compute-sanitizer racecheck / synccheck (r02): K4 forward (fast + safe),
K5 backward (bwd_prep, dq with Q in TMEM, dkv2), K7 paged decode, and the
K1 / K2 persistent stream kernels, at sizes where the tools
finish in minutes (GQA 8 / 2 heads, ragged N)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2511_12201_b200 import decode as gdec  # noqa: E402
from paper_2511_12201_b200 import ops  # noqa: E402
from paper_2511_12201_b200.autograd import sparse_attention  # noqa: E402
from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device  # noqa: E402
from paper_2511_12201_b200.synthetic import decode_queries_device, generate_device, unit_vision_mean  # noqa: E402

nv, nt = 1200, 77
Q, K, V = generate_device(8, 2, 128, nv, nt, seed=1)
res = sparse_prefill_device(Q, K, V, nv, SparsityConfig())
# the safe kernel too (status = NULL selects it)
O2 = torch.empty_like(Q)
lse = torch.empty(8, nv + nt, device="cuda")
sel = res.selection
ops._lib.call("omni_sparse_attn_fwd", ops._p(Q), ops._p(res.K_sel), ops._p(res.V_sel), ops._p(V), ops._p(res.rows),
              ops._p(res.counts), ops._p(sel.selected), ops._p(sel.counts), 8, 2, nv + nt, 128, res.K_sel.shape[1], 0,
              ops._p(O2), ops._p(lse), ops._stream())
Qg, Kg, Vg = (x.clone().requires_grad_(True) for x in (Q, K, V))
sparse_attention(Qg, Kg, Vg, nv, SparsityConfig()).backward(torch.randn_like(Q))
cache = gdec.cache_from_prompt(Q, K, V, nv, nt, SparsityConfig(), answer_capacity=8)
means = [unit_vision_mean(K, nv)]
for t in range(2):
    gdec.decode_attention_batch(decode_queries_device(8, 2, means, [0], 0.5, t), cache, 0.08)
    gdec.append_answer_batch(cache, torch.randn(1, 2, 128, device="cuda"), torch.randn(1, 2, 128, device="cuda"))
# K1 / K2 persistent streams with several items per CTA (ring wrap-around,
# slab double buffer, mbarrier hand-offs): 16K tokens, 8 Q / 2 KV heads =
# 512 K2 items over at most 148 CTAs
Qs, Ks, _ = generate_device(8, 2, 128, 16384 - 64, 64, seed=2)
kl, ka, _ = ops.kv_probe(Ks, 16384 - 64, 0, 256)
Oz = torch.empty_like(Qs)
ops.q_score(Qs, kl, ka, 16384 - 64, 0.08, True, 256, O_zero=Oz)
torch.cuda.synchronize()
print("ok")
