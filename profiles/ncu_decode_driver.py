"""Decode workload for ncu: batch 32 slim caches at 64K (bench shape), 3 steps."""
import sys, torch
sys.path.insert(0, ".")
from paper_2511_12201_b200 import decode as gdec, ops
from paper_2511_12201_b200.pipeline import SparsityConfig, select_device
from paper_2511_12201_b200.synthetic import decode_queries_device, generate_device, unit_vision_mean
n = 65536; nv = n - 64; B = 32; HQ, HKV, D = 28, 4, 128
cfg = SparsityConfig()
caches, means = [], []
for s in range(B):
    Q, K, V = generate_device(HQ, HKV, D, nv, 64, seed=1000 + s)
    k_lazy, k_act, _, _, _, _, _, _, mass, sel = select_device(Q, K, nv, cfg)
    b = min(int(sel.info[0]), nv)
    vsel = ops.select(mass, HKV, n, 256, cfg.p, "token", vision_limit=nv, budget_override=b)
    caches.append(gdec.build_cache_device(K, V, vsel.selected, b, nv, 64, k_lazy, k_act, HQ, answer_capacity=16))
    means.append(unit_vision_mean(K, nv))
    del Q, K, V
cache = gdec.stack_caches(caches); del caches
for t in range(3):
    q = decode_queries_device(HQ, HKV, means, range(B), 0.5, t)
    gdec.decode_attention_batch(q, cache, cfg.tau, log=False)
torch.cuda.synchronize()
