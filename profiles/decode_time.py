"""Decode step time at the bench shape (batch 32 x 64K, 28/4 heads), mean of
50 steps; OMNI_DECODE_IMPL selects the K7 variant."""
import json, sys, torch
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
q = decode_queries_device(HQ, HKV, means, range(B), 0.5, 0)
for _ in range(5): gdec.decode_attention_batch(q, cache, cfg.tau, log=False)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(50): gdec.decode_attention_batch(q, cache, cfg.tau, log=False)
e.record(); torch.cuda.synchronize()
out, fl = gdec.decode_attention_batch(q, cache, cfg.tau, log=False)
print(json.dumps({"ms": s.elapsed_time(e) / 50, "flags": int(fl.sum()), "out_sum": float(out.double().sum())}))
