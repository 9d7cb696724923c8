"""Decode workload for ncu: batch 32 paged slim caches at 64K (bench shape), 3 steps."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2511_12201_b200 import decode as gdec  # noqa: E402
from paper_2511_12201_b200.pipeline import SparsityConfig  # noqa: E402
from paper_2511_12201_b200.synthetic import decode_queries_device, generate_device, unit_vision_mean  # noqa: E402

n = 65536
nv = n - 64
B, HQ, HKV, D = 32, 28, 4, 128
cfg = SparsityConfig()
gdec.default_pool(torch.device("cuda")).reserve(B * HKV * (-(-int(0.6 * nv) // 64) + 4))
caches, means = [], []
for s in range(B):
    Q, K, V = generate_device(HQ, HKV, D, nv, 64, seed=1000 + s)
    caches.append(gdec.cache_from_prompt(Q, K, V, nv, 64, cfg, answer_capacity=16))
    means.append(unit_vision_mean(K, nv))
    del Q, K, V
cache = gdec.stack_caches(caches)
del caches
for t in range(3):
    q = decode_queries_device(HQ, HKV, means, range(B), 0.5, t)
    gdec.decode_attention_batch(q, cache, cfg.tau, log=False)
torch.cuda.synchronize()
