"""K1 / K2 alone at the bench workload (64K, 28/4 heads): mean of 20 launches."""
import json, sys, torch
sys.path.insert(0, ".")
from paper_2511_12201_b200 import ops
from paper_2511_12201_b200.synthetic import generate_device
n = 65536; nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=0)
O = torch.empty_like(Q)
def t(fn, k=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(k): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / k
kl, ka, _ = ops.kv_probe(K, nv, 0, 256)
k1 = t(lambda: ops.kv_probe(K, nv, 0, 256))
k2 = t(lambda: ops.q_score(Q, kl, ka, nv, 0.08, True, 256, O_zero=O))
act, *_ = ops.q_score(Q, kl, ka, nv, 0.08, True, 256, O_zero=O)
print(json.dumps({"k1_ms": k1, "k2_ms": k2, "active_sum": int(act.sum())}))
