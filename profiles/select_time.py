"""Times the selection-path kernels alone at the bench workload (64K tokens,
28 / 4 heads, reference defaults): K1 kv_probe, K2 q_score, compaction, K3a
probe_mass, K3b select, K6 gather; mean of 20 back-to-back calls each."""
import json, sys, torch
sys.path.insert(0, ".")
from paper_2511_12201_b200 import ops
from paper_2511_12201_b200.synthetic import generate_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=0)
O = torch.empty_like(Q)


def t(fn, k=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(k):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / k * 1e3  # us


kl, ka, pk = ops.kv_probe(K, nv, 0, 256)
act, _, pq, bact = ops.q_score(Q, kl, ka, nv, 0.08, True, 256, O_zero=O)
mass = ops.probe_mass(pq, pk)
sel = ops.select(mass, 4, n, 256, 0.82)
res = {
    "K1_kv_probe_us": t(lambda: ops.kv_probe(K, nv, 0, 256)),
    "K2_q_score_us": t(lambda: ops.q_score(Q, kl, ka, nv, 0.08, True, 256, O_zero=O)),
    "compact_us": t(lambda: ops.compact_rows(act, bact, 256)),
    "K3a_probe_mass_us": t(lambda: ops.probe_mass(pq, pk)),
    "K3b_select_us": t(lambda: ops.select(mass, 4, n, 256, 0.82)),
}
print(json.dumps(res))
