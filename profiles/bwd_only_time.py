"""K5 alone (ops.sparse_attn_bwd: prep + dq + dkv2) at 32K, 28/4 heads:
CUDA-event mean of 10 launches, 3 repeats."""
import json, sys, torch
sys.path.insert(0, ".")
from paper_2511_12201_b200 import ops
from paper_2511_12201_b200.pipeline import SparsityConfig, select_device
from paper_2511_12201_b200.synthetic import generate_device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=3)
_, _, _, _, _, _, rows, counts, _, sel = select_device(Q, K, nv, SparsityConfig())
cap = ops.round_up(n, ops.TILE)
K_sel = ops.gather_rows(K, sel.selected, sel.counts, cap, ops.TILE)
V_sel = ops.gather_rows(V, sel.selected, sel.counts, cap, ops.TILE)
O = torch.zeros_like(Q)
lse = torch.empty(28, n, device=Q.device, dtype=torch.float32)
ops.sparse_attn_fwd(Q, K_sel, V_sel, V, rows, counts, sel.selected, sel.counts, 0, O, lse)
dO = torch.randn_like(Q)
bwd = lambda: ops.sparse_attn_bwd(Q, K_sel, V_sel, O, dO, lse, rows, counts, sel.selected, sel.counts,
                                  dq_dtype=torch.bfloat16)
for _ in range(3): bwd()
torch.cuda.synchronize()
ms = []
for _ in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): bwd()
    e.record(); torch.cuda.synchronize()
    ms.append(s.elapsed_time(e) / 10)
dq, dk, dv, dvs = bwd()
print(json.dumps({"n": n, "bwd_ms": ms, "dk_sum": float(dk.double().abs().sum()), "dq_sum": float(dq.double().abs().sum())}))
