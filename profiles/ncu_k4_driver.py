"""K4 alone at the bench workload (64K, defaults) for ncu: selection once, then
3 K4 launches (capture the 3rd with -s 2 -c 1 -k regex:sparse_fwd)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2511_12201_b200 import ops
from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device
from paper_2511_12201_b200.synthetic import generate_device
n = 65536; nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=0)
O = torch.empty_like(Q)
r = sparse_prefill_device(Q, K, V, nv, SparsityConfig(), out=O)
for _ in range(3):
    ops.sparse_attn_fwd(Q, r.K_sel, r.V_sel, V, r.rows, r.counts, r.selection.selected, r.selection.counts, 0, O, r.lse)
torch.cuda.synchronize()
