import sys, torch
sys.path.insert(0, '.')
from paper_2511_12201_b200.autograd import SparseAttentionFn, plan_from_selection
from paper_2511_12201_b200.pipeline import SparsityConfig, select_device
from paper_2511_12201_b200.synthetic import generate_device
n = 32768; nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=3)
for t in (Q, K, V): t.requires_grad_(True)
dO = torch.randn_like(Q)
for _ in range(2):
    with torch.no_grad():
        _, _, _, _, _, _, rows, counts, _, sel = select_device(Q.detach(), K.detach(), nv, SparsityConfig())
    O = SparseAttentionFn.apply(Q, K, V, plan_from_selection(rows, counts, sel, 0))
    O.backward(dO)
torch.cuda.synchronize()
