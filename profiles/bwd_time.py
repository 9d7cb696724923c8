"""Times the C4 training step pieces at 32K (28/4 heads): selection, K4
forward, K5 backward (prep + dq + dkv), all on-device, mean of 10."""
import json, sys, torch
sys.path.insert(0, ".")
from paper_2511_12201_b200.autograd import SparseAttentionFn, plan_from_selection
from paper_2511_12201_b200.pipeline import SparsityConfig, select_device
from paper_2511_12201_b200.synthetic import generate_device
n = 32768; nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=3)
for t in (Q, K, V): t.requires_grad_(True)
dO = torch.randn_like(Q)
with torch.no_grad():
    _, _, _, _, _, _, rows, counts, _, sel = select_device(Q.detach(), K.detach(), nv, SparsityConfig())
plan = plan_from_selection(rows, counts, sel, 0)
def fwd():
    return SparseAttentionFn.apply(Q, K, V, plan)
def step():
    O = fwd(); O.backward(dO)
for _ in range(3): step()
torch.cuda.synchronize()
def t(fn, k=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(k): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / k
f = t(lambda: fwd())
fb = t(step)
print(json.dumps({"fwd_ms": f, "fwd_bwd_ms": fb, "bwd_ms": fb - f}))
