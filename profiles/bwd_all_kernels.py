"""Every device kernel / memset / copy of one C4 fwd+bwd step (CUPTI via
torch.profiler), to find time outside the K4 / K5 kernels."""
import sys, torch
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
def step():
    for t in (Q, K, V): t.grad = None
    O = SparseAttentionFn.apply(Q, K, V, plan); O.backward(dO)
for _ in range(3): step()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3): step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
