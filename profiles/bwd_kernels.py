"""Per-kernel device times of the C4 backward (32K, 28/4 heads) from a CUPTI
trace (torch.profiler): decision support for K5 variants, not a bench number.
Env knobs (OMNI_BWD_PROBE, OMNI_BWD_DKV) select kernel variants."""
import json, sys, torch
from collections import defaultdict
sys.path.insert(0, ".")
from paper_2511_12201_b200 import ops
from paper_2511_12201_b200.autograd import SparseAttentionFn, plan_from_selection
from paper_2511_12201_b200.pipeline import SparsityConfig, select_device
from paper_2511_12201_b200.synthetic import generate_device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=3)
for t in (Q, K, V): t.requires_grad_(True)
dO = torch.randn_like(Q)
with torch.no_grad():
    _, _, _, _, _, _, rows, counts, _, sel = select_device(Q.detach(), K.detach(), nv, SparsityConfig())
plan = plan_from_selection(rows, counts, sel, 0)
def step():
    O = SparseAttentionFn.apply(Q, K, V, plan); O.backward(dO)
for _ in range(3): step()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5): step()
    torch.cuda.synchronize()
acc = defaultdict(list)
for e in prof.events():
    if e.device_type.name == "CUDA" and ("omni" in e.name or "bwd" in e.name or "dkv" in e.name or "dq" in e.name
                                         or "fwd" in e.name):
        acc[e.name.split("(")[0][-60:]].append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time)
print(json.dumps({k: round(sum(v) / len(v) / 1000, 4) for k, v in acc.items()}))
