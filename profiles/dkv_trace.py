"""dkv2 per-phase cycle accounting (OMNI_BWD_PROBE=3) at C4 (32K, 28/4 heads)."""
import ctypes, json, os, sys
os.environ["OMNI_BWD_PROBE"] = "3"
sys.path.insert(0, ".")
import torch
from paper_2511_12201_b200 import _lib
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
lib = _lib.load()
buf = (ctypes.c_ulonglong * 8)()
O = SparseAttentionFn.apply(Q, K, V, plan); O.backward(dO); torch.cuda.synchronize()
lib.omni_debug_bwd_trace(buf)
O = SparseAttentionFn.apply(Q, K, V, plan); O.backward(dO); torch.cuda.synchronize()
lib.omni_debug_bwd_trace(buf)
v = list(buf)
g = {nm: v[k] / v[6] for k, nm in enumerate(["wait_ST", "P_phase", "wait_dPT"])}; g["dS_phase"] = v[4] / v[6]; g["mma_wait_QF"] = v[3] / v[7]
m = {"grad_wait_IF": v[5] / v[6]}
print(json.dumps({"grad_cycles_per_step": g, "mma_cycles_per_step": m, "steps": v[7]}))
