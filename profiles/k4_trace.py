"""K4 per-phase cycle accounting (OMNI_FWD_TRACE=1 build variant) at the bench workload."""
import ctypes, json, os, sys
os.environ["OMNI_FWD_TRACE"] = "1"
sys.path.insert(0, ".")
import torch
from paper_2511_12201_b200 import _lib, ops
from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device
from paper_2511_12201_b200.synthetic import generate_device
n = 65536; nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=0)
O = torch.empty_like(Q)
r = sparse_prefill_device(Q, K, V, nv, SparsityConfig(), out=O)
lib = _lib.load()
buf = (ctypes.c_ulonglong * 8)()
fa = lambda: ops.sparse_attn_fwd(Q, r.K_sel, r.V_sel, V, r.rows, r.counts, r.selection.selected, r.selection.counts, 0, O, r.lse)
fa(); torch.cuda.synchronize()
lib.omni_debug_fwd_trace(buf)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); fa(); e.record(); torch.cuda.synchronize()
lib.omni_debug_fwd_trace(buf)
v = list(buf)
tiles = v[5] / 8  # 8 softmax warps (per tile) each add nt... per (warp): count tile-iterations per warp
names = ["wait_S", "chunk0", "chunk1", "exchange", "tail+fixups+arrive"]
per = {nm: v[k] / v[5] for k, nm in enumerate(names)}
per["mma_wait_PF_per_tile"] = v[6] / (v[5] / 8)
print(json.dumps({"ms": s.elapsed_time(e), "cycles_per_warp_tile": per, "warp_tiles": v[5]}))
