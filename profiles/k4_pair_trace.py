"""CTA-pair K4 per-phase cycle accounting (OMNI_FWD_TRACE=1) at the bench workload.
argv[1]: OMNI_FWD_POLY (-1 = MMA/TMA pipeline only)."""
import ctypes, json, os, sys
os.environ["OMNI_FWD_TRACE"] = "1"
os.environ["OMNI_FWD_POLY"] = sys.argv[1] if len(sys.argv) > 1 else "4"
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
lib.omni_debug_fwd_pair_trace(buf)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); fa(); e.record(); torch.cuda.synchronize()
lib.omni_debug_fwd_pair_trace(buf)
v = list(buf)
steps = max(v[4], 1)
print(json.dumps({"ms": s.elapsed_time(e), "per_step_leader_mma": {"wait_P": v[0] / steps, "wait_V": v[1] / steps, "wait_K": v[2] / steps},
                  "per_step_softmax_warp": {"wait_S": v[5] / max(v[7], 1), "busy": v[6] / max(v[7], 1)}, "steps": v[4]}))
