"""Cycle accounting of the shared-S K4 variant (OMNI_FWD_IMPL=sp,
OMNI_FWD_TRACE=1, variants build) at the bench workload: where the MMA issuer
and the softmax warps wait, per MMA round / per softmax step."""
import ctypes, json, os, sys
os.environ["OMNI_FWD_TRACE"] = "1"
os.environ["OMNI_FWD_IMPL"] = "sp"
os.environ.setdefault("OMNI_LIBRARY", os.path.join("paper_2511_12201_b200", "lib", "libomnisparse_variants.so"))
sys.path.insert(0, ".")
import torch
from paper_2511_12201_b200 import _lib, ops
from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device
from paper_2511_12201_b200.synthetic import generate_device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=0)
O = torch.empty_like(Q)
r = sparse_prefill_device(Q, K, V, nv, SparsityConfig(), out=O)
lib = _lib.load()
lib.omni_debug_fwd_sp_trace.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 8)()
fa = lambda: ops.sparse_attn_fwd(Q, r.K_sel, r.V_sel, V, r.rows, r.counts, r.selection.selected, r.selection.counts, 0, O, r.lse)
fa(); torch.cuda.synchronize()
lib.omni_debug_fwd_sp_trace(buf)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); fa(); e.record(); torch.cuda.synchronize()
lib.omni_debug_fwd_sp_trace(buf)
v = list(buf)
rounds = v[7]
steps = rounds  # softmax steps per warp ~ rounds per CTA (per tile); normalised per round below
print(json.dumps({"ms": s.elapsed_time(e), "mma_rounds": rounds,
                  "mma_per_round": {"wait_S_free": v[0] / rounds, "wait_P": v[1] / rounds, "wait_KVQ": v[2] / rounds,
                                    "loop": v[3] / rounds},
                  "softmax_per_warp_round": {"wait_S": v[4] / (16 * rounds), "wait_PV": v[5] / (16 * rounds),
                                             "loop": v[6] / (16 * rounds)}}))
