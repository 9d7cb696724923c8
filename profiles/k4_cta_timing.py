"""Per-CTA phases of the fast K4 kernel (profiling build with
-DOMNI_FWD_CTA_TIMING, OMNI_LIBRARY=libomnisparse_variants.so): prologue
(CTA start -> first QK issued), epilogue (last PV complete -> exit), CTA
lifetime, and the SM-time they add up to against 148 x the kernel time."""
import ctypes, json, sys, torch
sys.path.insert(0, ".")
from paper_2511_12201_b200 import ops, _lib
from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device
from paper_2511_12201_b200.synthetic import generate_device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=0)
O = torch.empty_like(Q)
r = sparse_prefill_device(Q, K, V, nv, SparsityConfig(), out=O)
fa = lambda: ops.sparse_attn_fwd(Q, r.K_sel, r.V_sel, V, r.rows, r.counts, r.selection.selected, r.selection.counts, 0, O, r.lse)
lib = _lib.load()
buf = (ctypes.c_ulonglong * 8)()
for _ in range(3): fa()
torch.cuda.synchronize()
lib.omni_debug_fwd_trace(buf)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
k = 5
s.record()
for _ in range(k): fa()
e.record(); torch.cuda.synchronize()
lib.omni_debug_fwd_trace(buf)
ms = s.elapsed_time(e) / k
ctas = buf[3] / k
if buf[3] == 0:
    print(json.dumps({"n": n, "k4_ms": ms, "note": "no fast-kernel CTAs timed"})); sys.exit(0)
print(json.dumps({"n": n, "k4_ms": ms, "ctas_per_launch": ctas, "prologue_us_per_cta": buf[0] / buf[3] / 1e3,
                  "epilogue_us_per_cta": buf[1] / buf[3] / 1e3, "cta_us": buf[2] / buf[3] / 1e3,
                  "sm_time_used_frac": buf[2] / k / 1e6 / (148 * ms),
                  "prologue_plus_epilogue_frac_of_sm_time": (buf[0] + buf[1]) / k / 1e6 / (148 * ms),
                  "effective_sm_clock_mhz": buf[4] / buf[2] * 1e3,
                  "start_to_loads_us": buf[6] / buf[3] / 1e3, "start_to_vis_us": buf[7] / buf[3] / 1e3,
                  "start_to_setup_barrier_us": buf[5] / buf[3] / 1e3}))
