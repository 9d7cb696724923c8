"""Times K4 (sparse_fwd_kernel) alone at the bench workload (64K, defaults);
each OMNI_FWD_POLY variant in its own process (the choice is read once)."""
import json, os, subprocess, sys
code = r'''
import sys, torch, json
sys.path.insert(0, ".")
from paper_2511_12201_b200 import ops
from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device
from paper_2511_12201_b200.synthetic import generate_device
n = int(sys.argv[1]); nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=0)
O = torch.empty_like(Q)
r = sparse_prefill_device(Q, K, V, nv, SparsityConfig(), out=O)
fa = lambda: ops.sparse_attn_fwd(Q, r.K_sel, r.V_sel, V, r.rows, r.counts, r.selection.selected, r.selection.counts, 0, O, r.lse)
for _ in range(3): fa()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): fa()
e.record(); torch.cuda.synchronize()
print(json.dumps({"ms": s.elapsed_time(e) / 10}))
'''
n = sys.argv[1] if len(sys.argv) > 1 else "65536"
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["0"]
res = {}
for v in variants:
    out = subprocess.run([sys.executable, "-c", code, n], env=dict(os.environ, OMNI_FWD_POLY=v), capture_output=True, text=True)
    res[v] = json.loads(out.stdout.strip().splitlines()[-1])["ms"] if out.returncode == 0 else out.stderr[-400:]
print(json.dumps(res))
