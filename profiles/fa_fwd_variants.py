"""Times the K4 forward kernel variants (exp2 MUFU/FMA split) at the bench
workload; each variant runs in its own process (the choice is read once)."""
import os, subprocess, sys, json
code = r'''
import sys, torch, json
sys.path.insert(0, ".")
from paper_2511_12201_b200 import ops
from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device
from paper_2511_12201_b200.synthetic import generate_device
n=65536; nv=n-64
Q,K,V = generate_device(28,4,128,nv,64,seed=0)
O=torch.empty_like(Q)
r=sparse_prefill_device(Q,K,V,nv,SparsityConfig(),out=O)
fa=lambda: ops.sparse_attn_fwd(Q, r.K_sel, r.V_sel, V, r.rows, r.counts, r.selection.selected, r.selection.counts, 0, O, r.lse)
for _ in range(3): fa()
torch.cuda.synchronize()
s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): fa()
e.record(); torch.cuda.synchronize()
print(json.dumps({"ms": s.elapsed_time(e)/10}))
'''
res = {}
for v in range(4):
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, OMNI_FWD_POLY=str(v)),
                         capture_output=True, text=True)
    res[v] = json.loads(out.stdout.strip().splitlines()[-1])["ms"] if out.returncode == 0 else out.stderr[-300:]
print(json.dumps(res))
