"""K4 variants (OMNI_FWD_IMPL=pp / db / sp, variants build; other builds by
library suffix) against the default single-CTA kernel at the bench workload: output / LSE differences and
CUDA-event times, each implementation in its own process."""
import json, os, subprocess, sys
code = r'''
import sys, torch, json
sys.path.insert(0, ".")
from paper_2511_12201_b200 import ops
from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device
from paper_2511_12201_b200.synthetic import generate_device
n = int(sys.argv[1]); nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=0)
O = torch.zeros_like(Q)
r = sparse_prefill_device(Q, K, V, nv, SparsityConfig(), out=O)
fa = lambda: ops.sparse_attn_fwd(Q, r.K_sel, r.V_sel, V, r.rows, r.counts, r.selection.selected, r.selection.counts, 0, O, r.lse)
for _ in range(3): fa()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for rep in range(3):
    s.record()
    for _ in range(10): fa()
    e.record(); torch.cuda.synchronize()
    ms.append(s.elapsed_time(e) / 10)
torch.save({"O": O.cpu(), "lse": r.lse.cpu()}, sys.argv[2])
print(json.dumps({"ms": ms, "status": int(ops.last_fwd_status[0])}))
'''
n = sys.argv[1] if len(sys.argv) > 1 else "65536"
impls = sys.argv[2].split(",") if len(sys.argv) > 2 else ["single", "pp"]
lib = os.path.join("paper_2511_12201_b200", "lib", "libomnisparse_variants.so")
res = {}
for impl in impls:
    # "impl[:poly][@library-suffix]", e.g. "single@wpf" -> lib/libomnisparse_wpf.so
    spec, _, libsfx = impl.partition("@")
    name, _, poly = spec.partition(":")
    lib_i = os.path.join("paper_2511_12201_b200", "lib", f"libomnisparse_{libsfx}.so") if libsfx else lib
    env = dict(os.environ, OMNI_FWD_IMPL=name, OMNI_LIBRARY=lib_i, OMNI_FWD_POLY=poly or "6")
    out = subprocess.run([sys.executable, "-c", code, n, f"/tmp/k4_{impl}.pt"], env=env, capture_output=True, text=True)
    res[impl] = json.loads(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else out.stderr[-600:]
import torch
ref = torch.load(f"/tmp/k4_{impls[0]}.pt")
for impl in impls[1:]:
    if not isinstance(res[impl], dict):
        continue
    o = torch.load(f"/tmp/k4_{impl}.pt")
    d = (o["O"].float() - ref["O"].float()).abs()
    fin = torch.isfinite(ref["lse"])
    res[impl]["max_abs_O_vs_" + impls[0]] = float(d.max())
    res[impl]["max_abs_lse_vs_" + impls[0]] = float((o["lse"][fin] - ref["lse"][fin]).abs().max())
print(json.dumps({"n": n, **res}))
