#!/bin/bash
# Every kernel of one C4 training step (32K, fwd + bwd incl. selection and autograd glue), ncu durations.
mkdir -p gpurun_out
cat > /tmp/train_step.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2511_12201_b200.autograd import SparseAttentionFn, plan_from_selection
from paper_2511_12201_b200.pipeline import SparsityConfig, select_device
from paper_2511_12201_b200.synthetic import generate_device
n = 32768; nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=3)
for t in (Q, K, V): t.requires_grad_(True)
dO = torch.randn_like(Q)
def step():  # as bench.py's sparse_step: K2 zeroes the output's lazy rows during the selection
    out = torch.empty(Q.shape, device=Q.device, dtype=torch.bfloat16)
    with torch.no_grad():
        _, _, _, _, _, _, rows, counts, _, sel = select_device(Q.detach(), K.detach(), nv, SparsityConfig(), O_zero=out)
    O = SparseAttentionFn.apply(Q, K, V, plan_from_selection(rows, counts, sel, 0, out))
    O.backward(dO)
for _ in range(2): step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
PY
ncu --metrics gpu__time_duration.sum --profile-from-start off --csv --log-file gpurun_out/r02_train_launches.csv python /tmp/train_step.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r02_train_launches.csv')))
i=[k for k,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[i]; data=rows[i+1:]
ik=h.index('Kernel Name'); iv=h.index('Metric Value'); iu=h.index('Metric Unit')
out=open('gpurun_out/r02_train_launches.txt','w'); tot=0
for r in data:
    v=float(r[iv].replace(',','')); v = v/1000 if r[iu]=='us' else v/1e6 if r[iu]=='ns' else v
    tot+=v; print(f"{v:9.4f} ms  {r[ik][:120]}", file=out)
print(f"total {tot:.3f} ms", file=out)
PY
cat gpurun_out/r02_train_launches.txt
