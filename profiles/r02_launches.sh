#!/bin/bash
# Per-launch list (ncu, serialised, cold-ish caches) of the prefill bench step at 64K:
# every kernel of one untimed + timed step with its duration and DRAM bytes.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled -k regex:omni -c 44 --csv \
    --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-dense --no-knobs --no-e2e \
    --no-cpu --no-train --no-decode > gpurun_out/r02_launches.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r02_launches.csv')))
i=[k for k,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[i]; data=rows[i+1:]
ik=h.index('Kernel Name'); im=h.index('Metric Name'); iv=h.index('Metric Value'); iid=h.index('ID')
from collections import OrderedDict
k=OrderedDict()
for r in data:
    k.setdefault(r[iid],{'name':r[ik]})[r[im]]=r[iv]
out=open('gpurun_out/r02_launches.txt','w')
for id_,v in k.items():
    print(id_, v.get('gpu__time_duration.sum'), v.get('dram__bytes_read.sum'), v.get('dram__bytes_write.sum'), v['name'][:110], file=out)
PY
tail -40 gpurun_out/r02_launches.txt
