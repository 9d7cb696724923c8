"""Per-kernel device times of one prefill step (CUPTI via torch.profiler) at
N tokens (default 32K): where the non-K4 time goes."""
import json, sys, torch
from collections import defaultdict
sys.path.insert(0, ".")
from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device
from paper_2511_12201_b200.synthetic import generate_device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=0)
O = torch.empty_like(Q)
for _ in range(3): sparse_prefill_device(Q, K, V, nv, SparsityConfig(), out=O)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5): sparse_prefill_device(Q, K, V, nv, SparsityConfig(), out=O)
    torch.cuda.synchronize()
acc = defaultdict(list)
for e in prof.events():
    if e.device_type.name == "CUDA":
        acc[e.name.split("(")[0][-50:]].append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time)
tot = sum(sum(v) for v in acc.values()) / 5
print(json.dumps({"tokens": n, "sum_ms": tot / 1000, **{k: round(sum(v) / 5 / 1000, 4) for k, v in
                  sorted(acc.items(), key=lambda kv: -sum(kv[1]))}}))
