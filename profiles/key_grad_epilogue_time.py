"""Key-gradient epilogue at 32K (4 groups, bf16 leaves): fill + scatter.
Round-2 experiment: a single kernel writing every row (zeros where no key
maps, the ascending indices of a 256-row range found by two warp searches)
measured 21.4 us device time against 18.3 us for the fill + scatter pair
(CUDA graph of 20 calls) — the searches' latency outweighs the saved fill;
not kept. Times the current epilogue: eager and device time."""
import json, os, sys, torch
sys.path.insert(0, ".")
from paper_2511_12201_b200 import ops
from paper_2511_12201_b200.pipeline import SparsityConfig, select_device
from paper_2511_12201_b200.synthetic import generate_device
n = 32768; nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=3)
sel = select_device(Q, K, nv, SparsityConfig())[9]
cap = ops.round_up(n, ops.TILE)
src = torch.randn(4, cap, 128, device="cuda")
sink_add = torch.randn(4, 128, device="cuda")
two_step = True
def epi():
    out = (torch.zeros if two_step else torch.empty)(4, n, 128, device="cuda", dtype=torch.bfloat16)
    return ops.scatter_key_grads(src, sel.selected, sel.counts, out, 0, sink_add)
for _ in range(5): epi()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(50): epi()
e.record(); torch.cuda.synchronize()
eager = s.elapsed_time(e) / 50
sys.path.insert(0, ".")
from bench import time_graph  # device time: 20 calls in one CUDA graph
dev = time_graph(epi, 20, 5)
o = epi()
print(json.dumps({"two_step": two_step, "eager_ms": eager, "device_ms": dev, "checksum": float(o.double().sum())}))
