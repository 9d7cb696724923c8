"""K1 / K2 device time at the bench workload: eager calls (host overhead
included: allocations + ctypes per call) vs one CUDA graph of 20 calls
replayed (the kernels back to back on the device)."""
import json, sys, time, torch
sys.path.insert(0, ".")
from paper_2511_12201_b200 import ops
from paper_2511_12201_b200.synthetic import generate_device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
nv = n - 64
Q, K, V = generate_device(28, 4, 128, nv, 64, seed=0)
O = torch.empty_like(Q)
kl, ka, _ = ops.kv_probe(K, nv, 0, 256)
def eager(fn, k=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(k): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / k
def graphed(fn, k=20, reps=5):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()  # warm the allocator on the capture stream
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            for _ in range(k): fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); g.replay(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / k)
    return best
k1 = lambda: ops.kv_probe(K, nv, 0, 256)
k2 = lambda: ops.q_score(Q, kl, ka, nv, 0.08, True, 256, O_zero=O)
res = {"n": n, "k1_eager_ms": eager(k1), "k2_eager_ms": eager(k2)}
time.sleep(1.0)
try:
    res["k1_graph_ms"] = graphed(k1)
except Exception as ex:  # noqa: BLE001
    res["k1_graph_error"] = str(ex)[:300]
try:
    res["k2_graph_ms"] = graphed(k2)
except Exception as ex:  # noqa: BLE001
    res["k2_graph_error"] = str(ex)[:300]
kl2, ka2, _ = ops.kv_probe(K, nv, 0, 256)
res["k1_after_graph_equal"] = bool(torch.equal(kl, kl2) and torch.equal(ka, ka2))
print(json.dumps(res))
