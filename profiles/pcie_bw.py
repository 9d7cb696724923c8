"""Host<->device copy bandwidth on the bench box (pinned buffers of the e2e
workload's sizes): H2D / D2H alone, split over several streams, and both
directions at once. CUDA-event timed."""
import json, torch
MB = 1 << 20
h2d_bytes, d2h_bytes = 604 * MB, 470 * MB
hs = torch.empty(h2d_bytes // 2, dtype=torch.bfloat16).pin_memory()
ho = torch.empty(d2h_bytes // 2, dtype=torch.bfloat16).pin_memory()
ds = torch.empty(h2d_bytes // 2, dtype=torch.bfloat16, device="cuda")
do = torch.empty(d2h_bytes // 2, dtype=torch.bfloat16, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); s.record()
        fn()
        for st in streams: torch.cuda.current_stream().wait_stream(st)
        e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best
def split_copy(dst, src, k, off=0):
    n = src.numel(); step = (n + k - 1) // k
    cur = torch.cuda.current_stream()
    for i in range(k):
        st = streams[off + i]; st.wait_stream(cur)
        with torch.cuda.stream(st):
            dst[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step], non_blocking=True)
res = {}
for k in (1, 2, 4):
    ms = timed(lambda: split_copy(ds, hs, k)); res[f"h2d_{k}streams_GBs"] = h2d_bytes / ms / 1e6
    ms = timed(lambda: split_copy(ho, do, k)); res[f"d2h_{k}streams_GBs"] = d2h_bytes / ms / 1e6
for k in (1, 2):
    ms = timed(lambda: (split_copy(ds, hs, k), split_copy(ho, do, k, off=4)))
    res[f"both_{k}streams_ms"] = ms
    res[f"both_{k}streams_h2d_equiv_GBs"] = h2d_bytes / ms / 1e6
print(json.dumps(res))
