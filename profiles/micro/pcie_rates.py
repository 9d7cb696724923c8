"""Host<->device copy rates on the box: H2D alone, D2H alone, both at once
(separate streams), pinned memory, 470 MB / 604 MB payloads as in bench e2e."""
import json, torch, time
MB = 1 << 20
h_in = torch.empty(604 * MB, dtype=torch.uint8).pin_memory()
h_out = torch.empty(470 * MB, dtype=torch.uint8).pin_memory()
d_in = torch.empty(604 * MB, dtype=torch.uint8, device="cuda")
d_out = torch.empty(470 * MB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps
def h2d():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
def both():
    h2d(); d2h()
r = {"h2d_ms": 1e3 * timed(h2d), "d2h_ms": 1e3 * timed(d2h), "both_ms": 1e3 * timed(both)}
r["h2d_GBs"] = 604 * MB / (r["h2d_ms"] / 1e3) / 1e9
r["d2h_GBs"] = 470 * MB / (r["d2h_ms"] / 1e3) / 1e9
print(json.dumps(r))
