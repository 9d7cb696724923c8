"""Diagnostic: K3b general path on the near-tie p values of the parity test."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import selection as osel  # noqa: E402
from paper_2511_12201_b200 import ops  # noqa: E402

for n in (5000, 70001):
    rng = np.random.default_rng(n)
    a = np.abs(rng.standard_normal(n)) * np.exp(rng.standard_normal(n))
    cum = np.cumsum(np.sort(a)[::-1])
    ps = []
    for k in (n // 3, n // 2, (9 * n) // 10):
        p0 = cum[k] / cum[-1]
        ps += [p0, np.nextafter(p0, 0.0), np.nextafter(p0, 1.0), cum[k - 1] / cum[-1]]
    ps.append(1.0)
    t = torch.from_numpy(a[None]).cuda()
    for p in ps:
        try:
            sel = ops.select(t, 1, n, 1, float(p), "token")
            st = sel.stats.cpu().numpy()
            print(n, repr(float(p)), "ok", int(sel.info[0]), osel.budget(a, float(p))[0], st[3:5], flush=True)
        except Exception as e:  # noqa: BLE001
            print(n, repr(float(p)), "ERR", e, flush=True)
