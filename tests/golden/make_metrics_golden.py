"""Golden values for the reporting helpers, produced by the REFERENCE package
(build container only; /root/reference never travels to the GPU box):
``metrics.analytic_flops`` / ``metrics.kv_reduction`` on a grid of inputs,
``metrics.attention_recall`` on small maps, and an OMNT tensor file written
by ``tensorfile.save_tensor``. Writes tests/golden/metrics_golden.json and
tests/golden/omnt_ref.bin.

Usage: python tests/golden/make_metrics_golden.py (repo root).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))

from slimattn import metrics as r_m  # noqa: E402
from slimattn import tensorfile as r_tf  # noqa: E402


def main() -> None:
    out = {"analytic_flops": [], "kv_reduction": [], "recall": []}
    for n, nv, d, act, b, blk, probe in ((2048, 1984, 128, [2048, 1000, 1500, 700], 1054, 256, True),
                                         (65536, 65472, 128, [65536] + [33000] * 27, 30500, 256, True),
                                         (128, 120, 32, [128, 60, 70, 80], 55, None, False),
                                         (4096, 4000, 64, [4096, 2100], 2027, 16, True)):
        f = r_m.analytic_flops(n, nv, d, act, b, block_size=blk, probe_scores=probe)
        out["analytic_flops"].append({"args": [n, nv, d, act, b, blk, probe], "full": f.full, "sparse": f.sparse,
                                      "probe_overhead": f.probe_overhead, "reduction": f.reduction})
    for nv, b, d, ahs, ths in ((65472, 30500, 128, 900, 1000), (1984, 1054, 128, 0, 0), (120, 55, 32, 7, 8)):
        r = r_m.kv_reduction(nv, b, d, ahs, ths)
        out["kv_reduction"].append({"args": [nv, b, d, ahs, ths], "resident_reduction": r.resident_reduction,
                                    "fetch_reduction": r.fetch_reduction,
                                    "predicted_vision_tokens": r.predicted_vision_tokens,
                                    "predicted_vision_bytes": r.predicted_vision_bytes})
    rng = np.random.default_rng(5)
    for n in (16, 33):
        a = np.tril(rng.random((n, n)) + 0.01)
        a = a / a.sum(axis=1, keepdims=True)
        sel = np.sort(rng.choice(n, n // 2, replace=False))
        act = rng.random(n) < 0.6
        out["recall"].append({"map": a.tolist(), "selected": sel.tolist(), "active": act.tolist(),
                              "recall": r_m.attention_recall(a, sel, act)})
    t = rng.standard_normal((3, 5))
    r_tf.save_tensor(os.path.join(HERE, "omnt_ref.bin"), t)
    out["omnt_matrix"] = t.tolist()
    with open(os.path.join(HERE, "metrics_golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("written")


if __name__ == "__main__":
    main()
