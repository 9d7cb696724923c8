"""K4 kernel variants (the OMNI_VARIANTS build, libomnisparse_variants.so,
selected once per process by environment variables) against the oracle: the single-CTA ping-pong kernel at several MUFU / FMA-pipe
exp2 splits, the CTA-pair (cta_group::2) kernel, the row-per-thread kernel
the CTA-pair ping-pong kernel and the double-buffered-S kernel. Each variant runs in its
own subprocess on a GQA workload with ragged N (partial tiles, staircase)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, ".")
from oracle import attention as oatt
from oracle import pipeline as opipe
from oracle.workload import Spec, generate, round_bf16
from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device
Q, K, V = generate(Spec(heads=8, heads_kv=2, head_dim=128, n_vision=4999, n_text=77, seed=3))
Q, K, V = round_bf16(Q), round_bf16(K), round_bf16(V)
t = lambda x: torch.tensor(x, dtype=torch.bfloat16, device="cuda")
res = sparse_prefill_device(t(Q), t(K), t(V), 4999, SparsityConfig())
torch.cuda.synchronize()
ref = opipe.select(Q, K, 4999, 0, 0.08, 0.82, 256)
out = res.outputs.float().cpu().numpy()
lse = res.lse.cpu().numpy()
err = 0.0
for h in (0, 3, 4, 7):
    g = h // 4
    exp = oatt.sparse_head_attention(Q[h], K[g], V[g], ref.selected[g], ref.active[h], 0)
    err = max(err, float(np.max(np.abs(out[h] - exp) / (0.02 + 0.02 * np.abs(exp)))))
    act = np.flatnonzero(ref.active[h])
    el = oatt.sparse_head_lse(Q[h], K[g], ref.selected[g], ref.active[h])
    fin = np.isfinite(el[act])
    err = max(err, float(np.max(np.abs(lse[h][act][fin] - el[act][fin]))) / 0.02)
from paper_2511_12201_b200 import ops
status = int(ops.last_fwd_status[0])
print(json.dumps({"scaled_err": err, "nan": bool(np.isnan(out).any()), "fallback": status}))
"""


JUMP = r"""
# one late key aligned with its group's queries and with a huge norm: the
# logits of every later row jump far beyond the running max (> 2^64 in exp2
# units) -> the fast kernel must hand over to the safe re-run, and the result
# must still match the oracle
for _g in range(K.shape[0]):
    _u = Q[4 * _g:4 * _g + 4].mean(axis=(0, 1))
    K[_g, 1500, :] = 2000.0 * _u / np.linalg.norm(_u)
"""


RAMP = r"""
# keys drift along the group's mean query direction: the logits of a row rise
# by ~5 (exp2 units) per 128-key tile across the sequence, so the running max
# keeps growing past the 2^8 lazy-rescale threshold (many deferred rescales
# in the fast path) while no single tile jumps by 2^64 (no fallback)
for _g in range(K.shape[0]):
    _u = Q[4 * _g:4 * _g + 4].reshape(-1, Q.shape[2]).mean(axis=0)
    _u = _u / np.linalg.norm(_u)
    _qu = float(np.mean(np.abs(Q[4 * _g:4 * _g + 4].reshape(-1, Q.shape[2]) @ _u)))
    _alpha = 200.0 * np.sqrt(128.0) / (1.4426950408889634 * _qu)
    K[_g] += (_alpha * np.arange(K.shape[1]) / K.shape[1])[:, None] * _u[None, :]
"""


@pytest.mark.gpu
@pytest.mark.parametrize("impl,poly,fast,jump", [("single", "0", "1", False), ("single", "4", "1", False),
                                                 ("single", "8", "1", False), ("single", "4", "0", False),
                                                 ("single", "4", "1", True), ("single", "4", "0", True),
                                                 ("single", "6", "1", "ramp"), ("single", "6", "0", "ramp"),
                                                 ("pair", "0", "1", False), ("pair", "4", "1", False),
                                                 ("rpt", "6", "1", False), ("rpt", "6", "1", True),
                                                 ("rpt", "6", "1", "ramp"),
                                                 ("pp", "6", "1", False), ("pp", "6", "1", True),
                                                 ("pp", "6", "1", "ramp"), ("pp", "6", "0", False),
                                                 ("pp", "6", "0", "ramp"),
                                                 ("db", "6", "1", False), ("db", "6", "1", True),
                                                 ("db", "6", "1", "ramp"), ("db", "6", "0", False),
                                                 ("db", "6", "0", "ramp"), ("db", "0", "1", False),
                                                 ("sp", "6", "1", False), ("sp", "6", "1", True),
                                                 ("sp", "6", "1", "ramp"), ("sp", "6", "0", False),
                                                 ("sp", "6", "0", "ramp"), ("sp", "6", "0", True)])
def test_forward_variant_matches_oracle(impl, poly, fast, jump):
    env = dict(os.environ, OMNI_FWD_IMPL=impl, OMNI_FWD_POLY=poly, OMNI_FWD_FAST=fast,
               OMNI_LIBRARY=os.environ.get("OMNI_VARIANTS_LIBRARY",
                                           os.path.join(ROOT, "paper_2511_12201_b200", "lib", "libomnisparse_variants.so")))
    snippet = RAMP if jump == "ramp" else JUMP if jump else ""
    code = CODE.replace("Q, K, V = round_bf16(Q), round_bf16(K), round_bf16(V)",
                        snippet + "Q, K, V = round_bf16(Q), round_bf16(K), round_bf16(V)")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert not r["nan"]
    assert r["scaled_err"] <= 1.0, r  # |err| <= 0.02 + 0.02 |ref| (bf16 P, fp32 accumulation)
    if impl in ("single", "rpt", "pp", "db", "sp") and fast == "1":
        # the fast kernel hands over to the safe re-run exactly when a logit jump exceeds 2^64
        assert r["fallback"] == (1 if jump is True else 0), r
