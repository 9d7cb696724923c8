"""Command-line runner (reference SPEC.md:560-586, the ``run`` operation):
synthetic workload -> GPU pipeline -> MetricsReport JSON (schema v1).

    python -m paper_2511_12201_b200.cli --mode probe --tau 0.08 --p 0.82 \
        --heads 28 --kv-heads 4 --dim 128 --nv 16320 --nt 64 --seed 7 --out r.json

Modes: ``probe`` (block-probe scores, the hot path), ``sparse`` (exact score
source), ``full`` (sparsity disabled: tau = 0, p = 1), ``sweep`` (one report
per tau x p pair, ``--tau`` / ``--p`` comma lists) and ``decode`` (slim cache
+ ``--steps`` decode steps; fetch accounting in the report). Unknown flags are
rejected; every run is reproducible from (flags, seed). ``--dump-tensors DIR``
writes the per-head outputs as OMNT files; ``--import DIR`` reads Q/K/V from
OMNT files ``q{h}.omnt``, ``k{g}.omnt``, ``v{g}.omnt`` instead of generating.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

from . import decode as gdec
from . import metrics as gm
from . import ops, tensorfile
from .pipeline import SparsityConfig, select_device, sparse_prefill_device
from .synthetic import decode_queries_device, generate_device, unit_vision_mean


def _floats(s: str) -> list:
    return [float(x) for x in s.split(",") if x]


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="omnisparse-b200", allow_abbrev=False)
    ap.add_argument("--mode", choices=["full", "sparse", "probe", "decode", "sweep"], required=True)
    ap.add_argument("--tau", default="0.08")
    ap.add_argument("--p", default="0.82")
    ap.add_argument("--block-size", type=int, default=256)
    ap.add_argument("--granularity", choices=["token", "block"], default="token")
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--kv-heads", type=int, default=0, help="0: MHA (kv-heads = heads)")
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--nv", type=int, default=1984)
    ap.add_argument("--nt", type=int, default=64)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--lazy-fraction", type=float, default=0.5)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="-")
    ap.add_argument("--dump-tensors", default=None)
    ap.add_argument("--import", dest="import_dir", default=None)
    return ap


def _workload(a):
    hkv = a.kv_heads or a.heads
    if a.import_dir:
        ld = lambda name: torch.from_numpy(tensorfile.load_tensor(os.path.join(a.import_dir, name)))
        Q = torch.stack([ld(f"q{h}.omnt") for h in range(a.heads)])
        K = torch.stack([ld(f"k{g}.omnt") for g in range(hkv)])
        V = torch.stack([ld(f"v{g}.omnt") for g in range(hkv)])
        return (x.to("cuda", torch.bfloat16).contiguous() for x in (Q, K, V))
    return generate_device(a.heads, hkv, a.dim, a.nv, a.nt, seed=a.seed, lazy_fraction=a.lazy_fraction)


def _prefill_report(a, Q, K, V, tau, p, source):
    cfg = SparsityConfig(tau=tau, p=p, block_size=a.block_size, granularity=a.granularity)
    res = sparse_prefill_device(Q, K, V, a.nv, cfg, score_source=source)
    rep = gm.prefill_report(res, Q, K, V, a.nv, cfg)
    rep.mode = a.mode
    rep.config["score_source"] = source
    rep.workload["seed"] = a.seed
    return res, rep


def run(argv=None) -> int:
    a = _parser().parse_args(argv)
    taus, ps = _floats(a.tau), _floats(a.p)
    if a.mode != "sweep" and (len(taus) != 1 or len(ps) != 1):
        raise SystemExit("only --mode sweep takes lists for --tau / --p")
    ops.device_check()
    Q, K, V = _workload(a)
    reports = []
    res = None
    if a.mode in ("probe", "sparse", "full"):
        tau, p = (0.0, 1.0) if a.mode == "full" else (taus[0], ps[0])
        res, rep = _prefill_report(a, Q, K, V, tau, p, "exact" if a.mode == "sparse" else "probe")
        reports.append(rep)
    elif a.mode == "sweep":
        for tau in taus:
            for p in ps:
                reports.append(_prefill_report(a, Q, K, V, tau, p, "probe")[1])
    else:  # decode
        cfg = SparsityConfig(tau=taus[0], p=ps[0], block_size=a.block_size)
        k_lazy, k_act, _, _, _, _, _, _, mass, sel = select_device(Q, K, a.nv, cfg)
        b = min(int(sel.info[0]), a.nv)
        hkv = K.shape[0]
        vsel = ops.select(mass, hkv, a.nv + a.nt, cfg.block_size, cfg.p, "token", vision_limit=a.nv,
                          budget_override=b)
        cache = gdec.build_cache_device(K, V, vsel.selected, b, a.nv, a.nt, k_lazy, k_act, a.heads,
                                 answer_capacity=a.steps + 1)
        means = [unit_vision_mean(K, a.nv)]
        active_steps = total_steps = 0
        gen = torch.Generator(device="cuda")
        gen.manual_seed(a.seed)
        for t in range(a.steps):
            q = decode_queries_device(a.heads, hkv, means, [a.seed], a.lazy_fraction, t)
            _, flags = gdec.decode_attention_batch(q, cache, cfg.tau)
            fetched = flags.view(1, hkv, -1).any(dim=2)
            active_steps += int(fetched.sum())
            total_steps += hkv
            gdec.append_answer_batch(cache, torch.randn(1, hkv, a.dim, generator=gen, device="cuda"),
                               torch.randn(1, hkv, a.dim, generator=gen, device="cuda"))
        kv = gm.kv_reduction(a.nv, b, a.dim, active_steps, total_steps)
        rep = gm.MetricsReport(
            mode="decode", config={"tau": cfg.tau, "p": cfg.p, "block_size": cfg.block_size},
            workload={"heads": a.heads, "kv_heads": hkv, "head_dim": a.dim, "n_vision": a.nv, "n_text": a.nt,
                      "seed": a.seed, "steps": a.steps},
            flops_full=0, flops_sparse=0, flops_probe_overhead=0, flops_reduction=0.0, exponentials_full=0,
            exponentials_sparse=0, recall_per_head=[], recall_min=1.0, recall_flattest=1.0,
            flattest_retained_mass=float(sel.stats[hkv]), flattest_total_mass=float(sel.stats[hkv + 1]),
            budget=b, flattest_head=int(sel.info[1]), lazy_query_fraction=0.0, sparsity_gap=None,
            kv_resident_reduction=kv.resident_reduction, kv_fetch_reduction=kv.fetch_reduction,
            lazy_head_fraction_decode=1.0 - active_steps / total_steps if total_steps else 0.0,
            decode={"vision_tokens_fetched": cache.fetch.vision_tokens, "vision_bytes": cache.fetch.vision_bytes,
                    "text_answer_bytes": cache.fetch.text_answer_bytes,
                    "predicted_vision_tokens": kv.predicted_vision_tokens})
        reports.append(rep)
    if a.dump_tensors and res is not None:
        os.makedirs(a.dump_tensors, exist_ok=True)
        out = res.outputs.float().cpu()
        for h in range(out.shape[0]):
            tensorfile.save_tensor(os.path.join(a.dump_tensors, f"out{h}.omnt"), out[h])
    text = reports[0].to_json() if len(reports) == 1 else json.dumps([r.to_dict() for r in reports], sort_keys=True,
                                                                       indent=2) + "\n"
    if a.out == "-":
        sys.stdout.write(text)
    else:
        tmp = a.out + ".tmp"
        with open(tmp, "w") as f:
            f.write(text)
        os.replace(tmp, a.out)
    return 0


if __name__ == "__main__":
    raise SystemExit(run())
