#!/usr/bin/env python
"""Benchmark of the OmniSparse sparse-attention hot path on B200.

Headline (BASELINE.json ``metric``): prefill sparse-attention throughput of a
Qwen2-7B-shaped attention layer (28 Q / 4 KV heads, d=128) at 64K tokens
(65472 vision + 64 text, config C3 at 1 GPU), plus the speed-up over the
fastest dense causal bf16 flash-attention on the same GPU, and batch-32 decode
tok/s and KV bytes per step over the slimmed cache (C5 shape, 1 GPU).

One "step" = one full sparse prefill of the layer (K1 probe keys, K2 query
scoring, row compaction, K3 probe mass + selection, K6 KV regroup, K4
tcgen05 sparse attention) on HBM-resident synthetic inputs (Q alone is
470 MB > 126 MB L2, so no flush is needed between steps).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N (head-sharded, one
all_gather of block masses per step; strong scaling).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prefill sparse-attn latency @64K tok vs dense FA (×), decode tok/s & KV bytes"
HQ, HKV, D = 28, 4, 128
N_TEXT = 64


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--seq", type=int, default=65536)
    ap.add_argument("--lazy", type=float, default=0.5)
    ap.add_argument("--tau", type=float, default=0.08)
    ap.add_argument("--p", type=float, default=0.82)
    ap.add_argument("--decode-batch", type=int, default=32)
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--no-knobs", action="store_true", help="skip the second-operating-point sweep")
    ap.add_argument("--flashinfer", action="store_true", help="also time flashinfer's dense FMHA (JIT)")
    return ap.parse_args()


def log(msg: str) -> None:
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------ timing
def time_cuda(fn, steps: int, warmup: int, stream=None):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(steps):
        fn()
    e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


def time_graph(fn, calls: int, reps: int) -> float:
    """Device time per call of fn: `calls` calls captured in one CUDA graph
    (the caching allocator serves the captured allocations from the graph's
    pool), replayed `reps` times; best replay / calls, in ms."""
    import torch

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            for _ in range(calls):
                fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / calls)
    del g
    return best


def count_launches(fn) -> int:
    """Kernels one call of fn launches (torch.profiler / CUPTI)."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    names = [ev.name for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA]
    ours = [n for n in names if "omni" in n]
    return len(ours), len(names), sorted(set(ours))


def work_flops(res, n_kv_heads: int, d: int = D) -> float:
    """Algorithmic forward FLOPs = 4 d sum_h sum_{r in A_h} |{j in S_g : j <= r}|
    (SURVEY §8d), counted exactly from the produced index sets."""
    import torch

    hq = res.rows.shape[0]
    rep = hq // n_kv_heads
    counts = res.counts.cpu().tolist()
    b = res.selection.info[4:].cpu().tolist()
    total = 0
    for h in range(hq):
        g = h // rep
        sel = res.selection.selected[g, : b[g]].contiguous()
        rows = res.rows[h, : counts[h]].contiguous()
        total += int(torch.searchsorted(sel, rows, right=True).sum())
    return 4.0 * d * total


# ------------------------------------------------------------------ dense FA baselines
def dense_baselines(Q, K, V, steps, warmup, use_flashinfer=False):
    import torch

    hq, n, d = Q.shape
    out = {}
    q4, k4, v4 = Q.unsqueeze(0), K.unsqueeze(0), V.unsqueeze(0)
    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel

        def cudnn():
            with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
                return torch.nn.functional.scaled_dot_product_attention(q4, k4, v4, is_causal=True, enable_gqa=True)
        cudnn()
        out["cudnn_sdpa_ms"] = time_cuda(cudnn, steps, warmup)
    except Exception as e:  # noqa: BLE001
        out["cudnn_sdpa_error"] = str(e)[:160]
    try:
        from flash_attn import flash_attn_func

        qf, kf, vf = (x.transpose(0, 1).unsqueeze(0).contiguous() for x in (Q, K, V))
        fa = lambda: flash_attn_func(qf, kf, vf, causal=True)
        fa()
        out["flash_attn2_ms"] = time_cuda(fa, steps, warmup)
        del qf, kf, vf
    except Exception as e:  # noqa: BLE001
        out["flash_attn2_error"] = str(e)[:160]
    if use_flashinfer:
        try:
            import flashinfer

            qf, kf, vf = (x.transpose(0, 1).contiguous() for x in (Q, K, V))
            fi = lambda: flashinfer.single_prefill_with_kv_cache(qf, kf, vf, causal=True)
            fi()
            out["flashinfer_fa2_ms"] = time_cuda(fi, steps, warmup)
            # sm100 CUTLASS FMHA (JIT-compiled on first use)
            from flashinfer.prefill import fmha_varlen

            seg = torch.tensor([0, n], dtype=torch.int32, device=Q.device)
            fc = lambda: fmha_varlen(qf, kf, vf, seg, seg, max_qo_len=n, causal=True)
            fc()
            out["flashinfer_cutlass_fmha_ms"] = time_cuda(fc, steps, warmup)
            del qf, kf, vf
        except Exception as e:  # noqa: BLE001
            out["flashinfer_error"] = str(e)[:300]
    times = {k: v for k, v in out.items() if k.endswith("_ms")}
    if times:
        best = min(times, key=times.get)
        out["fastest"] = best[:-3]
        out["fastest_ms"] = times[best]
    out["dense_causal_flops"] = 4.0 * d * hq * n * (n + 1) / 2
    return out


# ------------------------------------------------------------------ CPU reference sample
def cpu_reference_sample(Q, K, V, n_vision, tau, p, head=13, rows_sample=1024, seed=0):
    """The oracle (float64 NumPy restatement of the reference path) timed on a
    bounded sample of the SAME workload: the full selection pass over all 28
    heads, then sparse_head_attention for `rows_sample` uniformly drawn active
    rows of one head; the attention time is extrapolated to every active row of
    every head. Returns (tok/s, seconds per full step, sample description)."""
    import numpy as np

    from oracle import attention as oatt
    from oracle import pipeline as opipe

    to64 = lambda t: t.float().cpu().numpy().astype(np.float64)
    Qh, Kh, Vh = to64(Q), to64(K), to64(V)
    n = Qh.shape[1]
    t0 = time.perf_counter()
    ref = opipe.select(Qh, Kh, n_vision, 0, tau, p, 256)
    t_sel = time.perf_counter() - t0
    rep = Qh.shape[0] // Kh.shape[0]
    rows = np.flatnonzero(ref.active[head])
    samp = np.sort(np.random.default_rng(seed).choice(rows, min(rows_sample, rows.size), replace=False))
    t0 = time.perf_counter()
    oatt.sparse_head_attention(Qh[head], Kh[head // rep], Vh[head // rep], ref.selected[head // rep],
                               ref.active[head], 0, rows_subset=samp)
    t_att = time.perf_counter() - t0
    total_rows = int(ref.active.sum())
    t_step = t_sel + t_att * total_rows / samp.size
    desc = (f"oracle (NumPy f64 restatement of slimattn) on the same {n}-token workload: full selection over "
            f"{Qh.shape[0]} heads ({t_sel:.2f} s) + sparse_head_attention of {samp.size} random active rows of head "
            f"{head} ({t_att:.2f} s), extrapolated to all {total_rows} active rows")
    return n / t_step, t_step, desc, ref


# ------------------------------------------------------------------ decode
def decode_section(args, steps, warmup, hbm_peak, tau=None, p=None, dense=True, world=1, rank=0):
    """C5: batch-32 decode over 64K-token slim caches. At N > 1 the batch is
    sequence-sharded (parallel.sequence_shard: rank r decodes its own
    sequences from its own caches, no collective); the step time is the max
    over ranks and tok/s counts the whole batch."""
    import torch

    from paper_2511_12201_b200 import decode as gdec
    from paper_2511_12201_b200.parallel import sequence_shard
    from paper_2511_12201_b200.pipeline import SparsityConfig
    from paper_2511_12201_b200.synthetic import decode_queries_device, generate_device, unit_vision_mean

    n = args.seq
    nv = n - N_TEXT
    B_all = args.decode_batch
    seqs = list(sequence_shard(B_all, world, rank))
    B = len(seqs)
    tau = args.tau if tau is None else tau
    p = args.p if p is None else p
    cfg = SparsityConfig(tau=tau, p=p)
    caches, k_means = [], []
    # one page-pool reservation for the whole batch (pages of 64 rows: ~0.47 N
    # vision rows per group at the defaults, text and answer pages)
    gdec.default_pool(torch.device("cuda")).reserve(B * HKV * (-(-int(0.6 * nv) // 64) + 4))
    for s in seqs:
        Q, K, V = generate_device(HQ, HKV, D, nv, N_TEXT, seed=1000 + s, lazy_fraction=args.lazy)
        caches.append(gdec.cache_from_prompt(Q, K, V, nv, N_TEXT, cfg, answer_capacity=warmup + steps + 8))
        k_means.append(unit_vision_mean(K, nv))
        del Q, K, V
    torch.cuda.empty_cache()
    cache = gdec.stack_caches(caches)
    del caches
    torch.cuda.empty_cache()
    n_steps = warmup + steps
    qs = [decode_queries_device(HQ, HKV, k_means, seqs, args.lazy, t) for t in range(n_steps)]
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7 + rank)
    kv_new = [(torch.randn(B, HKV, D, generator=gen, device="cuda").bfloat16(),
               torch.randn(B, HKV, D, generator=gen, device="cuda").bfloat16()) for _ in range(n_steps)]
    flags_log = []

    def step(t):
        out, fl = gdec.decode_attention_batch(qs[t], cache, tau, log=False)
        flags_log.append(fl)
        gdec.append_answer_batch(cache, *kv_new[t])

    for t in range(warmup):
        step(t)
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flags_log.clear()
    e0.record()
    for t in range(warmup, n_steps):
        step(t)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    # bytes each timed step read (vision of fetched groups + text + answer), bf16
    n_ans0 = cache.n_answer - steps
    tot_vis, tot_ta = 0, 0
    for i, fl in enumerate(flags_log):
        vt, vb, _ = gdec.step_bytes(cache, fl)
        tot_vis += vb
        tot_ta += B * HKV * (N_TEXT + n_ans0 + i) * 2 * D * 2
    slim_bytes = (tot_vis + tot_ta) / steps
    full_bytes = B * HKV * (n + n_ans0 + steps / 2) * 2 * D * 2
    q_bytes = B * HQ * D * (2 + 4)
    fetched = float(torch.stack([f.view(B, HKV, -1).any(dim=2) for f in flags_log]).float().mean())
    # The reference's own accounting (FetchLog, decode.py:180-190, and
    # kv_reduction, metrics.py:94-120): every Q head meters its own fetch —
    # b vision rows when active, text + answer always — against its own full
    # cache. Physically (above) a GQA group's vision rows are read once when
    # ANY of its 7 Q heads is active, so the two differ at rep > 1.
    act_q = torch.stack([f.view(B, HQ) for f in flags_log]).float().cpu()  # [steps, B, HQ]
    bud = torch.tensor([float(b) for b in cache.budgets])
    row = 2 * D * 2
    ref_fetched = ref_full = 0.0
    for i in range(act_q.shape[0]):
        ta = N_TEXT + n_ans0 + i
        ref_fetched += float((act_q[i] * bud[:, None]).sum() + B * HQ * ta) * row
        ref_full += B * HQ * (nv + ta) * row
    ref_vis_frac = float((act_q.sum(dim=(0, 2)) * bud).sum() / (act_q.shape[0] * HQ * nv * B))
    budgets = sum(cache.budgets)
    if world > 1:  # max time over ranks, bytes summed over ranks
        import torch.distributed as dist

        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        v = torch.tensor([slim_bytes, full_bytes, q_bytes, fetched * B, budgets], device="cuda", dtype=torch.float64)
        dist.all_reduce(v, op=dist.ReduceOp.SUM)
        ms = float(t)
        slim_bytes, full_bytes, q_bytes, fetched, budgets = (float(x) for x in v)
        fetched /= B_all
    res = {
        "batch": B_all, "context": n, "ms_per_step": ms, "tok_s": B_all / (ms / 1e3),
        "kv_bytes_per_step": slim_bytes, "full_cache_bytes_per_step": full_bytes,
        "kv_bytes_reduction": full_bytes / slim_bytes,
        "budgets_mean": budgets / B_all,
        "fetched_group_frac": fetched,
        "reference_accounting": {
            "kv_bytes_reduction_per_q_head": ref_full / ref_fetched if ref_fetched else None,
            "vision_fetch_reduction": 1.0 - ref_vis_frac,
            "active_q_head_frac": float(act_q.mean()),
            "note": "the reference's FetchLog / kv_reduction model (each Q head meters b vision rows when active, "
                    "text+answer always); kv_bytes_reduction above is the physical GQA read (a group's vision rows "
                    "once if any of its Q heads is active)",
        },
        "roofline": {"bound": "hbm", "achieved": (slim_bytes + q_bytes) / (ms / 1e3) / 1e9 / world,
                     "peak": hbm_peak, "unit": "GB/s per GPU",
                     "frac": (slim_bytes + q_bytes) / (ms / 1e3) / 1e9 / world / hbm_peak},
        "knobs": {"tau": tau, "p": p, "lazy_fraction": args.lazy},
        "sharding": f"sequence-sharded x{world} ({B} sequences on rank {rank})" if world > 1 else "single GPU",
    }
    if not dense or world > 1:
        cache.release()
        return res
    # dense full-cache decode baseline (flash-attn kv-cache kernel), same batch/context
    try:
        from flash_attn import flash_attn_with_kvcache

        cache.release()
        del cache
        torch.cuda.empty_cache()
        kc = torch.randn(B, n, HKV, D, device="cuda", dtype=torch.bfloat16)
        vc = torch.randn(B, n, HKV, D, device="cuda", dtype=torch.bfloat16)
        q1 = torch.randn(B, 1, HQ, D, device="cuda", dtype=torch.bfloat16)
        lens = torch.full((B,), n, dtype=torch.int32, device="cuda")
        fn = lambda: flash_attn_with_kvcache(q1, kc, vc, cache_seqlens=lens)
        dms = time_cuda(fn, steps, warmup)
        res["dense_decode"] = {"kernel": "flash_attn_with_kvcache (full cache)", "ms_per_step": dms,
                               "tok_s": B / (dms / 1e3)}
        res["speedup_vs_dense_decode"] = dms / ms
        del kc, vc
    except Exception as e:  # noqa: BLE001
        res["dense_decode_error"] = str(e)[:160]
    return res


# ------------------------------------------------------------------ training (C4)
def train_section(args, steps, warmup, tc_peak):
    """Config C4: sparse attention forward + backward at 32K tokens (28/4
    heads), selection under no_grad, vs cuDNN SDPA forward + backward."""
    import torch

    from paper_2511_12201_b200.autograd import SparseAttentionFn, plan_from_selection
    from paper_2511_12201_b200.pipeline import SparsityConfig, select_device
    from paper_2511_12201_b200.synthetic import generate_device

    n = 32768
    nv = n - N_TEXT
    cfg = SparsityConfig(tau=args.tau, p=args.p)
    Q, K, V = generate_device(HQ, HKV, D, nv, N_TEXT, seed=3, lazy_fraction=args.lazy)
    Q.requires_grad_(True)
    K.requires_grad_(True)
    V.requires_grad_(True)
    dO = torch.randn_like(Q)

    def sparse_step():  # = autograd.sparse_attention (the public API), keeping the plan for the FLOP count
        out = torch.empty(Q.shape, device=Q.device, dtype=torch.bfloat16)
        with torch.no_grad():
            _, _, _, _, _, _, rows, counts, _, sel = select_device(Q.detach(), K.detach(), nv, cfg, O_zero=out)
        O = SparseAttentionFn.apply(Q, K, V, plan_from_selection(rows, counts, sel, 0, out))
        O.backward(dO)
        return rows, counts, sel

    rows, counts, sel = sparse_step()
    ms = time_cuda(sparse_step, steps, warmup)
    res = {"workload": f"sparse attention fwd+bwd, {HQ}/{HKV} heads, d={D}, {n} tokens (C4)", "ms_per_step": ms,
           "tok_s": n / (ms / 1e3),
           "step": "selection (no_grad) + forward + backward, gradients accumulated into the leaves' .grad in "
                   "both arms"}
    # K5 roofline: backward FLOPs = 2.5 x the forward's algorithmic FLOPs
    # (dq: 3 GEMMs, dkv: 4 GEMMs per visible tile pair vs the forward's 2),
    # counted from this step's index sets; K5 = bwd_prep + dq + dkv, timed
    # alone on the current stream with CUDA events
    try:
        from paper_2511_12201_b200 import ops

        class _R:  # the fields work_flops reads
            pass

        r_ = _R()
        r_.rows, r_.counts, r_.selection = rows, counts, sel
        fwd_flops = work_flops(r_, HKV)
        cap = ops.round_up(n, ops.TILE)
        Qb, Kb, Vb = (x.detach() for x in (Q, K, V))
        K_sel = ops.gather_rows(Kb, sel.selected, sel.counts, cap, ops.TILE)
        V_sel = ops.gather_rows(Vb, sel.selected, sel.counts, cap, ops.TILE)
        O = torch.zeros_like(Qb)
        lse = torch.empty(HQ, n, device=Q.device, dtype=torch.float32)
        ops.sparse_attn_fwd(Qb, K_sel, V_sel, Vb, rows, counts, sel.selected, sel.counts, 0, O, lse)
        dOb = dO.to(torch.bfloat16)
        fwd_ms = time_cuda(lambda: ops.sparse_attn_fwd(Qb, K_sel, V_sel, Vb, rows, counts, sel.selected, sel.counts, 0,
                                                       O, lse), steps, 2)
        bwd_ms = time_cuda(lambda: ops.sparse_attn_bwd(Qb, K_sel, V_sel, O, dOb, lse, rows, counts, sel.selected,
                                                       sel.counts, dq_dtype=torch.bfloat16), steps, 2)
        ach = 2.5 * fwd_flops / (bwd_ms / 1e3) / 1e12
        res["roofline"] = {"bound": "tensor", "kernel": "K5 backward (bwd_prep + dq_kernel + dkv2_kernel)",
                           "achieved": ach, "peak": tc_peak, "unit": "TFLOP/s", "frac": ach / tc_peak,
                           "algorithmic_flops_per_launch": 2.5 * fwd_flops, "launch_ms": bwd_ms,
                           "traffic": None, "ncu": "profiles/r02_ncu_k5_details.txt",
                           # the kernels execute 7 GEMMs per visible tile pair (dq recomputes S and dP; the
                           # fifth 128x128 fp32 accumulator a fused dq+dkv needs does not fit in TMEM beside
                           # S^T, dP^T, dK, dV): executed FLOPs = 3.5 x forward, against the same peak
                           "executed_flops_per_launch": 3.5 * fwd_flops,
                           "frac_executed": 3.5 * fwd_flops / (bwd_ms / 1e3) / 1e12 / tc_peak}
        res["forward_roofline"] = {"achieved": fwd_flops / (fwd_ms / 1e3) / 1e12, "unit": "TFLOP/s",
                                   "frac": fwd_flops / (fwd_ms / 1e3) / 1e12 / tc_peak, "launch_ms": fwd_ms}
        del K_sel, V_sel, O, lse
    except Exception as e:  # noqa: BLE001
        res["roofline"] = {"error": str(e)[:200]}
    try:
        from torch.nn.attention import SDPBackend, sdpa_kernel

        q4, k4, v4 = (x.detach().unsqueeze(0).requires_grad_(True) for x in (Q, K, V))
        g4 = dO.unsqueeze(0)

        def dense_step():
            with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
                o = torch.nn.functional.scaled_dot_product_attention(q4, k4, v4, is_causal=True, enable_gqa=True)
            o.backward(g4)

        dense_step()
        dms = time_cuda(dense_step, steps, warmup)
        res["dense_cudnn_fwd_bwd_ms"] = dms
        res["speedup_vs_dense"] = dms / ms
    except Exception as e:  # noqa: BLE001
        res["dense_error"] = str(e)[:160]
    return res


# ------------------------------------------------------------------ main arms
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2511_12201_b200 import ops
    from paper_2511_12201_b200.parallel import shard_plan, sparse_prefill_sharded
    from paper_2511_12201_b200.pipeline import SparsityConfig, select_device, sparse_prefill_device
    from paper_2511_12201_b200.synthetic import generate_device

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # OMNI_BENCH_SHARED_GPU=1 (testing the N > 1 code path on a one-GPU box):
    # every rank on device 0, gloo instead of NCCL
    shared = os.environ.get("OMNI_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ops.device_check()
    hbm_peak, tc_peak, tc_sus, peak_src = peaks()
    n, nv = args.seq, args.seq - N_TEXT
    cfg = SparsityConfig(tau=args.tau, p=args.p)
    Q, K, V = generate_device(HQ, HKV, D, nv, N_TEXT, seed=0, lazy_fraction=args.lazy)
    plan = shard_plan(HQ, HKV, world, rank)
    if world > 1:
        Ql = Q[plan.q_start:plan.q_stop].contiguous()
        Kl = K[plan.g_start:plan.g_stop].contiguous()
        Vl = V[plan.g_start:plan.g_stop].contiguous()
        O = torch.empty_like(Ql)
        step = lambda: sparse_prefill_sharded(Ql, Kl, Vl, plan, nv, world, cfg, out=O)
    else:
        O = torch.empty_like(Q)
        step = lambda: sparse_prefill_device(Q, K, V, nv, cfg, out=O)

    res = step()
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            res = step()
        e1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
    value = n / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: reference generator construction (workload.py:88-129, GQA rule B) drawn with torch CUDA RNG",
            "config": {"workload": f"Qwen2-7B-shaped attention layer sparse prefill, {HQ} Q / {HKV} KV heads, d={D}, "
                                   f"{n} tokens ({nv} vision + {N_TEXT} text)",
                       "knobs": {"tau": args.tau, "p": args.p, "block_size": 256, "lazy_fraction": args.lazy,
                                 "granularity": "token", "preserve_first_head": True},
                       "parallelism": f"head-sharded x{world}" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (Q alone 470 MB at 64K); no flush"}}
    line["clocks"] = clk.summary()
    b = int(res.selection.info[0])
    line["selection"] = {"budget": b, "b_over_n": b / n, "flattest_group": int(res.selection.info[1]),
                         "active_frac": float(res.active.float().mean())}
    if world > 1:
        multi_rank_sections(args, line, step, res, plan, Ql, Kl, Vl, O, nv, cfg, world, tc_peak, peak_src)
        del res, Q, K, V, Ql, Kl, Vl, O
        torch.cuda.empty_cache()
        multi_rank_decode_train(args, line, world, rank, hbm_peak, plan)
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    flops = work_flops(res, HKV) if world == 1 else None
    if world == 1:
        line["selection"]["work_ratio_vs_dense_causal"] = flops / (4.0 * D * HQ * n * (n + 1) / 2)
        log("timed region done; per-kernel breakdown")
        # ----- per-kernel breakdown and the K4 roofline (dominant kernel, own stream events)
        rows, counts, sel = res.rows, res.counts, res.selection
        fa = lambda: ops.sparse_attn_fwd(Q, res.K_sel, res.V_sel, V, rows, counts, sel.selected, sel.counts, 0, O,
                                         res.lse)
        fa_ms = time_cuda(fa, args.steps, 2)
        sel_ms = time_cuda(lambda: select_device(Q, K, nv, cfg, O_zero=O), args.steps, 2)
        cap = ops.round_up(n, 128)
        gat_ms = time_cuda(lambda: (ops.gather_rows(K, sel.selected, sel.counts, cap, 128, out=res.K_sel),
                                    ops.gather_rows(V, sel.selected, sel.counts, cap, 128, out=res.V_sel)),
                           args.steps, 2)
        achieved = flops / (fa_ms / 1e3) / 1e12
        traffic = None
        try:  # dram bytes per K4 launch from the committed ncu capture of the same workload
            with open(os.path.join(ROOT, "profiles", "r02_k4_traffic.json")) as f:
                traffic = json.load(f)["dram_bytes_per_launch"]
        except Exception:  # noqa: BLE001
            pass
        line["roofline"] = {"bound": "tensor", "kernel": "omni sparse_fwd_kernel (K4)", "achieved": achieved,
                            "peak": tc_peak, "unit": "TFLOP/s", "frac": achieved / tc_peak, "traffic": traffic,
                            "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch "
                                            "(profiles/r02_k4_traffic.json); K4 is tensor-bound, its DRAM traffic "
                                            "(Q rows, K/V tiles re-read past L2, O rows) is ~1.16 GB per ~9 ms",
                            "peak_source": f"{peak_src} bf16 burst (MEASURED_PEAKS.json)",
                            "peak_sustained": tc_sus, "frac_of_sustained": achieved / tc_sus,
                            "algorithmic_flops_per_launch": flops, "launch_ms": fa_ms}
        # parity: this run's decision margins + the committed oracle report
        st = res.selection.stats.cpu().tolist()
        kurt = sorted(st[:HKV])
        par = {"this_run": {"budget_margin_rel_to_total": st[HKV + 2], "budget_replayed": bool(st[HKV + 3]),
                            "kurtosis_gap_rel": (kurt[1] - kurt[0]) / abs(kurt[0])}}
        try:
            with open(os.path.join(ROOT, "profiles", "r02_parity.json")) as f:
                rep = json.load(f)
            par["oracle_report"] = {
                "source": "profiles/r02_parity.json (tests/test_gpu_parity_report.py, same kernels)",
                "prefill_c1_outputs_max_abs": max(v["outputs"]["max_abs"] for v in rep["c1_fp32_validation"].values()),
                "prefill_64k_outputs_max_abs": rep["c3_64k"]["outputs_sampled_rows"]["max_abs"],
                "prefill_64k_outputs_max_rel": rep["c3_64k"]["outputs_sampled_rows"]["max_rel"],
                "grad_max_rel": {k: rep["backward_gqa_8_2_n2048"][k]["max_rel"] for k in ("dQ", "dK", "dV")},
                "decode_outputs_max_abs": rep["decode_reference_trace"]["outputs"]["max_abs"],
                "selections": "bit-exact vs the oracle (C1-C3 sizes, tests/test_gpu_select_parity.py)"}
        except Exception:  # noqa: BLE001
            pass
        line["parity"] = par
        line["breakdown_ms"] = {"select_path_K1_K2_compact_K3": sel_ms, "gather_K6": gat_ms, "sparse_fa_K4": fa_ms,
                                "k4_share_of_step": fa_ms / ms}
        # ----- HBM-bound kernels against the measured copy bandwidth (algorithmic bytes),
        # each timed alone (the burst peak's condition): after an idle second,
        # so they do not inherit the power state of the tensor-bound step above
        try:
            hb = {}
            torch.cuda.synchronize()
            time.sleep(1.0)
            k1_ms = time_graph(lambda: ops.kv_probe(K, nv, 0, 256), 20, 5)
            k1_bytes = HKV * n * D * 2
            kl_, ka_, _ = ops.kv_probe(K, nv, 0, 256)
            k2_ms = time_graph(lambda: ops.q_score(Q, kl_, ka_, nv, args.tau, True, 256, O_zero=O), 20, 5)
            lazy_rows = int((res.active == 0).sum())
            k2_bytes = HQ * n * D * 2 + lazy_rows * D * 2 + HQ * n  # Q read, lazy O rows zeroed, flags
            bsum = int(sel.info[4:].sum())
            k6_bytes = 2 * (bsum * D * 2 + HKV * cap * D * 2)  # K and V: selected rows read, padded rows written
            for name, kms, kb in (("K1_kv_probe", k1_ms, k1_bytes), ("K2_q_score", k2_ms, k2_bytes),
                                  ("K6_gather_KV", gat_ms, k6_bytes)):
                gbs = kb / (kms / 1e3) / 1e9
                hb[name] = {"ms": kms, "bytes": kb, "achieved_GBs": gbs, "frac_of_peak": gbs / hbm_peak}
            hb["timing"] = ("K1 / K2: one CUDA graph of 20 back-to-back calls, replayed 5 times, best replay / 20 "
                            "(device time; the eager per-call host overhead of ~20 us exceeds K1 itself); "
                            "K6: the gathers inside the timed step")
            line["hbm_kernels"] = hb
        except Exception as e:  # noqa: BLE001
            line["hbm_kernels"] = {"error": str(e)[:200]}
        n_ours, n_all, names = count_launches(step)
        line["gpu_launches"] = n_ours * args.steps
        line["gpu_launches_per_step"] = {"ours": n_ours, "all": n_all, "kernels": names}
        log("dense FA baselines")
        # ----- dense FA comparators on the same tensors
        if not args.no_dense:
            dense = dense_baselines(Q, K, V, args.steps, 2, args.flashinfer)
            line["dense_fa"] = dense
            if "fastest_ms" in dense:
                line["speedup_vs_dense_fa"] = dense["fastest_ms"] / ms
                line["dense_fa_tflops"] = dense["dense_causal_flops"] / (dense["fastest_ms"] / 1e3) / 1e12
        log("knob sweep")
        # ----- second operating point (paper's tau=0.12, p=0.75) and lazier workload
        if not args.no_knobs and not args.no_dense and "fastest_ms" in line.get("dense_fa", {}):
            sweep = []
            for lz, tau, p in ((0.5, 0.12, 0.75), (0.7, 0.08, 0.82), (0.7, 0.12, 0.75)):
                Q2, K2, V2 = generate_device(HQ, HKV, D, nv, N_TEXT, seed=0, lazy_fraction=lz)
                c2 = SparsityConfig(tau=tau, p=p)
                O2 = torch.empty_like(Q2)
                st2 = lambda: sparse_prefill_device(Q2, K2, V2, nv, c2, out=O2)
                r2 = st2()
                ms2 = time_cuda(st2, args.steps, 2)
                sweep.append({"lazy_fraction": lz, "tau": tau, "p": p, "ms_per_step": ms2,
                              "speedup_vs_dense_fa": line["dense_fa"]["fastest_ms"] / ms2,
                              "budget": int(r2.selection.info[0]),
                              "work_ratio": work_flops(r2, HKV) / (4.0 * D * HQ * n * (n + 1) / 2)})
                del Q2, K2, V2, O2, r2
            line["knob_sweep"] = sweep
        log("size sweep")
        # ----- C2 (32K) and C3 upper size (128K) at the reference defaults
        if not args.no_knobs and not args.no_dense:
            sizes = []
            for n2 in (32768, 131072):
                try:
                    Q2, K2, V2 = generate_device(HQ, HKV, D, n2 - N_TEXT, N_TEXT, seed=0, lazy_fraction=args.lazy)
                    O2 = torch.empty_like(Q2)
                    st2 = lambda: sparse_prefill_device(Q2, K2, V2, n2 - N_TEXT, cfg, out=O2)
                    r2 = st2()
                    ms2 = time_cuda(st2, args.steps, 2)
                    dn = dense_baselines(Q2, K2, V2, max(3, args.steps // 2), 2)
                    sizes.append({"tokens": n2, "ms_per_step": ms2, "tok_s": n2 / (ms2 / 1e3),
                                  "dense_fastest": dn.get("fastest"), "dense_ms": dn.get("fastest_ms"),
                                  "speedup_vs_dense_fa": (dn["fastest_ms"] / ms2) if "fastest_ms" in dn else None,
                                  "budget": int(r2.selection.info[0]),
                                  "work_ratio": work_flops(r2, HKV) / (4.0 * D * HQ * n2 * (n2 + 1) / 2)})
                    del Q2, K2, V2, O2, r2
                    torch.cuda.empty_cache()
                except Exception as e:  # noqa: BLE001
                    sizes.append({"tokens": n2, "error": str(e)[:200]})
            line["size_sweep"] = sizes
        log("e2e")
        # ----- end-to-end through the public API with host buffers
        if not args.no_e2e:
            hQ, hK, hV = (x.cpu().pin_memory() for x in (Q, K, V))
            hO = torch.empty(Q.shape, dtype=torch.bfloat16).pin_memory()

            def e2e():
                Q.copy_(hQ, non_blocking=True)
                K.copy_(hK, non_blocking=True)
                V.copy_(hV, non_blocking=True)
                sparse_prefill_device(Q, K, V, nv, cfg, out=O)
                hO.copy_(O, non_blocking=True)

            serial_ms = time_cuda(e2e, max(3, args.steps // 2), 1)
            h2d = sum(x.numel() * x.element_size() for x in (hQ, hK, hV))
            # streamed serving API: each request's copies overlap other requests' kernels
            from paper_2511_12201_b200.pipeline import PrefillStreamer

            res = None
            torch.cuda.empty_cache()
            streamer = PrefillStreamer(HQ, HKV, n, D, nv, cfg, depth=3)
            reqs = [(hQ, hK, hV)] * args.steps
            streamer.run(reqs[:2], [hO, hO])  # warm-up
            streamer.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(streamer.h2d)
            streamer.run(reqs, [hO] * args.steps)
            ev1.record(streamer.d2h)
            streamer.synchronize()
            s_ms = ev0.elapsed_time(ev1) / args.steps
            line["e2e"] = {"value": n / (s_ms / 1e3), "unit": "tok/s", "ms_per_step": s_ms,
                           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": hO.numel() * hO.element_size(),
                           "api": "pipeline.PrefillStreamer: pinned host Q/K/V in, host O out, per request; "
                                  "copies of neighbouring requests overlap compute (CUDA events, H2D start to D2H end)",
                           "serial_ms_per_step": serial_ms}
            del streamer
            torch.cuda.empty_cache()
        log("cpu baseline")
        # ----- CPU reference path on the host cores (bounded sample)
        if not args.no_cpu:
            try:
                tps, t_step, desc, _ = cpu_reference_sample(Q, K, V, nv, args.tau, args.p)
                line["cpu_baseline"] = {"value": tps, "unit": "tok/s", "cores": os.cpu_count(), "kind": "port",
                                        "seconds_per_step_extrapolated": t_step, "sample": desc}
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline"] = {"error": str(e)[:200]}
        log("decode section")
        # ----- training step (C4: fwd + bwd at 32K)
        if not args.no_train:
            log("train section")
            try:
                line["train"] = train_section(args, max(3, args.steps // 2), 2, tc_peak)
            except Exception as e:  # noqa: BLE001
                line["train"] = {"error": str(e)[:300]}
            torch.cuda.empty_cache()
        # ----- decode (C5 shape at 1 GPU, sequence-sharded across ranks at N>1)
        if not args.no_decode:
            res = None
            torch.cuda.empty_cache()
            try:
                line["decode"] = decode_section(args, args.steps, args.warmup, hbm_peak)
                if not args.no_knobs:
                    torch.cuda.empty_cache()
                    line["decode_second_operating_point"] = decode_section(args, args.steps, args.warmup, hbm_peak,
                                                                           tau=0.12, p=0.75, dense=False)
            except Exception as e:  # noqa: BLE001
                line["decode"] = {"error": str(e)[:300]}
    print(json.dumps(headline_first(line)), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def headline_first(line: dict) -> dict:
    """The metric's own numbers first (the driver keeps the head of the line):
    speed-up over dense FA at both operating points, decode KV-bytes
    reduction and tok/s, the rooflines and the parity summary, then the
    rest."""
    head = {"metric": line["metric"], "value": line["value"], "unit": line["unit"]}
    sweep = {(k["lazy_fraction"], k["tau"], k["p"]): k for k in line.get("knob_sweep", [])}
    dec, dec2 = line.get("decode", {}), line.get("decode_second_operating_point", {})
    head["headline"] = {
        "speedup_vs_dense_fa_tau0.08_p0.82": line.get("speedup_vs_dense_fa"),
        "speedup_vs_dense_fa_tau0.12_p0.75": sweep.get((0.5, 0.12, 0.75), {}).get("speedup_vs_dense_fa"),
        "ms_per_step": line.get("ms_per_step"),
        "dense_fa_ms": line.get("dense_fa", {}).get("fastest_ms"),
        "train_speedup_vs_dense": line.get("train", {}).get("speedup_vs_dense"),
        "decode_tok_s": dec.get("tok_s"),
        "decode_kv_bytes_reduction_tau0.08_p0.82": dec.get("kv_bytes_reduction"),
        "decode_kv_bytes_reduction_tau0.12_p0.75": dec2.get("kv_bytes_reduction"),
        "decode_kv_bytes_reduction_reference_accounting_tau0.08_p0.82":
            dec.get("reference_accounting", {}).get("kv_bytes_reduction_per_q_head"),
    }
    for k in ("roofline", "parity"):
        if k in line:
            head[k] = line[k]
    if isinstance(line.get("train"), dict) and "roofline" in line["train"]:
        head["train_roofline"] = line["train"]["roofline"]
    for k, v in line.items():
        if k not in head:
            head[k] = v
    return head


def work_flops_shard(res, plan, d: int = D) -> float:
    """work_flops for one rank's Q heads (rows / counts local, selection global)."""
    import torch

    rep = plan.n_q_heads // plan.n_kv_heads
    counts = res.counts.cpu().tolist()
    b = res.selection.info[4:].cpu().tolist()
    total = 0
    for hl in range(res.rows.shape[0]):
        g = (plan.q_start + hl) // rep
        sel = res.selection.selected[g, : b[g]].contiguous()
        rows = res.rows[hl, : counts[hl]].contiguous()
        total += int(torch.searchsorted(sel, rows, right=True).sum())
    return 4.0 * d * total


def multi_rank_sections(args, line, step, res, plan, Ql, Kl, Vl, O, nv, cfg, world, tc_peak, peak_src):
    """N > 1 (every rank, same collective order): the K4 roofline over the
    shards (sum of the ranks' algorithmic FLOPs / the slowest rank's K4 time,
    per GPU), this rank's launch count, and the end-to-end metric through host
    buffers (each rank copies its shard of Q/K/V in and its O rows out)."""
    import torch
    import torch.distributed as dist

    from paper_2511_12201_b200 import ops
    from paper_2511_12201_b200.parallel import sparse_prefill_sharded

    sel_loc = res.selection.selected[plan.g_start:plan.g_stop]
    cnt_loc = res.selection.info[4 + plan.g_start: 4 + plan.g_stop]
    fa = lambda: ops.sparse_attn_fwd(Ql, res.K_sel, res.V_sel, Vl, res.rows, res.counts, sel_loc, cnt_loc,
                                     cfg.sink_index, O, res.lse)
    fa_ms = time_cuda(fa, args.steps, 2)
    flops = work_flops_shard(res, plan)
    t = torch.tensor([fa_ms], device="cuda")
    f = torch.tensor([flops], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(f, op=dist.ReduceOp.SUM)
    achieved = float(f) / (float(t) / 1e3) / 1e12 / world
    line["roofline"] = {"bound": "tensor", "kernel": "omni sparse_fwd_kernel (K4), per GPU over the shards",
                        "achieved": achieved, "peak": tc_peak, "unit": "TFLOP/s", "frac": achieved / tc_peak,
                        "traffic": None, "peak_source": f"{peak_src} bf16 burst (MEASURED_PEAKS.json)",
                        "launch_ms_max_over_ranks": float(t)}
    n_ours, n_all, names = count_launches(step)
    line["gpu_launches"] = n_ours * args.steps
    line["gpu_launches_per_step"] = {"ours_per_rank": n_ours, "all_per_rank": n_all, "kernels": names}
    if not args.no_e2e:
        hQ, hK, hV = (x.cpu().pin_memory() for x in (Ql, Kl, Vl))
        hO = torch.empty(O.shape, dtype=torch.bfloat16).pin_memory()

        def e2e():
            Ql.copy_(hQ, non_blocking=True)
            Kl.copy_(hK, non_blocking=True)
            Vl.copy_(hV, non_blocking=True)
            sparse_prefill_sharded(Ql, Kl, Vl, plan, nv, world, cfg, out=O)
            hO.copy_(O, non_blocking=True)

        dist.barrier()
        e_ms = time_cuda(e2e, max(3, args.steps // 2), 1)
        te = torch.tensor([e_ms], device="cuda")
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        n = Ql.shape[1]
        nb = torch.tensor([sum(x.numel() * x.element_size() for x in (hQ, hK, hV)), hO.numel() * hO.element_size()],
                          device="cuda", dtype=torch.float64)
        dist.all_reduce(nb, op=dist.ReduceOp.SUM)
        line["e2e"] = {"value": n / (float(te) / 1e3), "unit": "tok/s", "ms_per_step": float(te),
                       "h2d_bytes_per_step": int(nb[0]), "d2h_bytes_per_step": int(nb[1]),
                       "api": "parallel.sparse_prefill_sharded per rank: pinned host shard in, host O rows out "
                              "(time: max over ranks; bytes: summed over ranks)"}


def multi_rank_decode_train(args, line, world, rank, hbm_peak, plan):
    """N > 1, every rank: C5 decode sequence-sharded (no collective) and the C4
    training step head-sharded (parallel.sparse_attention_sharded: one
    all_gather of block masses forward, one dK / dV all-reduce per split KV
    group backward); step times are the max over ranks."""
    import torch
    import torch.distributed as dist

    if not args.no_decode:
        log("decode section (sequence-sharded)")
        line["decode"] = decode_section(args, args.steps, args.warmup, hbm_peak, world=world, rank=rank)
        torch.cuda.empty_cache()
    if not args.no_train:
        log("train section (head-sharded)")
        from paper_2511_12201_b200.parallel import kv_grad_group, sparse_attention_sharded
        from paper_2511_12201_b200.pipeline import SparsityConfig
        from paper_2511_12201_b200.synthetic import generate_device

        n = 32768
        nv = n - N_TEXT
        cfg = SparsityConfig(tau=args.tau, p=args.p)
        kvg = kv_grad_group(HQ, HKV, world, rank)
        Q, K, V = generate_device(HQ, HKV, D, nv, N_TEXT, seed=3, lazy_fraction=args.lazy)
        Ql = Q[plan.q_start:plan.q_stop].clone().requires_grad_(True)
        Kl, Vl = (x[plan.g_start:plan.g_stop].clone().requires_grad_(True) for x in (K, V))
        dO = torch.randn_like(Ql)
        del Q, K, V

        def train_step():
            O = sparse_attention_sharded(Ql, Kl, Vl, plan, nv, world, cfg, kv_group=kvg)
            O.backward(dO)

        train_step()
        dist.barrier()
        ms = time_cuda(train_step, max(3, args.steps // 2), 2)
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        line["train"] = {"workload": f"sparse attention fwd+bwd, {HQ}/{HKV} heads, d={D}, {n} tokens (C4), "
                                     f"head-sharded x{world}", "ms_per_step": float(t),
                         "tok_s": n / (float(t) / 1e3)}


def _reference_step(sa, Q, K, V, nv, tau, p, rows_sample, seed, heads=(0, 13, 27)):
    """One bounded sample step of the REFERENCE package (slimattn, its own
    functions and Cython/NumPy core) on the bench workload under GQA rule B:
    the complete selection over all 28 Q heads — build_probe_keys,
    classify_queries, probe_attention + block_scores_to_token_scores per Q
    head, group sums, key_scores_from_vectors, flattest_head,
    budget_with_retained_mass, build_key_masks — then sparse_head_attention
    for `rows_sample` random active rows of each of three heads (the
    reference's own function, its `active` mask restricted to the sample).
    Returns (seconds of this step, seconds of a full step extrapolated, desc)."""
    import numpy as np

    att, qs, bp, kv, pf = sa["attention"], sa["query_select"], sa["block_probe"], sa["kv_select"], sa["prefill"]
    hq, hkv = len(Q), len(K)
    rep = hq // hkv
    n = Q[0].shape[0]
    layout = att.TokenLayout(n_vision=nv, n_text=n - nv)
    t0 = time.perf_counter()
    probes = [qs.build_probe_keys(K[g], layout) for g in range(hkv)]
    active = []
    for h in range(hq):
        _, verdict = qs.classify_queries(Q[h][:nv], probes[h // rep], tau)
        a = np.ones(n, dtype=bool)
        a[:nv] = verdict
        active.append(a if h else np.ones(n, dtype=bool))  # preserve_first_head
    per_head = [bp.block_scores_to_token_scores(bp.probe_attention(Q[h], K[h // rep], 256), n) for h in range(hq)]
    groups = []
    for g in range(hkv):
        acc = per_head[g * rep].copy()
        for r in range(1, rep):
            acc += per_head[g * rep + r]
        groups.append(acc)
    scores = kv.key_scores_from_vectors(groups)
    flat = kv.flattest_head(scores)
    b, _, _ = kv.budget_with_retained_mass(scores.scores[flat], p)
    sel = kv.build_key_masks(scores, b)
    t_sel = time.perf_counter() - t0
    rng = np.random.default_rng(seed)
    t0 = time.perf_counter()
    sampled = 0
    for h in heads:
        rows = np.flatnonzero(active[h])
        pick = np.zeros(n, dtype=bool)
        pick[rng.choice(rows, min(rows_sample, rows.size), replace=False)] = True
        pf.sparse_head_attention(Q[h], K[h // rep], V[h // rep], sel.selected[h // rep], pick, 0)
        sampled += int(pick.sum())
    t_att = time.perf_counter() - t0
    total_rows = int(sum(int(a.sum()) for a in active))
    full = t_sel + t_att * total_rows / sampled
    desc = (f"slimattn {sa['version']} ({sa['backend']} core) from baseline/_ref, float64: full selection over {hq} "
            f"Q heads ({t_sel:.2f} s) + sparse_head_attention of {sampled} random active rows of heads {list(heads)} "
            f"({t_att:.2f} s); full step extrapolated to all {total_rows} active rows = {full:.1f} s")
    return t_sel + t_att, full, desc


def _load_reference():
    """The unmodified reference package installed in baseline/_ref (pip
    install --target), or None."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "slimattn")):
        return None
    sys.path.insert(0, ref)
    try:
        import importlib

        mods = {m: importlib.import_module(f"slimattn.{m}") for m in
                ("attention", "query_select", "block_probe", "kv_select", "prefill", "backend")}
        mods["backend_name"] = mods["backend"].ACTIVE_BACKEND
        mods["backend"] = mods["backend_name"]
        mods["version"] = "0.1.0"
        return mods
    except Exception as e:  # noqa: BLE001
        log(f"reference import failed: {e}")
        return None


def run_reference(args):
    """--impl reference: the reference's own CPU implementation (slimattn from
    baseline/_ref, Cython core, OpenBLAS on all host threads) on this arm's
    config and metric; rank 0 only. Each step is a bounded sample of the 64K
    layer (the full selection + a row sample of the attention); `ms_per_step`
    is that sample's measured time, `value` the layer throughput it
    extrapolates to. Falls back to the oracle port when baseline/_ref is
    absent (kind "port")."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import torch

    from paper_2511_12201_b200.synthetic import generate_device

    n, nv = args.seq, args.seq - N_TEXT
    dev = "cuda" if torch.cuda.is_available() else "cpu"  # same tensors as our arm when a GPU is present
    Qd, Kd, Vd = generate_device(HQ, HKV, D, nv, N_TEXT, seed=0, lazy_fraction=args.lazy, device=dev)
    to64 = lambda t: list(t.float().cpu().numpy().astype(np.float64))
    Q, K, V = to64(Qd), to64(Kd), to64(Vd)
    del Qd, Kd, Vd
    sa = _load_reference()
    times, fulls, desc = [], [], ""
    for i in range(args.warmup + args.steps):
        if sa is not None:
            t, full, desc = _reference_step(sa, Q, K, V, nv, args.tau, args.p, 128, seed=i)
        else:
            t0 = time.perf_counter()
            _, full, desc, _ = cpu_reference_sample(torch.from_numpy(np.stack(Q)), torch.from_numpy(np.stack(K)),
                                                    torch.from_numpy(np.stack(V)), nv, args.tau, args.p,
                                                    rows_sample=256, seed=i)
            t = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(t)
            fulls.append(full)
    ms = 1e3 * sum(times) / len(times)
    full_s = sum(fulls) / len(fulls)
    value = n / full_s
    kind = "reference" if sa is not None else "port"
    line = {"metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "impl": "reference",
            "data": "synthetic: reference generator construction (GQA rule B), the same tensors as the GPU arm",
            "config": {"workload": f"Qwen2-7B-shaped attention layer sparse prefill, {HQ} Q / {HKV} KV heads, d={D}, "
                                   f"{n} tokens ({nv} vision + {N_TEXT} text)",
                       "knobs": {"tau": args.tau, "p": args.p, "block_size": 256, "lazy_fraction": args.lazy,
                                 "granularity": "token", "preserve_first_head": True}},
            "full_step_seconds_extrapolated": full_s,
            "timing_note": "ms_per_step = measured time of one bounded sample step; value = 64K-token layer "
                           "throughput extrapolated from it (full selection timed, attention rows sampled)",
            "cpu_baseline": {"value": value, "unit": "tok/s", "cores": os.cpu_count(), "kind": kind, "sample": desc},
            "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
