"""Head-sharded prefill (parallel.py) run for real on the GPU:
world 2 / 4 / 8 processes share the one visible device (gloo carries the
block-mass all_gather; NCCL is what bench.py uses across GPUs). Every rank's
outputs must equal the single-process pipeline's bit for bit — the shards
compute the same kernels on the same heads and the selection is redundant."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

HQ, HKV, D, NV, NT = 28, 4, 128, 4000, 96


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs():
    from paper_2511_12201_b200.synthetic import generate_device

    return generate_device(HQ, HKV, D, NV, NT, seed=21)


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    from paper_2511_12201_b200.parallel import shard_plan, sparse_prefill_sharded
    from paper_2511_12201_b200.pipeline import SparsityConfig

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    Q, K, V = _inputs()
    plan = shard_plan(HQ, HKV, world, rank)
    Ql = Q[plan.q_start:plan.q_stop].contiguous()
    Kl, Vl = (x[plan.g_start:plan.g_stop].contiguous() for x in (K, V))
    res = sparse_prefill_sharded(Ql, Kl, Vl, plan, NV, world, SparsityConfig())
    torch.cuda.synchronize()
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), q_start=plan.q_start, q_stop=plan.q_stop,
             out=res.outputs.view(torch.int16).cpu().numpy(), info=res.selection.info.cpu().numpy(),
             sel=res.selection.selected.cpu().numpy(), active=res.active.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_prefill_equals_single_gpu(tmp_path, world):
    from paper_2511_12201_b200.pipeline import SparsityConfig, sparse_prefill_device

    Q, K, V = _inputs()
    ref = sparse_prefill_device(Q, K, V, NV, SparsityConfig())
    torch.cuda.synchronize()
    ref_out = ref.outputs.view(torch.int16).cpu().numpy()
    ref_info = ref.selection.info.cpu().numpy()
    ref_sel = ref.selection.selected.cpu().numpy()
    ref_act = ref.active.cpu().numpy()
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    covered = []
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        a, b = int(z["q_start"]), int(z["q_stop"])
        covered += list(range(a, b))
        np.testing.assert_array_equal(z["info"], ref_info)
        b_ = int(ref_info[0])
        np.testing.assert_array_equal(z["sel"][:, :b_], ref_sel[:, :b_])
        np.testing.assert_array_equal(z["active"], ref_act[a:b])
        np.testing.assert_array_equal(z["out"], ref_out[a:b])  # bf16 bits
    assert sorted(covered) == list(range(HQ))


# ------------------------------------------------------------ sequence-sharded decode
B_DEC, HQ_D, HKV_D, NV_D, NT_D = 6, 8, 2, 3000, 40


def _decode_batch(seqs, steps=3):
    """Slim caches of the given sequences, batched, decoded for `steps` steps
    with answer growth; returns the outputs of every step [steps, len, Hq, d]."""
    from paper_2511_12201_b200 import decode as gdec
    from paper_2511_12201_b200.pipeline import SparsityConfig
    from paper_2511_12201_b200.synthetic import decode_queries_device, generate_device, unit_vision_mean

    caches, means = [], []
    for s in seqs:
        Q, K, V = generate_device(HQ_D, HKV_D, D, NV_D, NT_D, seed=300 + s)
        caches.append(gdec.cache_from_prompt(Q, K, V, NV_D, NT_D, SparsityConfig(), answer_capacity=8))
        means.append(unit_vision_mean(K, NV_D))
    batch = gdec.stack_caches(caches)
    outs = []
    for t in range(steps):
        q = decode_queries_device(HQ_D, HKV_D, means, seqs, 0.5, t)
        out, _ = gdec.decode_attention_batch(q, batch, 0.08)
        outs.append(out)
        gen = torch.Generator(device="cuda")
        gen.manual_seed(t)
        kv = torch.randn(B_DEC, HKV_D, D, generator=gen, device="cuda").bfloat16()
        idx = torch.tensor(list(seqs), device="cuda")
        gdec.append_answer_batch(batch, kv[idx], -kv[idx])
    return torch.stack(outs)


def _decode_worker(rank, world, port, out_dir):
    import torch.distributed as dist

    from paper_2511_12201_b200.parallel import gather_decode_outputs, sequence_shard

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    mine = list(sequence_shard(B_DEC, world, rank))
    outs = _decode_batch(mine)
    full = gather_decode_outputs(outs[-1].cpu(), B_DEC, world)
    np.savez(os.path.join(out_dir, f"d{rank}.npz"), seqs=np.array(mine), outs=outs.cpu().numpy(), full=full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sequence_sharded_decode_equals_single_gpu(tmp_path, world):
    """C5's sharding: each rank builds and decodes only its sequences (no
    collective); every sequence's outputs equal the single-process batch's
    bit for bit, and the gathered last step is the full batch's."""
    ref = _decode_batch(list(range(B_DEC))).cpu().numpy()
    mp.start_processes(_decode_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        z = np.load(tmp_path / f"d{r}.npz")
        seqs = list(z["seqs"])
        np.testing.assert_array_equal(z["outs"], ref[:, seqs])
        np.testing.assert_array_equal(z["full"], ref[-1])


# ------------------------------------------------------------ head-sharded training
NV_T, NT_T = 3000, 72


def _train_inputs():
    from paper_2511_12201_b200.synthetic import generate_device

    Q, K, V = generate_device(HQ, HKV, D, NV_T, NT_T, seed=33)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    dO = torch.randn(Q.shape, generator=gen, device="cuda").bfloat16()
    return Q, K, V, dO


def _train_worker(rank, world, port, out_dir):
    import torch.distributed as dist

    from paper_2511_12201_b200.parallel import kv_grad_group, shard_plan, sparse_attention_sharded
    from paper_2511_12201_b200.pipeline import SparsityConfig

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    Q, K, V, dO = _train_inputs()
    plan = shard_plan(HQ, HKV, world, rank)
    kvg = kv_grad_group(HQ, HKV, world, rank)
    Ql = Q[plan.q_start:plan.q_stop].clone().requires_grad_(True)
    Kl, Vl = (x[plan.g_start:plan.g_stop].clone().requires_grad_(True) for x in (K, V))
    O = sparse_attention_sharded(Ql, Kl, Vl, plan, NV_T, world, SparsityConfig(), kv_group=kvg)
    O.backward(dO[plan.q_start:plan.q_stop])
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy()
    np.savez(os.path.join(out_dir, f"t{rank}.npz"), q0=plan.q_start, q1=plan.q_stop, g0=plan.g_start,
             g1=plan.g_stop, o=f(O.detach()), dq=f(Ql.grad), dk=f(Kl.grad), dv=f(Vl.grad))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_head_sharded_training_equals_single_gpu(tmp_path, world):
    """Training forward + backward sharded by heads: outputs and
    dQ equal the single-process autograd bit for bit. dK / dV are fp32 sums
    over a group's Q heads accumulated with vector atomics (summation order
    varies run to run, in one process too), then rounded to the bf16 leaf
    dtype: equal to one bf16 ulp. At 8 ranks each group's Q heads are split
    3 + 4 and the two fp32 partials are all-reduced before that rounding."""
    from paper_2511_12201_b200.autograd import sparse_attention
    from paper_2511_12201_b200.pipeline import SparsityConfig

    Q, K, V, dO = _train_inputs()
    Qg, Kg, Vg = (x.clone().requires_grad_(True) for x in (Q, K, V))
    O = sparse_attention(Qg, Kg, Vg, NV_T, SparsityConfig())
    O.backward(dO)
    torch.cuda.synchronize()
    f = lambda t: t.float().cpu().numpy()
    ref = dict(o=f(O.detach()), dq=f(Qg.grad), dk=f(Kg.grad), dv=f(Vg.grad))
    mp.start_processes(_train_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        z = np.load(tmp_path / f"t{r}.npz")
        q0, q1, g0, g1 = (int(z[k]) for k in ("q0", "q1", "g0", "g1"))
        np.testing.assert_array_equal(z["o"], ref["o"][q0:q1])
        np.testing.assert_array_equal(z["dq"], ref["dq"][q0:q1])
        for key in ("dk", "dv"):
            r_ = ref[key][g0:g1]
            # one bf16 ulp (2^-7 relative at worst), tiny absolute floor near zero
            np.testing.assert_allclose(z[key], r_, rtol=2.0 ** -7, atol=1e-6 * float(np.abs(r_).max()))
