"""Multi-process host logic of the head-sharded prefill (CPU, gloo backend).

The CUDA kernels cannot run here, so each rank computes its local Q heads'
block column masses with the oracle (the quantity K3a produces), exchanges
them through parallel.gather_block_mass (the same all_gather the NCCL path
runs) and runs the selection on the gathered masses. The result must be
bit-identical to the single-process selection."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_12201_b200.parallel import shard_plan


def test_shard_plan_covers_every_head_once():
    for world in (1, 2, 4, 8):
        plans = [shard_plan(28, 4, world, r) for r in range(world)]
        heads = sorted(h for p in plans for h in range(p.q_start, p.q_stop))
        assert heads == list(range(28))
        for p in plans:
            # every local Q head belongs to a local KV group (rule B, rep = 7)
            for h in range(p.q_start, p.q_stop):
                assert p.g_start <= h // 7 < p.g_stop
    # the rank holding the fully active head 0 takes one head fewer
    assert [shard_plan(28, 4, 8, r).q_heads for r in range(8)] == [3, 4] * 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_dir):
    from oracle import pipeline as opipe
    from oracle import selection as osel
    from oracle.workload import Spec, generate
    from paper_2511_12201_b200.parallel import gather_block_mass

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    Q, K, V = generate(Spec(heads=8, heads_kv=2, head_dim=32, n_vision=1000, n_text=24, seed=4))
    plan = shard_plan(8, 2, world, rank)
    rep = 4
    local = np.stack([osel.block_mass(osel.probe_map(Q[h], K[h // rep], 64)) for h in range(plan.q_start, plan.q_stop)])
    full = gather_block_mass(torch.from_numpy(local), plan, world).numpy()
    res = opipe.select(Q, K, 1000, 0, 0.08, 0.82, 64, block_mass_override=full)
    np.savez(os.path.join(result_dir, f"rank{rank}.npz"), mass=full, budget=res.budget, flattest=res.flattest,
             selected=np.stack(res.selected))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gathered_selection_matches_single_process(tmp_path, world):
    from oracle import pipeline as opipe
    from oracle.workload import Spec, generate

    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    Q, K, V = generate(Spec(heads=8, heads_kv=2, head_dim=32, n_vision=1000, n_text=24, seed=4))
    ref = opipe.select(Q, K, 1000, 0, 0.08, 0.82, 64)
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npz")
        np.testing.assert_array_equal(got["mass"], ref.block_mass)
        assert int(got["budget"]) == ref.budget and int(got["flattest"]) == ref.flattest
        np.testing.assert_array_equal(got["selected"], np.stack(ref.selected))


def test_sequence_shard_covers_the_batch():
    from paper_2511_12201_b200.parallel import sequence_shard

    for batch, world in ((32, 8), (32, 1), (30, 8), (5, 2), (3, 4)):
        seqs = [s for r in range(world) for s in sequence_shard(batch, world, r)]
        assert seqs == list(range(batch))
    assert [len(sequence_shard(32, 8, r)) for r in range(8)] == [4] * 8  # C5: 4 sequences per GPU


def _grad_worker(rank, world, port, result_dir):
    from paper_2511_12201_b200.parallel import ReduceGradOverGroup, gather_decode_outputs, kv_grad_group

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    # 4 ranks over 2 KV groups: ranks {0, 1} share group 0, {2, 3} group 1
    grp = kv_grad_group(8, 2, world, rank)
    x = torch.arange(6, dtype=torch.float32).requires_grad_(True)
    y = ReduceGradOverGroup.apply(x, grp)
    (y * float(rank + 1)).sum().backward()
    # decode outputs of a 5-sequence batch sharded over the ranks, reassembled
    from paper_2511_12201_b200.parallel import sequence_shard

    mine = sequence_shard(5, world, rank)
    local = torch.stack([torch.full((2, 3), float(s)) for s in mine]) if len(mine) else torch.zeros(0, 2, 3)
    full = gather_decode_outputs(local, 5, world)
    np.savez(os.path.join(result_dir, f"g{rank}.npz"), grad=x.grad.numpy(), full=full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_split_group_kv_gradients_are_summed_and_decode_outputs_gathered(tmp_path):
    """world 4 over 2 KV groups (the 8-GPU / 4-group split at small scale):
    a group's dK / dV partials are summed over exactly the ranks sharing it;
    sequence-sharded decode outputs reassemble in sequence order."""
    world = 4
    mp.spawn(_grad_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        z = np.load(tmp_path / f"g{r}.npz")
        share = (1 + 2) if r < 2 else (3 + 4)  # sum of the weights (rank + 1) in this rank's group
        np.testing.assert_array_equal(z["grad"], np.full(6, float(share)))
        np.testing.assert_array_equal(z["full"][:, 0, 0], np.arange(5, dtype=np.float32))
