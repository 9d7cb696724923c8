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
