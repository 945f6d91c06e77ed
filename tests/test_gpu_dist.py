"""The multi-GPU data plane on one B200 (SURVEY §8 row e): two ranks share cuda:0
over gloo (the box has one GPU; the product uses NCCL, same calls) and run the
config-4 (Student-t moments) and config-5 (Monte-Carlo call sweep) pipelines of
shard.py through the kernels; the all-reduced sums must be bit-identical to the
one-rank run (fixed chunks, one contributor per row, fixed-order reduction)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N4 = 37 * 65536 + 1234           # config 4 samples (not a multiple of the chunk)
N5 = (1 << 23) + (1 << 20) + 999  # config 5 samples
STRIKES = list(np.linspace(50, 150, 17))


def _pipelines(rank, world):
    from paper_0901_0638_b200 import shard as S
    sums4, _ = S.student_moments(N4, 5.0, 16, 4.6506, 0x5EEDC0FFEE123457, rank, world)
    price, se = S.mc_call_sweep(N5, 2024, 100.0, 0.05, 0.2, 1.0, STRIKES, rank, world)
    torch.cuda.synchronize()
    return sums4.cpu().numpy(), price.cpu().numpy(), se.cpu().numpy()


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = _pipelines(rank, world)
    if rank == 0:
        q.put(res)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_on_one_gpu_bit_identical_to_one_rank():
    one = _pipelines(0, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    two = q.get(timeout=600)
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    for a, b in zip(one, two):
        assert np.array_equal(a, b), (a, b)
