"""Multi-GPU host logic on CPU (gloo, world size 2): sharding of the Philox
stream and the exact, order-independent all-reduce of moment rows (SURVEY §8
rows a8, e).  The per-chunk sums are computed here with numpy as a stand-in for
the device kernel -- these tests cover the exchange, not the kernel."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0901_0638_b200.shard import QM_MOMENT_CHUNK, allreduce_rows, global_rows, shard


@pytest.mark.parametrize("n", [0, 1, 65535, 65536, 65537, 10 * 65536 + 123, 1 << 22])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shards_tile_the_stream(n, world):
    shards = [shard(n, world, r, 4) for r in range(world)]
    pos, row = 0, 0
    for s in shards:
        assert s.start == pos and s.count >= 0
        assert s.start % QM_MOMENT_CHUNK == 0 or s.count == 0
        assert s.counter_offset * 4 == s.start
        assert s.row0 == row
        pos += s.count
        row += s.nrows
    assert pos == n and row == global_rows(n)
    s64 = shard(n, world, world - 1, 8)
    assert s64.counter_offset * 2 == s64.start


def _rows_of(x, lo, hi):
    """numpy stand-in for qm_moment_rows on samples [lo, hi) of the global stream."""
    out = []
    for c in range(lo // QM_MOMENT_CHUNK, -(-hi // QM_MOMENT_CHUNK)):
        seg = x[c * QM_MOMENT_CHUNK:min((c + 1) * QM_MOMENT_CHUNK, hi)].astype(np.float64)
        out.append([seg.sum(), (seg ** 2).sum(), (seg ** 3).sum(), (seg ** 4).sum()])
    return np.array(out, dtype=np.float64).reshape(-1, 4)


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = np.random.default_rng(7).standard_normal(n)
    s = shard(n, world, rank, 8)
    rows = torch.zeros((global_rows(n), 4), dtype=torch.float64)
    if s.count:
        rows[s.row0:s.row0 + s.nrows] = torch.from_numpy(_rows_of(x, s.start, s.start + s.count))
    allreduce_rows(rows)
    if rank == 0:
        q.put(rows.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, PORT[world], n, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


PORT = {1: _free_port(), 2: _free_port()}


def test_gloo_allreduce_of_rows_is_exact_and_world_size_independent():
    n = 5 * QM_MOMENT_CHUNK + 777
    one = _run(1, n)
    two = _run(2, n)
    x = np.random.default_rng(7).standard_normal(n)
    ref = _rows_of(x, 0, n)
    assert np.array_equal(one, ref)
    assert np.array_equal(two, ref)          # bit-identical: every row has one contributor
