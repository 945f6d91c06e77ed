"""Multi-GPU sharding of the sample stream and the one collective of the path
(SURVEY §8 row e): samples are independent, so rank r of G maps a contiguous
slice of the global Philox stream (counter offset = first sample / samples per
Philox block) and no data crosses GPUs; the only exchange is the all-reduce of
the moment / Monte-Carlo sums (row a8).

Exactness across G: partial sums live in fixed chunks of the GLOBAL stream
(``QM_MOMENT_CHUNK`` samples per row, see include/qm.h).  Each rank writes its
rows into a zeroed global row matrix; all_reduce(SUM) of that matrix is exact
(one non-zero contributor per row) and the fixed-order ``qm_reduce_rows`` gives
the same bits for any number of ranks.
"""
from __future__ import annotations

from dataclasses import dataclass

QM_MOMENT_CHUNK = 65536
QM_MC_CHUNK = 1 << 20
WORDS_PER_BLOCK = {4: 4, 8: 2}     # fp32: 4 samples per Philox block, fp64: 2


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int          # first global sample index of this rank
    count: int          # samples owned by this rank
    counter_offset: int  # Philox block counter of `start`
    row0: int           # first global moment row of this rank
    nrows: int          # moment rows owned by this rank


def shard(n_total: int, world: int, rank: int, itemsize: int = 4, chunk: int = QM_MOMENT_CHUNK) -> Shard:
    """Contiguous shard of a global stream of n_total samples.

    Shard boundaries fall on `chunk` multiples (QM_MOMENT_CHUNK for moment rows,
    QM_MC_CHUNK for Monte-Carlo rows), so every row has exactly one owner and
    Philox blocks never straddle ranks; the last rank takes the remainder."""
    if world < 1 or not (0 <= rank < world) or n_total < 0:
        raise ValueError("bad shard arguments")
    nchunks = -(-n_total // chunk)
    c0 = (nchunks * rank) // world
    c1 = (nchunks * (rank + 1)) // world
    start = min(c0 * chunk, n_total)
    end = min(c1 * chunk, n_total)
    wpb = WORDS_PER_BLOCK[itemsize]
    return Shard(rank, world, start, end - start, start // wpb, c0, c1 - c0)


def global_rows(n_total: int) -> int:
    return -(-n_total // QM_MOMENT_CHUNK)


def allreduce_rows(rows, group=None):
    """all_reduce(SUM) of a zero-padded global row matrix (exact: one non-zero
    contributor per row).  Works on NCCL (CUDA tensors) and gloo (CPU)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(rows, op=dist.ReduceOp.SUM, group=group)
    return rows


def student_moments(n_total: int, nu: float, K: int, zstar: float, seed: int, rank: int = 0, world: int = 1,
                    dtype=None, group=None, device=None):
    """Config 4 on G GPUs: rank r draws its slice of 2^k fp64 standard normals
    (fused Philox + breakless quantile), recycles them into Student-t (row a6),
    writes its moment rows, all-reduces the row matrix over NCCL and reduces it
    in a fixed order.  Returns (sums[4] on the device, local t samples)."""
    import torch

    from . import qm as Q
    dtype = dtype or torch.float64
    itemsize = torch.tensor([], dtype=dtype).element_size()
    sh = shard(n_total, world, rank, itemsize)
    z = Q.qm_normal_philox(sh.count, seed, sh.counter_offset, dtype=dtype, device=device)
    rows = torch.zeros((global_rows(n_total), 4), dtype=torch.float64, device=z.device)
    if sh.count:   # the map with the moment rows fused (one pass over t)
        t, _ = Q.qm_recycle_normal_to_t_moments(z, nu, K, zstar, rows=rows[sh.row0:sh.row0 + sh.nrows])
    else:
        t = z
    allreduce_rows(rows, group)
    return Q.qm_reduce_rows(rows), t


def mc_call_sweep(n_total: int, seed: int, S0: float, r: float, sigma: float, T: float, strikes,
                  rank: int = 0, world: int = 1, group=None, device=None):
    """Config 5 on G GPUs: rank r prices its slice of the exponential-base
    Monte-Carlo stream (qm_mc_european_call), writes its rows into a zeroed
    global row matrix, all-reduces it over NCCL and reduces it in a fixed order.
    Returns (prices[nstrikes], standard errors[nstrikes]) as CUDA tensors."""
    import math

    import torch

    from . import qm as Q
    ks = list(strikes)
    sh = shard(n_total, world, rank, 4, QM_MC_CHUNK)
    rows = torch.zeros((-(-n_total // QM_MC_CHUNK), 2 * len(ks)), dtype=torch.float64, device=device or "cuda")
    if sh.count:
        Q.qm_mc_european_call(sh.count, seed, sh.counter_offset, S0, r, sigma, T, ks,
                              out=rows[sh.row0:sh.row0 + sh.nrows])
    allreduce_rows(rows, group)
    sums = Q.qm_reduce_rows(rows).view(-1, 2)
    disc = math.exp(-r * T)
    mean = sums[:, 0] / n_total
    var = sums[:, 1] / n_total - mean * mean
    return disc * mean, disc * torch.sqrt(var.clamp_min(0) / n_total)
