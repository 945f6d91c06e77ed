"""Programmatic dependent launch (qm_lib.cu launch_pdl, qm_tma.cuh pdl_begin): a
launch may start while the previous grid on the stream drains, and must wait for
it before touching global memory.  A chain of maps where every launch reads the
previous launch's output, enqueued back to back (and captured in a CUDA graph),
must give bit for bit the result of the same chain with a synchronize after each
launch."""
import numpy as np
import pytest
import torch

from synth import inputs as I

pytestmark = pytest.mark.gpu
Q = pytest.importorskip("paper_0901_0638_b200.qm")


def _chain(v0, steps, sync):
    a, b = v0.clone(), torch.empty_like(v0)
    for _ in range(steps):
        Q.qm_recycle_exp_to_normal(a, out=b)          # TMA tiles + LDG remainder, both PDL-launched
        if sync:
            torch.cuda.synchronize()
        a, b = b, a
    return a


@pytest.mark.parametrize("n", [(1 << 23) + 37, 4099])
def test_dependent_chain_matches_synchronised_chain(n):
    v0 = torch.from_numpy(I.laplace(n, dtype=np.float32)).cuda()
    ref = _chain(v0, 12, sync=True)
    got = _chain(v0, 12, sync=False)
    torch.cuda.synchronize()
    assert torch.equal(got.nan_to_num(), ref.nan_to_num()) and torch.equal(got.isnan(), ref.isnan())


def test_dependent_chain_in_a_graph():
    n = (1 << 23) + 37
    v0 = torch.from_numpy(I.laplace(n, dtype=np.float32)).cuda()
    ref = _chain(v0, 8, sync=True)
    a, b = v0.clone(), torch.empty_like(v0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        x, y = a, b
        for _ in range(8):
            Q.qm_recycle_exp_to_normal(x, out=y, stream=s)
            x, y = y, x
    a.copy_(v0)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(x.nan_to_num(), ref.nan_to_num())


def test_uniforms_then_quantile_back_to_back():
    """producer (Philox) and consumer (the map) enqueued without a sync, repeatedly
    overwriting the producer's buffer: the map always sees the finished uniforms"""
    n = (1 << 23) + 5
    u = torch.empty(n, dtype=torch.float32, device="cuda")
    outs = []
    for seed in range(4):
        Q.qm_philox_uniform(n, seed, 0, out=u)
        outs.append(Q.qm_normal_quantile(u))
    torch.cuda.synchronize()
    for seed in range(4):
        ref = Q.qm_normal_quantile(Q.qm_philox_uniform(n, seed, 0))
        torch.cuda.synchronize()
        assert torch.equal(outs[seed], ref)
