"""Full-size parity in the launch configurations bench.py times (BASELINE.json
configs 2-5): sampled outputs checked one by one against the oracle, plus
whole-array properties that hold at any size."""
import numpy as np
import pytest
import torch

import oracle as O
from _parity import summary, ulp_errors

pytestmark = pytest.mark.gpu
Q = pytest.importorskip("paper_0901_0638_b200")
SEED = 0x5EEDC0FFEE123457


def _sample(n, k, seed):
    return np.sort(np.random.default_rng(seed).choice(n, k, replace=False))


def test_fp64_streaming_2p28():
    """2^28 fp64 odd-grid uniforms -> App D through the TMA pipeline (bench variant
    stream_f64_D13_2^28)."""
    n = 1 << 28
    u = Q.qm_philox_uniform(n, SEED, 0, dtype=torch.float64)
    z = Q.qm_normal_quantile(u)
    idx = _sample(n, 1 << 18, 3)
    ti = torch.from_numpy(idx).cuda()
    us, zs = u[ti].cpu().numpy(), z[ti].cpu().numpy()
    assert np.array_equal(us, O.philox_uniform_at(idx, SEED, 0, np.float64))
    err = ulp_errors(zs, O.normal_breakless(us, O.D13, 64), np.float64)
    assert err.max() <= 2.0, summary(err)
    assert bool(torch.isfinite(z).all()) and float(z.abs().max()) < 8.6   # v <= 37.4 on the grid
    assert int((z > 0).sum()) == int((u > 0.5).sum())
    del u, z


def test_fused_fp64_2p31():
    """configs[2] fp64: Philox-fused 2^31 fp64 normals, sampled parity."""
    n = 1 << 31
    z = Q.qm_normal_philox(n, SEED, 0, dtype=torch.float64)
    idx = _sample(n, 1 << 17, 4)
    zs = z[torch.from_numpy(idx).cuda()].cpu().numpy()
    us = O.philox_uniform_at(idx, SEED, 0, np.float64)
    err = ulp_errors(zs, O.normal_breakless(us, O.D13, 64), np.float64)
    assert err.max() <= 2.0, summary(err)
    del z


@pytest.mark.parametrize("nu,K,zstar", [(3.0, 16, 3.5667), (5.0, 16, 4.6506), (10.0, 16, 6.9584)])
def test_student_2p30(nu, K, zstar):
    """configs[3]: 2^30 fp64 normals (the fused producer) -> Student-t through the
    TMA pipeline with the unrolled series; sampled parity, and the tail lanes."""
    n = 1 << 30
    zn = Q.qm_normal_philox(n, SEED, 0, dtype=torch.float64)
    t = Q.qm_recycle_normal_to_t(zn, nu, K, zstar)
    idx = _sample(n, 1 << 16, 5)
    ti = torch.from_numpy(idx).cuda()
    zs, ts = zn[ti].cpu().numpy(), t[ti].cpu().numpy()
    err = ulp_errors(ts, O.student_map(zs, nu, K, zstar), np.float64)
    assert err.max() <= 2.0, summary(err)
    # every tail sample of the whole array (|z| >= z*, ~1e-4 .. 1e-11 of them)
    tail = (zn.abs() >= zstar).nonzero().flatten()[:4096]
    if tail.numel():
        zt, tt = zn[tail].cpu().numpy(), t[tail].cpu().numpy()
        err = ulp_errors(tt, O.student_map(zt, nu, K, zstar), np.float64)
        assert err.max() <= 2.0, summary(err)
    assert bool(torch.equal(torch.sign(t), torch.sign(zn)))               # odd, monotone map
    del zn, t


def test_exp_to_normal_2p28():
    """configs[4] building block: 2^28 fp32 Laplace samples -> normal (no log)."""
    n = 1 << 28
    u = Q.qm_philox_uniform(n, SEED, 0)
    v = torch.where(u < 0.5, torch.log(2 * u), -torch.log(2 * (1 - u)))     # Laplace (input only)
    z = Q.qm_recycle_exp_to_normal(v)
    idx = _sample(n, 1 << 18, 6)
    ti = torch.from_numpy(idx).cuda()
    vs, zs = v[ti].cpu().numpy(), z[ti].cpu().numpy()
    err = ulp_errors(zs, O.exp_to_normal(vs.astype(np.float64), O.C55, 32), np.float32)
    assert err.max() <= 4.0, summary(err)
    del u, v, z
