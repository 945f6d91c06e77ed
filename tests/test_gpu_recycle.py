"""GPU parity of the recycling maps and the reductions."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import inputs as I
from _parity import summary, ulp_errors

pytestmark = pytest.mark.gpu

Q = pytest.importorskip("paper_0901_0638_b200")

# (nu, K, zstar): the paper's configuration and the min-max crossovers of
# tests/golden/student_crossover.txt
STUDENT = [(4.0, 10, 3.93473), (3.0, 16, 3.5667), (5.0, 16, 4.6506), (10.0, 16, 6.9584)]


def _z_inputs(dtype):
    z = np.concatenate([I.normals(200000, dtype=np.float64),
                        np.linspace(-9, 9, 20001),
                        [0.0, -0.0, 1e-300, 3.93473, -3.93473, 12.0, -20.0, 37.0, np.inf, -np.inf, np.nan]])
    return z.astype(dtype)


@pytest.mark.parametrize("nu,K,zstar", STUDENT)
@pytest.mark.parametrize("dtype,bar", [(np.float64, 2.0), (np.float32, 4.0)])
def test_student_parity(nu, K, zstar, dtype, bar):
    z = _z_inputs(dtype)
    g = Q.qm_recycle_normal_to_t(torch.from_numpy(z).cuda(), nu, K, zstar).cpu().numpy()
    ref = O.student_map(z.astype(np.float64), nu, K, zstar)
    err = ulp_errors(g, ref, dtype)
    assert err.max() <= bar, summary(err)


def test_student_default_crossover_is_the_papers():
    z = _z_inputs(np.float64)
    a = Q.qm_recycle_normal_to_t(torch.from_numpy(z).cuda(), 4.0, 10, 0.0)
    b = Q.qm_recycle_normal_to_t(torch.from_numpy(z).cuda(), 4.0, 10, 3.93473)
    assert torch.equal(a.nan_to_num(), b.nan_to_num())


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_moments(dtype):
    x = I.normals((1 << 22) + 3, dtype=dtype)
    ws = Q.qm_moments(torch.from_numpy(x).cuda(), 4)
    S = ws[:4].cpu().numpy()
    ref = O.moments(x, 4).astype(np.float64)
    absum = np.array([np.sum(np.abs(x.astype(np.float64)) ** k) for k in range(1, 5)])
    # fp64 accumulation, fixed tree of depth ~log2(n): |error| <= c log2(n) eps sum|x|^k
    assert np.all(np.abs(S - ref) <= 64 * np.finfo(np.float64).eps * absum)
    ws2 = Q.qm_moments(torch.from_numpy(x).cuda(), 4)
    assert torch.equal(ws[:4], ws2[:4])          # deterministic
