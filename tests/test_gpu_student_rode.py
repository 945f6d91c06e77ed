"""GPU parity of the Student map by the "purely numerical method" of §3.6
(P:282-283): the Recycling ODE solved on the host into a table,
sampled by quintic Hermite interpolation in the kernel (row a6 by the RODE;
SURVEY E14).  Reference: the oracle's exact map F_n^-1(Phi(z)) (inverse
incomplete beta, pinned in test_oracle_student.py).
Bar (fp64): 4e-15 + 16 eps (1 + kappa(z)), kappa = |z t'/t| the map's condition
number (_parity.student_rode_bar): the table nodes are within ~1e-16 and the
quintic's error is < 5e-15, and the roundings of the node coordinate
s = n (|z|/4.5)^(1/4) (centre) or of the interpolated log|t| (|z| > 9) are amplified
by kappa (<= 40 on |z| <= 6, ~z^2/nu in the tail).  The paper's own claim is
5e-8 on |z| < 6.  fp32: 1 ulp (a double result within ~1e-13 rounded to float)."""
import numpy as np
import pytest
import torch

import oracle as O
from _parity import student_rode_bar, ulp_errors

pytestmark = pytest.mark.gpu
Q = pytest.importorskip("paper_0901_0638_b200.qm")


def _z(n, seed=3):
    rng = np.random.default_rng(seed)
    edges = [1e-300, -5e-324, 1e-10, 2.0, -2.0, np.nextafter(2.0, 0), 6.0, -6.0, np.nextafter(6.0, 9), 1.76, -1.77,
             10.0, -15.5, 25.0, 38.4, -38.46, 38.5]
    return np.concatenate([rng.standard_normal(n), rng.uniform(-38.4, 38.4, n // 4), edges])


def _bar(z, ex, nu):
    return student_rode_bar(z, ex, nu)


@pytest.mark.parametrize("nu", [1.0, 1.5, 3.0, 4.0, 5.0, 10.0, 30.0, 200.0])
def test_student_rode_vs_exact_map(nu):
    tab = Q.qm_normal_target_table(Q.STUDENT, [nu])
    z = _z(3000)
    g = Q.qm_recycle_normal_to_t_rode(torch.from_numpy(z).cuda(), tab).cpu().numpy()
    ex = O.student_exact(z, nu).astype(np.float64)
    fin = np.isfinite(ex) & (z != 0)
    rel = np.abs(g[fin] / ex[fin] - 1)
    bar = _bar(z[fin], ex[fin], nu)
    assert np.all(rel <= bar), (np.max(rel / bar), z[fin][np.argmax(rel / bar)])
    # beyond the double range (nu = 1 past |z| ~ 37.5): +-inf like the exact value
    assert np.array_equal(g[~np.isfinite(ex)], ex[~np.isfinite(ex)])
    z32 = z.astype(np.float32)
    g32 = Q.qm_recycle_normal_to_t_rode(torch.from_numpy(z32).cuda(), tab).cpu().numpy()
    ex32 = O.student_exact(z32.astype(np.float64), nu)
    ok = np.isfinite(ex32.astype(np.float32))
    assert ulp_errors(g32[ok], ex32[ok], np.float32).max() <= 1.0
    assert np.array_equal(g32[~ok], ex32[~ok].astype(np.float32))


def test_student_rode_specials_and_symmetry():
    tab = Q.qm_normal_target_table(Q.STUDENT, [4.0])
    z = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 50.0, -60.0])
    g = Q.qm_recycle_normal_to_t_rode(torch.from_numpy(z).cuda(), tab).cpu().numpy()
    assert g[0] == 0 and not np.signbit(g[0]) and g[1] == 0 and np.signbit(g[1])
    assert g[2] == np.inf and g[3] == -np.inf and np.isnan(g[4])
    # beyond the table (|z| > 38.5, no double uniform gets there): log-linear, finite, monotone
    assert np.isfinite(g[5]) and g[5] > 0 and g[6] < 0
    zz = np.random.default_rng(2).standard_normal(10000)
    a = Q.qm_recycle_normal_to_t_rode(torch.from_numpy(zz).cuda(), tab).cpu().numpy()
    b = Q.qm_recycle_normal_to_t_rode(torch.from_numpy(-zz).cuda(), tab).cpu().numpy()
    assert np.array_equal(a, -b)


def test_student_rode_agrees_with_series_composite():
    """The two recyclings of §3 side by side on the paper's case n = 4: the series
    composite (K = 10, z* = 3.93473) is within its printed 1.4e-5 of the
    RODE map."""
    tab = Q.qm_normal_target_table(Q.STUDENT, [4.0])
    z = torch.from_numpy(np.random.default_rng(8).standard_normal(1 << 16) * 2.0).cuda()
    a = Q.qm_recycle_normal_to_t_rode(z, tab)
    b = Q.qm_recycle_normal_to_t(z, 4.0, K=10)
    nz = z != 0
    assert float(((b[nz] / a[nz]) - 1).abs().max()) < 1.4e-5


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_student_rode_pipeline_equals_ldg_kernel(dtype):
    """2^23 + 37 normal samples: whole tiles through the TMA pipeline (3600 staged
    centre nodes per side), the rest and a misaligned view through the LDG kernel
    (4097 staged): bitwise equal; sampled parity with the exact map."""
    tab = Q.qm_normal_target_table(Q.STUDENT, [3.0])
    z = np.random.default_rng(11).standard_normal((1 << 23) + 37)
    z[:8] = [0.0, -0.0, np.inf, -np.inf, np.nan, 1.76, 7.5, -9.0]
    z = z.astype(dtype)
    zd = torch.from_numpy(np.concatenate([[dtype(0.5)], z]).astype(dtype)).cuda()
    tiled = Q.qm_recycle_normal_to_t_rode(zd[1:].clone(), tab)
    ldg = Q.qm_recycle_normal_to_t_rode(zd[1:], tab)
    assert torch.equal(tiled.nan_to_num(), ldg.nan_to_num()) and torch.equal(tiled.isnan(), ldg.isnan())
    idx = np.concatenate([np.arange(5, 8), np.random.default_rng(4).choice(z.size - 8, 4096, replace=False) + 8])
    g = tiled.cpu().numpy()[idx].astype(np.float64)
    ex = O.student_exact(z[idx].astype(np.float64), 3.0).astype(np.float64)
    if dtype == np.float64:
        assert np.all(np.abs(g / ex - 1) <= _bar(z[idx].astype(np.float64), ex, 3.0))
    else:
        assert ulp_errors(g.astype(np.float32), ex, np.float32).max() <= 1.0
