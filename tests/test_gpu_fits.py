"""GPU parity of rows f3/f4 through the C ABI: the (12,12) and (8,8) single-patch
rationals, the two-region variant and Moro's quantile,
element by element against the oracle's long-double evaluation of the same
formula (4 ulp fp32, 2 ulp fp64)."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import inputs as I
from _parity import summary, ulp_errors

pytestmark = pytest.mark.gpu
Q = pytest.importorskip("paper_0901_0638_b200")

CASES = [  # dtype, alg, oracle formula, coefficient precision, ulp bar
    (np.float64, Q.BREAKLESS1212, O.F1212, 64, 2.0),
    (np.float64, Q.BREAKLESS88, O.F88, 64, 2.0),
    (np.float32, Q.BREAKLESS88, O.F88, 32, 4.0),
]


def _gpu(x_np, alg):
    return Q.qm_normal_quantile(torch.from_numpy(np.ascontiguousarray(x_np)).cuda(), alg=alg).cpu().numpy()


def _deep(dtype, n=20000, seed=7):
    rng = np.random.default_rng(seed)
    lo = -37 if dtype == np.float32 else -300
    t = 10.0 ** rng.uniform(lo, -1, n)
    return np.concatenate([t, 1 - t[: n // 10]]).astype(dtype)


@pytest.mark.parametrize("n", [(1 << 20) + 37, (1 << 23) + 37])
@pytest.mark.parametrize("dtype,alg,formula,prec,bar", CASES)
def test_single_patch_fits(dtype, alg, formula, prec, bar, n):
    u = np.concatenate([I.mixed_uniforms(n, dtype=dtype), _deep(dtype)])
    g = _gpu(u, alg)
    err = ulp_errors(g, O.normal_breakless(u.astype(np.float64), formula, prec), dtype)
    assert err.max() <= bar, summary(err)


def test_fp32_88_covers_the_fp32_range():
    """(8,8) keeps ~6e-10 out to v = 74: fp32 inputs down to u ~ 1e-32 stay
    within a few fp32 ulp of the exact quantile, where App C (v <= 37) has left its range."""
    u = np.array([1e-32, 1e-30, 1e-25, 1e-20, 3e-18], dtype=np.float32)
    g = _gpu(u, Q.BREAKLESS88).astype(np.float64)
    ex = O.ndtri_exact(u.astype(np.float64)).astype(np.float64)
    assert np.all(np.abs(g / ex - 1) < 4 * 2.0 ** -24)


def _two_region_ref(u):
    """Oracle value; within 1e-6 of the break v = 10 either region is correct (the
    kernel's fp32 z and the oracle's exact z can fall on different sides)."""
    ref = O.normal_breakless(u.astype(np.float64), O.TWO_REGION, 32)
    vv = np.minimum(u.astype(np.float64), 1 - u.astype(np.float64))
    with np.errstate(divide="ignore"):
        v = -np.log(2 * vv)
    near = np.abs(v - 10.0) < 1e-5
    alt = np.where(v < 10, O.normal_breakless(u.astype(np.float64), O.C55, 32),
                   O.normal_breakless(u.astype(np.float64), O.F44, 32))
    return ref, alt, near


@pytest.mark.parametrize("n", [(1 << 20) + 37, (1 << 23) + 37])
def test_two_region_fp32(n):
    u = np.concatenate([I.mixed_uniforms(n, dtype=np.float32), _deep(np.float32),
                        (np.exp(-10.0) / 2 * (1 + np.linspace(-1e-4, 1e-4, 2001))).astype(np.float32)])
    g = _gpu(u, Q.TWO_REGION)
    ref, alt, near = _two_region_ref(u)
    err = np.minimum(ulp_errors(g, ref, np.float32), np.where(near, ulp_errors(g, alt, np.float32), np.inf))
    assert err.max() <= 4.0, summary(err)


def test_two_region_fp32_grid_and_fast_path():
    """The whole fp32 odd grid; and warps entirely below the break give exactly the
    short (4,4) rational (the vote's fast path), above it App C."""
    k = np.arange(1 << 22, dtype=np.float64)
    lo = np.ldexp(2 * k + 1, -24).astype(np.float32)           # (0, 1/2)
    u = np.concatenate([lo, (1 - lo.astype(np.float64)).astype(np.float32)])
    g = _gpu(u, Q.TWO_REGION)
    ref, alt, near = _two_region_ref(u)
    err = np.minimum(ulp_errors(g, ref, np.float32), np.where(near, ulp_errors(g, alt, np.float32), np.inf))
    assert err.max() <= 4.0, summary(err)
    assert np.array_equal(g[lo.size:], -g[:lo.size])             # odd symmetry
    # samples far from the break agree bitwise with a run where every warp is fast
    central = u[(u > 0.01) & (u < 0.99)][: 1 << 16]
    assert np.array_equal(_gpu(central, Q.TWO_REGION), g[(u > 0.01) & (u < 0.99)][: 1 << 16])


def test_moro_specials_and_break():
    u = np.array([0.0, 1.0, 0.5, -1.0, 2.0, np.nan, 0.08, 0.92, 1e-300, 1 - 2 ** -53, 5e-324])
    g = _gpu(u, Q.MORO)
    ref = O.normal_moro(u, 64)
    err = ulp_errors(g, ref, np.float64)
    assert err.max() <= 2.0, summary(err)
    assert g[2] == 0 and not np.signbit(g[2])
