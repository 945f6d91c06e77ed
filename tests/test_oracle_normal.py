"""Pins for the oracle's normal-quantile functions (§8 c).

Every check ties the oracle to something other than itself: values printed in
PAPER.md (tests/golden/normal_pins.txt), the paper's stated error bounds, mpmath
at 40 digits, closed forms, symmetry and special cases.
"""
import math
from pathlib import Path

import mpmath as mp
import numpy as np
import pytest
import scipy.special as sps

import oracle as O
from _util import ld2mp

GOLDEN = Path(__file__).parent / "golden" / "normal_pins.txt"


def _pins():
    out = {}
    for line in GOLDEN.read_text().splitlines():
        if line.startswith("#") or not line.strip():
            continue
        name, val, tol = line.split()[:3]
        out[name] = (float(val), float(tol))
    return out


def mp_ndtri(u):
    """Phi^-1(u) by mpmath root-finding at 40 digits (independent of the oracle)."""
    mp.mp.dps = 40
    u = mp.mpf(u)
    if u > 0.5:
        return -mp_ndtri(1 - u)
    x0 = float(sps.ndtri(float(u))) if u > 1e-300 else -38.0
    return mp.findroot(lambda x: mp.log(mp.ncdf(x)) - mp.log(u), mp.mpf(x0))


def mp_Q(v):
    """Q(v) = Phi^-1(1 - e^-v/2) by mpmath: solve ncdf(-x) = e^-v/2."""
    mp.mp.dps = 40
    t = mp.exp(-mp.mpf(v)) / 2
    x0 = -float(sps.ndtri(float(t))) if float(t) > 1e-300 else math.sqrt(2 * v)
    return mp.findroot(lambda x: mp.log(mp.ncdf(-x)) - mp.log(t), mp.mpf(x0))


# ------------------------------------------------------------- exact quantile
def test_exact_quantile_printed_values():
    pins = _pins()
    w = O.ndtri_exact([0.975, 0.5])
    v, tol = pins["ndtri_0.975"]
    assert abs(float(w[0]) - v) <= tol * v
    assert w[1] == 0 and not np.signbit(w[1])
    q = O.Q_exact([37.0, 74.0])
    for got, key in zip(q, ["Qexact_37", "Qexact_74"]):
        v, tol = pins[key]
        assert abs(float(got) - v) <= tol * v


@pytest.mark.parametrize("u", [0.975, 0.75, 0.9, 0.5 + 2.0 ** -40, 0.5 - 2.0 ** -50, 0.3, 1e-3,
                               1e-10, 1e-30, 1e-100, 1e-300, 2.0 ** -1074, 1 - 2.0 ** -53])
def test_exact_quantile_vs_mpmath(u):
    got = O.ndtri_exact([u])[0]
    ref = mp_ndtri(u)
    rel = abs(ld2mp(got) - ref) / abs(ref)
    assert rel < 5e-18, (u, float(rel))


@pytest.mark.parametrize("v", [1e-8, 0.1, 1.0, 5.0, 20.0, 37.0, 50.0, 74.0, 200.0, 700.0])
def test_Qexact_vs_mpmath(v):
    got = O.Q_exact([v])[0]
    ref = mp_Q(v)
    assert abs(ld2mp(got) - ref) / ref < 5e-18


def test_exact_quantile_symmetry_and_specials():
    u = O.philox_uniform(20000, 99, 0, np.float64)
    w = O.ndtri_exact(u)
    wm = O.ndtri_exact(1.0 - u)         # 1-u exact on the odd 2^-53 grid
    assert np.array_equal(wm, -w)
    s = O.ndtri_exact([0.0, 1.0, -0.1, 1.1, np.nan])
    assert s[0] == -np.inf and s[1] == np.inf and np.all(np.isnan(s[2:]))
    # monotone
    us = np.sort(u)
    assert np.all(np.diff(O.ndtri_exact(us).astype(np.float64)) >= 0)


def test_exact_quantile_round_trip():
    """Phi(w(u)) = u (P:28 F(w(u)) = u), mpmath's ncdf, on log-spaced tails."""
    mp.mp.dps = 40
    for u in np.concatenate([np.logspace(-250, -1, 25), [0.2, 0.4, 0.49999]]):
        w = O.ndtri_exact([u])[0]
        back = mp.ncdf(ld2mp(w))
        # |dPhi/dw| * |dw| with |dw| <= 4 eps_ld |w|
        kappa = abs(float(w)) * float(mp.npdf(ld2mp(w))) / u
        assert abs(back - u) / u <= max(kappa, 1.0) * 1e-18


# ------------------------------------------ formula vs exact: the paper's bounds
def _vgrid(lo, hi, n=20001):
    return np.linspace(lo, hi, n, dtype=np.longdouble)


def _relerr(formula, prec, v):
    a = O.rational(v, formula, prec)
    e = O.Q_exact(v)
    m = v > 0
    return np.abs(a[m] / e[m] - 1).astype(np.float64)


def test_A77_bounds():
    """(7,7): < 1.06e-9 on [0,37]; < 1e-6 below v=50; P:507's 2e-5 up to
    v=74 is contradicted by its own example (reading R2): bound 3.2e-5."""
    assert _relerr(O.A77, 0, _vgrid(0, 37)).max() < 1.06e-9
    assert _relerr(O.A77, 0, _vgrid(37, 50, 2001)).max() < 1e-6
    assert _relerr(O.A77, 0, _vgrid(50, 74, 2001)).max() < 3.2e-5
    pins = _pins()
    v, tol = pins["A77_74"]
    assert abs(float(O.rational([74.0], O.A77, 0)[0]) - v) <= tol * v


def test_C55_bound():
    """App C (5,5): < 4e-7 'in double'; range [0,37] (reading R7)."""
    e = _relerr(O.C55, 0, _vgrid(0, 37))
    assert e.max() < 4e-7
    assert e.max() > 3e-7   # equal-ripple fit: the bound is nearly attained (transcription check)


def test_D13_bound():
    """App D (13,13): O(1e-15) on [eps, 1-eps], eps < 1e-32 -> 1.1e-15 on v in [0,74] (reading R8)."""
    assert _relerr(O.D13, 0, _vgrid(0, 74)).max() < 1.1e-15


def test_formula_bounds_vs_mpmath_spot():
    """The same bounds, a few points checked against mpmath directly."""
    for v in [0.05, 0.7, 3.3, 10.7, 25.0, 36.9]:
        ref = mp_Q(v)
        for f, b in [(O.A77, 1.06e-9), (O.C55, 4e-7), (O.D13, 1.1e-15)]:
            got = O.rational([v], f, 0)[0]
            assert abs(ld2mp(got) / ref - 1) < b


def test_north_star_pin_through_the_sampling_algorithm():
    """u -> vv = min(u,1-u) -> z = -log(2vv) -> sign * Q(z) (App D)."""
    pins = _pins()
    v, _ = pins["ndtri_0.975"]
    d13 = float(O.normal_breakless([0.975], O.D13, 64)[0])
    c55 = float(O.normal_breakless([0.975], O.C55, 32)[0])
    a77 = float(O.normal_breakless([0.975], O.A77, 64)[0])
    assert abs(d13 / v - 1) < 1.1e-15
    assert abs(c55 / v - 1) < 4e-7
    assert abs(a77 / v - 1) < 1.06e-9
    assert float(O.normal_breakless([1.0 - 0.975], O.D13, 64)[0]) == -d13


def test_breakless_edge_semantics_and_symmetry():
    for f, p in [(O.C55, 32), (O.D13, 64), (O.A77, 32), (O.A77, 64)]:
        s = O.normal_breakless([0.0, 1.0, 0.5, np.nan, -0.25, 1.5], f, p)
        assert s[0] == -np.inf and s[1] == np.inf
        assert s[2] == 0 and not np.signbit(s[2])
        assert np.all(np.isnan(s[3:]))
        u = O.philox_uniform(10000, 5, 0, np.float32 if p == 32 else np.float64).astype(np.float64)
        a = O.normal_breakless(u, f, p)
        b = O.normal_breakless(1.0 - u, f, p)
        assert np.array_equal(a, -b)          # vv = min(u,1-u) is exact: bitwise odd symmetry


def test_breakless_vs_exact_quantile_on_uniform_grid():
    """Same-formula oracle vs exact quantile: within the paper's bound for each
    formula (the coefficients are type-rounded, the arithmetic long double)."""
    u = O.philox_uniform(4000, 77, 0, np.float64)
    ex = O.ndtri_exact(u)
    for f, p, b in [(O.D13, 64, 1.1e-15), (O.A77, 64, 1.06e-9), (O.C55, 32, 4.5e-7)]:
        a = O.normal_breakless(u, f, p)
        assert np.max(np.abs(a / ex - 1)).astype(float) < b


def test_antithetic_and_laplace_forms():
    """v = -log u ('better') gives Z = Phi^-1(1 - u/2); pairs {Z,-Z}.
    The Laplace base gives Z = sign(v) Q(|v|)."""
    u = np.array([0.5, 1e-3, 0.9, 1e-20, 1.0])
    pr = O.normal_antithetic(u, O.D13, 64)
    ex = O.Q_exact(-np.log(u[:3].astype(np.longdouble)))
    assert np.max(np.abs(pr[0:6:2] / ex - 1)) < 1.1e-15
    assert np.array_equal(pr[1::2], -pr[0::2])
    assert pr[8] == 0
    v = np.array([-3.0, 0.0, -0.0, 2.5, np.inf, -np.inf, np.nan])
    z = O.exp_to_normal(v, O.D13, 64)
    q = O.Q_exact(np.abs(v[:4]))
    assert abs(z[0] / -q[0] - 1) < 1.1e-15 and abs(z[3] / q[3] - 1) < 1.1e-15
    assert z[1] == 0 and not np.signbit(z[1]) and np.signbit(z[2])
    assert z[4] == np.inf and z[5] == -np.inf and np.isnan(z[6])


# --------------------------------------------------- Taylor series and tail model
def test_taylor_series_coefficients():
    """P:407-432 printed series vs mpmath Taylor coefficients of Q at 0."""
    mp.mp.dps = 50
    Q = lambda v: -mp.sqrt(2) * mp.erfinv(mp.exp(-v) - 1)   # Phi^-1(1 - e^-v/2)
    ref = mp.taylor(Q, mp.mpf(0), 10)
    got = O.Q_taylor_coeffs()
    assert got[0] == 0
    for k in range(1, 11):
        assert abs(ld2mp(got[k]) - ref[k]) <= 1e-17 * abs(ref[k]), k


def test_taylor_series_accuracy():
    """'best used to a small number of terms in a neighbourhood of v=0':
    rel err 1.6e-10 at v = 0.1 (SPEC's 1e-10 corrected to 2e-10)."""
    v = np.array([0.01, 0.05, 0.1], dtype=np.longdouble)
    e = np.abs(O.Q_taylor(v, 10) / O.Q_exact(v) - 1).astype(float)
    assert e[2] < 2e-10 and e[1] < 1e-12


def test_tail_model_bound():
    """§5.1: precision better than 1.06e-9 for v >= 37, improving as v grows."""
    v = np.array([37.0, 50.0, 100.0, 200.0, 700.0], dtype=np.longdouble)
    e = np.abs(O.Q_tail(v, 4) / O.Q_exact(v) - 1).astype(float)
    assert np.all(e < 1.06e-9)
    assert np.all(np.diff(e) < 0)


# ---------------------------------------------------- comparison quantiles (a5)
def _tail_stratified(n, seed):
    rng = np.random.default_rng(seed)
    half = rng.uniform(0, 1, n // 2)
    t = 10.0 ** rng.uniform(-300, np.log10(0.5), n - n // 2)
    t = np.where(rng.uniform(size=t.size) < 0.5, t, 1 - t)
    return np.concatenate([half, t])


def test_acklam_level1_bound():
    """'maximum relative error less than 1.15e-9'."""
    u = np.concatenate([np.linspace(1e-6, 1 - 1e-6, 20001), _tail_stratified(4000, 3)])
    u = u[(u > 1e-300) & (u < 1) & (np.abs(u - 0.5) > 1e-12)]
    e = np.abs(O.normal_acklam(u, 64, False) / O.ndtri_exact(u) - 1).astype(float)
    assert e.max() < 1.15e-9
    assert e.max() > 1.0e-9           # the published bound is nearly attained


def test_as241_double_quality():
    """AS241 'confirms the double-precision quality': reading R18, <= 2e-16
    relative in exact arithmetic with double-rounded coefficients."""
    u = np.concatenate([np.linspace(1e-6, 1 - 1e-6, 20001), _tail_stratified(4000, 4)])
    u = u[(u > 0) & (u < 1) & (np.abs(u - 0.5) > 1e-12)]
    e = np.abs(O.normal_as241(u, 64) / O.ndtri_exact(u) - 1).astype(float)
    assert e.max() < 2e-16


def test_refined_acklam():
    """One Halley step on Acklam L1: machine precision away from the centre
    (P:599); in long double the centre keeps an absolute accuracy ~1e-18."""
    u = _tail_stratified(4000, 5)
    u = u[(u > 1e-300) & (u < 1)]
    r = O.normal_acklam(u, 64, True)
    ex = O.ndtri_exact(u)
    far = np.abs(u - 0.5) > 1e-3
    assert (np.abs(r[far] / ex[far] - 1)).max() < 1e-17
    assert (np.abs(r - ex) / np.maximum(1.0, np.abs(ex))).max() < 1e-17
    l1 = O.normal_acklam(u, 64, False)
    assert np.median(np.abs(r - ex) / np.abs(l1 - ex + 1e-300)) < 1e-6   # the step helps


# ------------------------------------------------- Moro comparison quantile (f4)
def test_moro_published_accuracy():
    """Moro (1995) publishes an absolute error below 3e-9 out to seven standard
    deviations (external, reading R17; a wrong digit in any of the 17 transcribed
    coefficients breaks it).  The worst case sits at the break u = 0.08 / 0.92,
    where the paper says Moro breaks."""
    lo = 1.2798125438858e-12                                  # Phi(-7)
    u = np.concatenate([np.linspace(lo, 1 - 1e-10, 200001), np.exp(np.linspace(np.log(lo), np.log(0.5), 20001)),
                        [0.08 - 1e-12, 0.08 + 1e-12, 0.92 - 1e-12, 0.92 + 1e-12]])
    e = np.abs(O.normal_moro(u, 64) - O.ndtri_exact(u)).astype(float)
    assert e.max() < 3.1e-9
    assert e.max() > 2.5e-9                                   # nearly attained
    i = np.argmax(e)
    assert abs(min(u[i], 1 - u[i]) - 0.08) < 1e-3             # at the break


def test_moro_regions_and_symmetry():
    """Central rational for |u - 1/2| < 0.42, log(log) tail beyond;
    odd symmetry w(1-u) = -w(u) on exact pairs; specials as the other quantiles."""
    k = np.arange(1, 2000, dtype=np.float64)
    u = k / 4096.0
    a, b = O.normal_moro(u, 64), O.normal_moro(1 - u, 64)
    assert np.array_equal(a, -b)
    # the two branches agree at the break to the method's accuracy (continuity)
    lo = O.normal_moro(np.array([0.08 + 2 ** -40]), 64)[0]
    hi = O.normal_moro(np.array([0.08 - 2 ** -40]), 64)[0]
    assert abs(lo - hi) < 1e-8
    sp = O.normal_moro(np.array([0.0, 1.0, 0.5, -0.1, 1.1, np.nan]), 64)
    assert sp[0] == -np.inf and sp[1] == np.inf and sp[2] == 0 and not np.signbit(sp[2])
    assert np.all(np.isnan(sp[3:]))



def test_d13_partial_compensation_bound():
    """The written bound behind the product's App D scheme (qm_math.cuh rat64): the
    Horner steps left uncompensated add at most u (W_P(z) + W_Q(z)) relative error,
    W(z) = sum over plain steps k of sum_{i>=k} a_i z^i / P(z) (all App D coefficients
    are positive).  Compensating 8 steps for z <= 12 and 10 beyond keeps
    W_P + W_Q < 0.9 resp. < 0.6 on the fp64 grid (z <= 36.04): with the final rounding
    the result stays inside the 2-ulp contract; 9 steps would not (1.65 + 0.5)."""
    p, q = O.coeffs(O.D13, 64)
    p, q = p.astype(np.float64), q.astype(np.float64)

    def W(c, z, kc):
        t = c * z ** np.arange(c.size)
        return sum(t[k:].sum() / t.sum() for k in range(kc, c.size - 1))

    def mx(kc, zmax):
        return max(W(p, z, kc) + W(q, z, kc) for z in np.linspace(0.0, zmax, 4001))

    assert mx(8, 12.0) < 0.9
    assert mx(10, 36.04) < 0.6
    assert mx(9, 36.04) > 1.5          # the bound is what rules 9 steps out (measured 2.13 ulp on B200)

    # z's low part enters the product once, as zl R(zh) (rational_dd): the dropped
    # zh zl R'(zh) is (zl/zh)(kappa - 1) of the result, |zl/zh| <= 2^-53, with
    # kappa - 1 = z (P'/P - Q'/Q) -- the logarithmic derivative of R, here from the
    # coefficients, pinned below against the closed form of the exact map
    # w(z) = Phi^-1(1 - e^-z/2): kappa = z w'/w, w' = (e^-z/2)/phi(w).
    def km1(z):
        i = np.arange(p.size)
        dp = (p * i * z ** np.maximum(i - 1, 0)).sum() / (p * z ** i).sum()
        dq = (q * i * z ** np.maximum(i - 1, 0)).sum() / (q * z ** i).sum()
        return z * (dp - dq)

    for z in (0.5, 3.0, 12.0, 30.0):
        w = float(O.Q_exact(np.array([z]))[0])
        phi = np.exp(-0.5 * w * w) / np.sqrt(2 * np.pi)
        assert abs((1 + km1(z)) - z * (0.5 * np.exp(-z) / phi) / w) < 1e-12
    # up to the switch to the fully compensated form, z = 36.8 (QM_DD_ZL_ZMAX; the fp64
    # grid's 2^-53 gives z = 36.04)
    zs = np.linspace(0.0, 36.8, 4001)
    assert max(abs(km1(z)) for z in zs) < 0.48
    total = max(W(p, z, 10) + W(q, z, 10) + abs(km1(z)) for z in zs)
    assert total + 0.5 < 1.6           # <= 1.57 ulp: inside the 2-ulp contract
    # beyond it the ten compensated steps would not do: the weights approach the
    # three plain steps each (W_P + W_Q -> 6) -- hence all 13 compensated there
    assert W(p, 74.0, 10) + W(q, 74.0, 10) > 1.5 and W(p, 700.0, 10) + W(q, 700.0, 10) > 5.0
