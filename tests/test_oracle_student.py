"""Pins for the oracle's normal -> Student-t recycling map and
moment sums (row a8).

The recurrence is pinned by the eleven coefficients the paper prints for n = 4
(tests/golden/student_n4_coeffs.txt) and by the independent closed
forms for c_1, c_2 and gamma.  The exact
map is pinned by closed-form Student quantiles (n = 1, 2, 4) and by mpmath.
"""
from pathlib import Path

import mpmath as mp
import numpy as np
import pytest

import oracle as O
from _util import ld2mp

GOLD = Path(__file__).parent / "golden" / "student_n4_coeffs.txt"


def _printed_n4():
    return [mp.mpf(l.strip()) for l in GOLD.read_text().splitlines()
            if l.strip() and not l.startswith("#")]


def test_gamma_printed_and_closed_form():
    mp.mp.dps = 30
    g4 = ld2mp(O.student_gamma(4.0))
    assert abs(g4 - mp.mpf("1.06384608107048714")) <= 5e-18           # P:250 (printed to 18 digits)
    assert abs(g4 - mp.mpf(4) / 3 * mp.sqrt(2 / mp.pi)) < 1e-18        # P:250 closed form
    for n in [1.0, 2.5, 3.0, 7.0, 30.0]:
        ref = mp.sqrt(n / 2) * mp.gamma(n / 2) / mp.gamma((n + 1) / 2)
        assert abs(ld2mp(O.student_gamma(n)) / ref - 1) < 1e-17
    # the 1/n expansion of P:233-236 at n = 1e4 (next term 399/8192 n^-5 ~ 5e-22)
    n = 1e4
    ser = 1 + 1 / (4 * n) + 1 / (32 * n ** 2) - 5 / (128 * n ** 3) - 21 / (2048 * n ** 4)
    assert abs(float(O.student_gamma(n)) - ser) < 1e-15


def test_recurrence_reproduces_printed_n4_coefficients():
    """All 11 printed c_k for n = 4 to 1e-15 relative."""
    c = O.student_coeffs(4.0, 10)
    for k, ref in enumerate(_printed_n4()):
        assert abs(ld2mp(c[k]) / ref - 1) < 1e-15, k


@pytest.mark.parametrize("n", [1.0, 2.0, 4.0, 10.0, 100.0])
def test_recurrence_vs_closed_forms_c1_c2(n):
    """c_1 = ((n+1)g^3 - n g)/(6n), c_2 = ((7n^2+8n+1)g^5 - (10n^2+10n)g^3 + 3n^2 g)/(120 n^2)."""
    mp.mp.dps = 30
    g = mp.sqrt(mp.mpf(n) / 2) * mp.gamma(mp.mpf(n) / 2) / mp.gamma((mp.mpf(n) + 1) / 2)
    c1 = ((n + 1) * g ** 3 - n * g) / (6 * n)
    c2 = ((7 * n * n + 8 * n + 1) * g ** 5 + (-10 * n * n - 10 * n) * g ** 3 + 3 * n * n * g) / (120 * n * n)
    c = O.student_coeffs(n, 4)
    assert abs(ld2mp(c[1]) / c1 - 1) < 1e-14
    assert abs(ld2mp(c[2]) / c2 - 1) < 1e-13


def test_recurrence_conditioning_documented():
    """The long-double recurrence loses digits exponentially (why the oracle uses mpmath)."""
    hi = O.student_coeffs(10.0, 16)
    lo = O.student_coeffs_ld(10.0, 16)
    assert abs(float(lo[16] / hi[16] - 1)) > 1e-12
    assert abs(float(lo[1] / hi[1] - 1)) < 1e-17


def test_large_n_limit_is_identity():
    """n -> infinity: Q'' + vQ' = Q(Q')^2 has the solution Q = v."""
    c = O.student_coeffs(1e8, 16)
    assert abs(float(c[0]) - 1) < 1e-8 and np.all(np.abs(c[1:].astype(float)) < 1e-6)


# --------------------------------------------------------------- exact map
def _mp_t_from_tail(n, tail):
    """closed-form Student quantile from the upper-tail mass (n = 1, 2, 4)."""
    if n == 1:
        return mp.cot(mp.pi * tail)                    # tan(pi(u - 1/2)), u = 1 - tail
    if n == 2:                                          # (2u-1)/sqrt(2u(1-u)), u = 1 - tail
        return (1 - 2 * tail) / mp.sqrt(2 * tail * (1 - tail))
    if n == 4:                                          # Shaw's form (SPEC S:~)
        a = 4 * tail * (1 - tail)
        q = mp.cos(mp.acos(mp.sqrt(a)) / 3) / mp.sqrt(a)
        return 2 * mp.sqrt(q - 1)
    raise ValueError


@pytest.mark.parametrize("n", [1.0, 2.0, 4.0])
def test_exact_map_vs_closed_forms(n):
    mp.mp.dps = 40
    z = np.concatenate([np.linspace(0.01, 8.3, 40), [1e-8, 12.0, 20.0]])
    t = O.student_exact(z, n)
    for zi, ti in zip(z, t):
        ref = _mp_t_from_tail(n, mp.ncdf(-mp.mpf(zi)))
        assert abs(ld2mp(ti) / ref - 1) < 3e-17, (n, zi)


@pytest.mark.parametrize("n", [3.0, 5.0, 10.0, 2.5])
def test_exact_map_vs_mpmath_betainc(n):
    """P(T > t) = 1/2 I_{n/(n+t^2)}(n/2, 1/2) evaluated by mpmath at the oracle's t."""
    mp.mp.dps = 40
    z = np.array([1e-6, 0.3, 1.0, 2.5, 4.0, 6.0, 8.2])
    t = O.student_exact(z, n)
    for zi, ti in zip(z, t):
        tt = ld2mp(ti)
        up = mp.betainc(n / 2, 0.5, 0, n / (n + tt * tt), regularized=True) / 2
        tgt = mp.ncdf(-mp.mpf(zi))
        dens = mp.gamma((n + 1) / 2) / (mp.sqrt(n * mp.pi) * mp.gamma(n / 2)) * (1 + tt * tt / n) ** (-(n + 1) / 2)
        # |dt| = |dP| / f(t)
        assert abs(up - tgt) / dens <= 3e-18 * max(1, abs(tt)), (n, zi)


def test_exact_map_symmetry_and_specials():
    z = np.array([-2.0, 2.0, 0.0, -0.0, np.inf, -np.inf, np.nan])
    t = O.student_exact(z, 5.0)
    assert t[0] == -t[1] and t[2] == 0 and np.signbit(t[3])
    assert t[4] == np.inf and t[5] == -np.inf and np.isnan(t[6])


# ---------------------------------------------- composite map: paper's claims
def test_n4_crossover_is_printed_value():
    """'The optimal crossover is then in fact at z=3.93473': the first root of
    central(z) = tail(z) (reading R13)."""
    assert abs(O.student_crossover(4.0, 10) - 3.93473) < 5e-6


def test_n4_composite_accuracy():
    """central < 2e-5 on |z| < 4; composite < 1.4e-5 over the range."""
    z = np.linspace(1e-4, 12.0, 12001)
    ex = O.student_exact(z, 4.0)
    cen, tl = O.student_branches(z, 4.0, 10)
    m = z < 4
    assert np.max(np.abs(cen[m] / ex[m] - 1)).astype(float) < 2e-5
    comp = O.student_map(z, 4.0, 10, 3.93473)
    assert np.max(np.abs(comp / ex - 1)).astype(float) < 1.4e-5
    # the crossover is near-optimal: shifting it by +-0.1 does not help by > 10% (SPEC acc. 5)
    e0 = np.max(np.abs(comp / ex - 1)).astype(float)
    for dz in (-0.1, 0.1):
        e1 = np.max(np.abs(O.student_map(z, 4.0, 10, 3.93473 + dz) / ex - 1)).astype(float)
        assert e1 > 0.9 * e0


@pytest.mark.parametrize("n,zstar", [(3.0, 3.5667), (5.0, 4.6506), (10.0, 6.9584)])
def test_other_n_composite_accuracy(n, zstar):
    """The paper is silent for n != 4 (reading R13): K = 16 and the min-max crossover
    recorded in tests/golden/student_crossover.txt keep the composite within 1.4e-5."""
    z = np.linspace(1e-4, 12.0, 6001)
    ex = O.student_exact(z, n)
    comp = O.student_map(z, n, 16, zstar)
    assert np.max(np.abs(comp / ex - 1)).astype(float) < 1.4e-5


def test_composite_odd_and_specials():
    z = np.array([-1.5, 1.5, -5.0, 5.0, 0.0, np.inf, np.nan])
    t = O.student_map(z, 4.0, 10, 3.93473)
    assert t[0] == -t[1] and t[2] == -t[3] and t[4] == 0
    assert t[5] == np.inf and np.isnan(t[6])


# ------------------------------------------------------------------ moments
def test_moments_exact_sums():
    rng = np.random.default_rng(0)
    x = rng.standard_normal(10001)
    S = O.moments(x, 4)
    mp.mp.dps = 50
    for k in range(4):
        ref = mp.fsum(mp.mpf(float(v)) ** (k + 1) for v in x)
        assert abs(ld2mp(S[k]) - ref) <= 1e-15 * mp.fsum(abs(mp.mpf(float(v))) ** (k + 1) for v in x)
    xf = x.astype(np.float32)
    Sf = O.moments(xf, 2)
    assert abs(float(Sf[1]) - float(np.sum(xf.astype(np.float64) ** 2))) < 1e-9


# ---- §3.6 purely numerical method: the RODE solved by explicit RK ----
@pytest.mark.parametrize("n", [3.0, 4.0, 5.0, 10.0])
def test_rode_rk_meets_printed_5e8_on_z6(n):
    """the direct numerical solution of the Student RODE from the
    centre conditions has precision better than 5e-8 on |z| < 6.  The
    oracle's forward RK4 (h = 1e-4) against the exact map (pinned above to the
    closed forms and mpmath): a dropped term, a wrong sign in the ODE or a wrong
    gamma fails by orders of magnitude."""
    z = np.linspace(-6.0, 6.0, 49)
    e = O.student_exact(z, n)
    r = O.student_rode(z, n, 1e-4)
    m = z != 0
    assert np.max(np.abs(r[m] / e[m] - 1)) < 5e-8
    assert r[z == 0][0] == 0 and np.array_equal(np.sign(r), np.sign(z))


def test_rode_rk_order_and_large_n_series():
    """Fourth-order convergence (h -> h/2 cuts the error ~16x), and for large n the
    solution follows the textbook expansion A&S 26.7.5 quoted at P:222-227,
    t = z + (z^3 + z)/(4n) + (5z^5 + 16z^3 + 3z)/(96n^2) + O(n^-3)."""
    z = np.array([1.0, 2.5, 4.0])
    e = O.student_exact(z, 4.0)
    e1 = np.abs(O.student_rode(z, 4.0, 4e-3) / e - 1).max()
    e2 = np.abs(O.student_rode(z, 4.0, 2e-3) / e - 1).max()
    assert 12 < e1 / e2 < 20
    n = 1e4
    cf = z + (z**3 + z) / (4 * n) + (5 * z**5 + 16 * z**3 + 3 * z) / (96 * n**2)
    r = O.student_rode(z, n, 1e-3).astype(np.float64)
    assert np.max(np.abs(r - cf)) < 1e-8          # next term (3z^7 + ...)/(384 n^3) < 2e-9 here
    assert np.max(np.abs(r - z - (z**3 + z) / (4 * n))) > 1e-7   # the n^-2 term is resolved
