"""Pins for the oracle's exponential-base recycling map (§4,
P:284-395): masses p+- (P:307-314), the centre slope f0(0+)/f(0)
(P:336), the VG lambda = 1 identity, closed-form CDFs, mpmath."""
import mpmath as mp
import numpy as np
import pytest

import oracle as O
from _parity import student_rode_bar
from _util import ld2mp

HYP = [(1.0, 0.0, 1.0), (1.0, 0.5, 1.0), (2.0, -1.0, 0.5)]


def _mp_hyp_masses(a, b, d):
    mp.mp.dps = 30
    f = lambda x: mp.exp(-a * mp.sqrt(d * d + x * x) + b * x)
    zp, zm = mp.quad(f, [0, mp.inf]), mp.quad(f, [-mp.inf, 0])
    return zm / (zp + zm), zp / (zp + zm)


@pytest.mark.parametrize("par", HYP)
def test_hyperbolic_masses_vs_mpmath(par):
    m = O.target_masses(O.HYPERBOLIC, par)
    pm, pp = _mp_hyp_masses(*par)
    assert abs(ld2mp(m[0]) - pm) < 1e-17 and abs(ld2mp(m[1]) - pp) < 1e-17
    if par[1] == 0.0:
        assert abs(float(m[0]) - 0.5) < 1e-18          # beta = 0 -> p+ = p- = 1/2 (symmetric density)


def test_hyperbolic_centre_slope_is_K1e():
    """alpha = delta = 1, beta = 0: Q'(0) = p+ (a-b) 2 a d K1(d g) e^{a d}/g = K1(1) e ~ 1.63615
    (SPEC S:263)."""
    f0 = O.target_density(O.HYPERBOLIC, [1.0, 0.0, 1.0], [0.0])[0]
    slope = 0.5 * 1.0 / f0
    mp.mp.dps = 30
    assert abs(ld2mp(slope) - mp.besselk(1, 1) * mp.e) < 1e-17
    # and the normalised density matches the closed form g/(2 a d K1(d g))
    x = np.array([-3.0, 0.2, 1.7])
    got = O.target_density(O.HYPERBOLIC, [1.0, 0.5, 1.0], x)
    g = mp.sqrt(1 - 0.25)
    for xi, gi in zip(x, got):
        ref = g / (2 * 1.0 * 1.0 * mp.besselk(1, g)) * mp.exp(-mp.sqrt(1 + xi * xi) + 0.5 * xi)
        assert abs(ld2mp(gi) / ref - 1) < 5e-17


@pytest.mark.parametrize("par", HYP)
def test_hyperbolic_map_vs_mpmath(par):
    """Q(v) = F^-1(F0(v)) at a few v, checked by mpmath quadrature of the tail."""
    mp.mp.dps = 30
    a, b, d = par
    pm, pp = _mp_hyp_masses(*par)
    f = lambda x: mp.exp(-a * mp.sqrt(d * d + x * x) + b * x)
    Z = mp.quad(f, [-mp.inf, 0, mp.inf])
    v = np.array([0.3, 2.0, 8.0, -0.4, -3.0])
    q = O.recycle_exp_to_target(O.HYPERBOLIC, par, v)
    for vi, qi in zip(v, q):
        qq = ld2mp(qi)
        if vi > 0:
            lhs, rhs = mp.quad(f, [qq, mp.inf]) / Z, pp * mp.exp(-(a - b) * vi)
        else:
            lhs, rhs = mp.quad(f, [-mp.inf, qq]) / Z, pm * mp.exp((a + b) * vi)
        dens = f(qq) / Z
        assert abs(lhs - rhs) / dens <= 1e-16 * max(1, abs(qq))          # |dQ| = |dF|/f


def test_hyperbolic_symmetry_beta0():
    v = np.array([0.1, 1.0, 5.0, 12.0])
    a = O.recycle_exp_to_target(O.HYPERBOLIC, [1.0, 0.0, 1.0], v)
    b = O.recycle_exp_to_target(O.HYPERBOLIC, [1.0, 0.0, 1.0], -v)
    assert np.all(np.abs(a + b) <= 1e-17 * np.abs(a))


def test_vg_lambda1_is_identity_and_masses():
    """'if lambda = 1 the VG model is ... identical to the base, so that Q(v) = v';
    its split is the two-sided exponential's, p+ = (a+b)/(2a)."""
    par = [1, 2.0, 0.5]
    m = O.target_masses(O.VG, par)
    assert abs(float(m[1]) - 2.5 / 4.0) < 1e-18
    v = np.array([-5.0, -0.3, 0.2, 3.0, 9.0])
    assert np.all(np.abs(O.recycle_exp_to_target(O.VG, par, v) - v) <= 1e-17 * np.abs(v))


def test_vg_lambda2_closed_form_cdf():
    """lambda = 2: K_{3/2}(z) = sqrt(pi/2z) e^-z (1 + 1/z), so f ~ e^{bx - a|x|}(|x| + 1/a)
    and the tails integrate in closed form; p+-  and Q against them."""
    a, b = 2.0, 0.5
    mp.mp.dps = 30
    r, l = mp.mpf(a - b), mp.mpf(a + b)
    # integral_q^inf e^{-r x}(x + 1/a) dx = e^{-r q}((q + 1/a)/r + 1/r^2)
    tail_r = lambda q: mp.exp(-r * q) * ((q + 1 / mp.mpf(a)) / r + 1 / r ** 2)
    tail_l = lambda q: mp.exp(l * q) * ((-q + 1 / mp.mpf(a)) / l + 1 / l ** 2)
    Z = tail_r(0) + tail_l(0)
    m = O.target_masses(O.VG, [2, a, b])
    assert abs(ld2mp(m[1]) - tail_r(0) / Z) < 1e-18
    for vi in (0.5, 4.0, -1.0, -6.0):
        q = ld2mp(O.recycle_exp_to_target(O.VG, [2, a, b], [vi])[0])
        if vi > 0:
            err = tail_r(q) / Z - (tail_r(0) / Z) * mp.exp(-r * vi)
            dens = mp.exp(-r * q) * (q + 1 / mp.mpf(a)) / Z
        else:
            err = tail_l(q) / Z - (tail_l(0) / Z) * mp.exp(l * vi)
            dens = mp.exp(l * q) * (-q + 1 / mp.mpf(a)) / Z
        assert abs(err) / dens <= 1e-16 * max(1, abs(q))


# ------------------------------------------- the product's host-side table builder
def _node_w(tab, side, j, ks):
    """positions of nodes k0 + ks of segment j (qm_rode_params.h): uniform, octave
    levels (g = 1: level 0 = [0, Wc/64], level l = [Wc 2^(l-7), Wc 2^(l-6)], 512
    intervals each) or quartic-graded (g = 4)"""
    w0, h, ih, k0, n, w1, G, g = tab[32 + 8 * (3 * side + j):32 + 8 * (3 * side + j) + 8]
    ks = np.asarray(ks)
    if g == 1:
        lv, i = ks // 512, ks % 512
        return np.where(lv == 0, w1 * np.ldexp(i / 512.0, -6), w1 * np.ldexp(1 + i / 512.0, lv - 7))
    if g == 4:
        return G * ks.astype(np.float64) ** 4
    return w0 + ks * h


@pytest.mark.parametrize("kind,par", [(O.HYPERBOLIC, p) for p in HYP] +
                         [(O.VG, [1, 2.0, 0.5]), (O.VG, [2, 2.0, 0.5]), (O.VG, [3, 1.0, -0.4]),
                          (O.VG, [1.5, 2.0, 0.5]), (O.VG, [2.7, 1.0, -0.6])])
def test_product_rode_table_vs_oracle(kind, par):
    """libqm's table (RODE integrated backward in long double, the centre segment
    forward) at sampled nodes of each segment vs the oracle's exact map, R' and R''
    vs differences of it; Q(0) = 0 and the centre slopes of P:336/P:344 as residuals."""
    from paper_0901_0638_b200.qm import qm_rode_table_host
    tab = qm_rode_table_host(kind, par)
    H, SEG = 80, 32
    NT, NC = int(tab[1]), int(tab[SEG + 4])                              # layout from the header
    assert tab[1] == NT and tab[30] == 3
    assert np.all(np.abs(tab[12:14]) < 1e-12) and np.all(np.abs(tab[14:16]) < 1e-12)
    assert np.all(np.abs(tab[22:24]) < 1e-14 * (1 + 2.0 / (tab[10:12])))         # forward/backward joint
    m = O.target_masses(kind, par)
    assert abs(tab[8] - float(m[1])) < 1e-15 and abs(tab[9] - float(m[0])) < 1e-15
    for side in (0, 1):
        sg = 1 if side == 0 else -1
        nodes = tab[H + side * 4 * (NT + 1):H + (side + 1) * 4 * (NT + 1)].reshape(-1, 4)
        assert nodes[0, 0] == 0.0
        for j, js in enumerate([[1, 2, 37, 1800, 3583], [1, 500, 5000, 16383], [1, 100, 2000, 4096]]):
            w0, h, ih, k0, n, w1, G, g = tab[SEG + 8 * (3 * side + j):SEG + 8 * (3 * side + j) + 8]
            assert int(k0) == [0, NC, NC + 16384][j] and abs(w0 + n * h - w1) <= 1e-12 * w1
            js = np.array(js)
            # centre nodes at Wc (k/n)^4 (Wc = 2/rate for real-lambda VG (R29), else 10/rate)
            wk = _node_w(tab, side, j, js)
            real = kind == O.VG and par[0] != int(par[0])
            assert g == (0 if j else (4 if real else 1)) and (j or abs(w1 * tab[10 + side] - (2 if real else 10)) < 1e-12)
            ex = O.recycle_exp_to_target(kind, par, wk * sg).astype(np.float64)
            assert np.abs(nodes[int(k0) + js, 0] / ex - 1).max() < 1e-13, j
        # R' and R'' against central differences of the exact map (long double; O(hh^2) ~ 1e-8)
        ks = np.array([300, 500, 1000, 2000, 3500])
        w = _node_w(tab, side, 0, ks)
        hh = 1e-2 * tab[SEG + 8 * 3 * side + 1]                           # 1e-2 Wc/n
        qp = O.recycle_exp_to_target(kind, par, (w + hh) * sg)
        q0 = O.recycle_exp_to_target(kind, par, w * sg)
        qm = O.recycle_exp_to_target(kind, par, (w - hh) * sg)
        d1 = ((qp - qm) / (2 * np.longdouble(hh))).astype(np.float64)
        d2 = ((qp - 2 * q0 + qm) / np.longdouble(hh) ** 2).astype(np.float64)
        assert np.abs(d1 / nodes[ks, 1] - 1).max() < 1e-7
        assert np.abs(d2 - nodes[ks, 2]).max() < 1e-6 * (1 + np.abs(nodes[ks, 2]).max())


# ------------------------------------------- VG with real lambda > 1 (reading R29)
def _mp_lam(lam):
    return mp.mpf(float(lam))          # the double the oracle receives, exactly


@pytest.mark.parametrize("nu,z", [(0.6, 3.0), (1.0, 0.5), (2.2, 1e-3), (2.2, 1.0), (3.0, 2.0), (5.5, 30.0),
                                  (7.3, 1e-5), (2.2, 500.0), (4.75, 12.0)])
def test_besselk_trapezoid_vs_mpmath(nu, z):
    """The oracle's K_nu (trapezoidal rule on A&S 9.6.24) vs mpmath besselk."""
    mp.mp.dps = 40
    rel = abs(ld2mp(O.besselk(nu, z)) / mp.besselk(nu, z) - 1)
    assert rel < (2e-17 if z < 100 else 1e-16), rel


@pytest.mark.parametrize("m", [0, 1, 2, 4])
def test_besselk_half_integer_closed_form(m):
    """K_{m+1/2}(z) = sqrt(pi/2z) e^-z sum_k (m+k)!/(k!(m-k)!) (2z)^-k (A&S 10.2.15), the
    form the oracle uses for integer lambda: the two VG paths describe one density."""
    mp.mp.dps = 40
    for z in (0.05, 1.0, 7.5):
        cf = mp.sqrt(mp.pi / (2 * z)) * mp.exp(-z) * mp.fsum(
            mp.factorial(m + k) / (mp.factorial(k) * mp.factorial(m - k)) * (2 * mp.mpf(z)) ** (-k) for k in range(m + 1))
        assert abs(ld2mp(O.besselk(m + 0.5, z)) / cf - 1) < 2e-17


def _vg_masses_2f1(lam, a, b):
    """p+ and p- as printed in P:372-393 (A&S/G&R 6.621.3), mpmath hyp2f1."""
    L = _mp_lam(lam)
    a, b = mp.mpf(a), mp.mpf(b)
    pre = 2 ** (2 * L - 1) * mp.gamma(L + mp.mpf(1) / 2) / (mp.sqrt(mp.pi) * mp.gamma(L + 1))
    pp = pre * ((a + b) / (a - b)) ** L * mp.hyp2f1(2 * L, L, L + 1, (a + b) / (b - a))
    pm = pre * ((a - b) / (a + b)) ** L * mp.hyp2f1(2 * L, L, L + 1, (b - a) / (a + b))
    return pm, pp


@pytest.mark.parametrize("lam,a,b", [(2, 2.0, 0.5), (3, 1.0, -0.4), (1.5, 2.0, 0.5), (2.7, 2.0, 0.5),
                                     (2.7, 1.0, -0.6), (3.3, 1.5, 0.2), (5.25, 2.0, 1.2), (1.2, 1.0, 0.3)])
def test_vg_masses_vs_printed_2f1(lam, a, b):
    """p+- of the oracle (quadrature of the density) vs the paper's closed forms
    (P:372-393), and vs the regularized incomplete beta I_{(a+b)/2a}(lambda, lambda)
    (VG = difference of two Gamma(lambda) variables with rates a-b and a+b)."""
    mp.mp.dps = 50
    m = O.target_masses(O.VG, [lam, a, b])
    pm, pp = _vg_masses_2f1(lam, a, b)
    assert abs(pp + pm - 1) < mp.mpf(10) ** -40
    assert abs(ld2mp(m[1]) - pp) < 2e-17 and abs(ld2mp(m[0]) - pm) < 2e-17, (ld2mp(m[1]) - pp)
    ib = mp.betainc(_mp_lam(lam), _mp_lam(lam), 0, (mp.mpf(a) + b) / (2 * mp.mpf(a)), regularized=True)
    assert abs(ib - pp) < mp.mpf(10) ** -40
    if b == 0:
        assert abs(ld2mp(m[1]) - mp.mpf(1) / 2) < 1e-18


@pytest.mark.parametrize("par", [[1.5, 2.0, 0.5], [2.7, 1.0, -0.6], [1.2, 1.0, 0.3]])
def test_vg_real_lambda_map_vs_mpmath(par):
    """Q(v) = F^-1(F0(v)) for real lambda (K_nu of non-half-integer order): the tail
    mass beyond Q equals the base's, by mpmath quadrature of the printed density."""
    mp.mp.dps = 24
    lam, a, b = _mp_lam(par[0]), mp.mpf(par[1]), mp.mpf(par[2])
    f = lambda x: mp.exp(b * x) * abs(x) ** (lam - mp.mpf(1) / 2) * mp.besselk(lam - mp.mpf(1) / 2, a * abs(x))
    Z = mp.quad(f, [-mp.inf, -1, 0, 1, mp.inf])
    pm, pp = _vg_masses_2f1(par[0], par[1], par[2])
    v = np.array([0.05, 7.0, -0.3, -4.0])
    q = O.recycle_exp_to_target(O.VG, par, v)
    for vi, qi in zip(v, q):
        qq = ld2mp(qi)
        if vi > 0:
            lhs, rhs = mp.quad(f, [qq, qq + 1, mp.inf]) / Z, pp * mp.exp(-(a - b) * vi)
        else:
            lhs, rhs = mp.quad(f, [-mp.inf, qq - 1, qq]) / Z, pm * mp.exp((a + b) * vi)
        assert abs(lhs - rhs) / (f(qq) / Z) <= 1e-16 * max(1, abs(qq)), (vi, lhs - rhs)


# ------------------------------- Gaussian base: the Student table of §3.6
def _emulate_kernel(tab, z):
    """The kernel's interpolation (qm_rode.cuh) in numpy, to check the host table
    on CPU: segment select, quintic Hermite on (R, R', R''), log segment -> exp."""
    H, SEG = 80, 32
    NT, NC = int(tab[1]), int(tab[SEG + 4])                              # layout from the header
    out = np.empty(z.shape)
    for i, x in enumerate(z):
        side = 1 if x < 0 else 0
        a = abs(x)
        j = int(a >= tab[SEG + 24 * side + 8]) + int(a >= tab[SEG + 24 * side + 16])
        w0, h, ih, k0, n, w1, G, g = tab[SEG + 24 * side + 8 * j:SEG + 24 * side + 8 * j + 8]
        if g == 1:                       # octave levels: x = w/Wc = 2^e m, level l = e + 7, 512 intervals each
            x = a * ih
            m, e = np.frexp(x)           # x = m 2^e, m in [0.5, 1)
            lv = min(max(int(e) - 1 + 7, 0), 6) if x > 0 else 0
            u = (2 * m - 1) * 512.0                          # exact: 512 (mantissa - 1)
            s = x * 32768.0 if lv == 0 else np.floor(u) + 512 * lv + (u - np.floor(u))  # t kept exact
            h = w1 * 2.0 ** (max(lv, 1) - 16)
        else:
            s = (a - w0) * ih if g == 0 else n * (a * ih) ** (1.0 / g)  # graded: w = Wc (s/n)^g
        s = min(s, n)
        fk = min(np.floor(s), n - 1)
        k, t = int(k0) + int(fk), s - fk
        if g == 1 and lv > 0:
            k, t = int(k0) + 512 * lv + int(np.floor(u)), u - np.floor(u)
        nd = tab[H + side * 4 * (NT + 1):H + (side + 1) * 4 * (NT + 1)].reshape(-1, 4)
        (r0, d0, e0), (r1, d1, e1) = nd[k, :3], nd[k + 1, :3]
        if g <= 1:
            ws0 = ws1 = h
            wss0 = wss1 = 0.0
        else:                                                            # dw/ds, d2w/ds2 at the nodes
            ws0, ws1 = g * G * fk ** (g - 1), g * G * (fk + 1) ** (g - 1)
            wss0, wss1 = g * (g - 1) * G * fk ** (g - 2), g * (g - 1) * G * (fk + 1) ** (g - 2)
        m0, m1, dp = ws0 * d0, ws1 * d1, r1 - r0
        a0, a1 = ws0 * ws0 * e0 + wss0 * d0, ws1 * ws1 * e1 + wss1 * d1
        c3 = 10 * dp - 6 * m0 - 4 * m1 - 1.5 * a0 + 0.5 * a1
        c4 = -15 * dp + 8 * m0 + 7 * m1 + 1.5 * a0 - a1
        c5 = 6 * dp - 3 * m0 - 3 * m1 - 0.5 * a0 + 0.5 * a1
        q = r0 + t * (m0 + t * (0.5 * a0 + t * (c3 + t * (c4 + t * c5))))
        if j == 2 and tab[31]:
            q = -np.exp(q) if side else np.exp(q)
        out[i] = q
    return out


@pytest.mark.parametrize("nu", [1.0, 3.0, 4.0, 10.0, 200.0])
def test_product_student_table_vs_oracle(nu):
    """libqm's Student table (RODE backward from the far-tail anchor, in log t beyond
    |z| = 2; the centre forward from Q(0) = 0, Q'(0) = gamma): Q(0) and gamma come
    out as residuals, nodes of every segment equal the oracle's exact map, and the
    kernel's interpolation (emulated) is within student_rode_bar of it (<= 1e-13 on
    |z| <= 6; the paper's numerical solution promises 5e-8 there)."""
    from paper_0901_0638_b200.qm import STUDENT, qm_rode_table_host
    tab = qm_rode_table_host(STUDENT, [nu])
    H, SEG = 80, 32
    NT, NC = int(tab[1]), int(tab[SEG + 4])                              # layout from the header
    assert tab[0] == 3 and tab[1] == NT and tab[31] == 1
    assert abs(tab[12]) < 1e-15 and abs(tab[14]) < 1e-15 and abs(tab[22]) < 1e-15
    nodes = tab[H:H + 4 * (NT + 1)].reshape(-1, 4)
    left = tab[H + 4 * (NT + 1):H + 8 * (NT + 1)].reshape(-1, 4)
    for j, js in enumerate([[1, 37, 1800, 3200, 3400, 3584], [1, 5000, 16384], [0, 2000, 4094]]):
        w0, h, ih, k0, n, w1, G, g = tab[SEG + 8 * j:SEG + 8 * j + 8]
        assert int(k0) == [0, NC, NC + 16384 + 1][j] and abs(w0 + n * h - w1) <= 1e-15 * w1
        assert g == (1 if j == 0 else 0)                                 # centre on octave levels
        js = np.array(js)
        ex = O.student_exact(_node_w(tab, 0, j, js), nu)
        got = nodes[int(k0) + js, 0]
        if j == 2:
            assert np.max(np.abs(got / np.log(ex).astype(np.float64) - 1)) < 1e-15
            assert np.array_equal(left[int(k0) + js, :3], nodes[int(k0) + js, :3])   # log |t| is even
        else:
            assert np.max(np.abs(got / ex.astype(np.float64) - 1)) < 1e-15
            assert np.array_equal(left[int(k0) + js, :3], -nodes[int(k0) + js, :3])  # t is odd
    z = np.concatenate([np.linspace(-6, 6, 401), np.random.default_rng(1).uniform(-38.4, 38.4, 200)])
    z = z[z != 0]
    ex = O.student_exact(z, nu).astype(np.float64)
    g = _emulate_kernel(tab, z)
    fin = np.isfinite(ex)
    rel = np.abs(g[fin] / ex[fin] - 1)
    assert np.all(rel <= student_rode_bar(z[fin], ex[fin], nu))


def test_product_student_table_rejects():
    from paper_0901_0638_b200.qm import STUDENT, qm_rode_table_host
    for nu in (0.5, 0.0, -1.0, 201.0, float("nan")):
        with pytest.raises(ValueError):
            qm_rode_table_host(STUDENT, [nu])

@pytest.mark.parametrize("kind,par", [("hyp", [1.0, 0.5, 1.0]), ("hyp", [2.0, -0.7, 0.3]), ("student", [3.0]),
                                      ("student", [1.0])])
def test_centre_second_derivative_is_the_rode(kind, par):
    """The stored R'' of the centre nodes (the builder's long double, rounded) is the
    RODE evaluated at the stored (R, R') and the node -- R'' = H(R) R'^2 - w R'
    (Gaussian base) or H(R) R'^2 - rate R' (exponential base), H = -(log f)' of the
    target -- within rounding (also what the A/B fast path
    QM_RODE_ODE_D2 = 1 of qm_rode.cuh computes on the fly)."""
    from paper_0901_0638_b200.qm import HYPERBOLIC, STUDENT, qm_rode_table_host
    tab = qm_rode_table_host(HYPERBOLIC if kind == "hyp" else STUDENT, par)
    H, SEG, NT = 80, 32, int(tab[1])
    ks = np.arange(0, 3584, 7)
    for side in ((0, 1) if kind == "hyp" else (0,)):
        nd = tab[H + side * 4 * (NT + 1):H + (side + 1) * 4 * (NT + 1)].reshape(-1, 4)[ks]
        r, rp, rpp = nd[:, 0], nd[:, 1], nd[:, 2]
        if kind == "hyp":
            a, b, d = par
            assert (tab[3], tab[4], tab[5]) == (a, b, d * d)          # the kernel's parameters
            Hr = a * r / np.sqrt(d * d + r * r) - b
            f = Hr * rp * rp - tab[10 + side] * rp
        else:
            n = par[0]
            assert tab[2] == n
            w = _node_w(tab, side, 0, ks)
            f = (n + 1) * r / (n + r * r) * rp * rp - w * rp
        scale = np.abs(Hr * rp * rp if kind == "hyp" else (n + 1) * r / (n + r * r) * rp * rp) + np.abs(
            (tab[10 + side] if kind == "hyp" else w) * rp)
        assert np.all(np.abs(f - rpp) <= 1e-14 * scale + 1e-300), np.max(np.abs(f - rpp) / scale)
