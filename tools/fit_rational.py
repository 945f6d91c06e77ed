"""Design-time minimax fits of the exponential-coordinate normal quantile
(§5).

    Q(v) = Phi^-1(1 - e^-v / 2)
    Q(v) ~ v P(v) / Qd(v),  P, Qd of degree n, Qd(0) = 1   (the form of App A-D)

P:544: "Each time we increase the degree of the numerator and denominator,
keeping the interval fixed, the maximum relative error decreases by a factor of
about 20.  For example, a (12,12) rational approximation exists that covers the
same interval 0 <= v <= 37 with maximum relative error ... less than 5e-16 ...
An (8,8) approximation exists with precision about 6e-10 on the range
0 <= v <= 74."  Their coefficients are not printed; this tool computes them.

Method (all in mpmath at 60 digits): g(v) = Q(v)/v is fitted by P/Qd in the
relative-error norm.  (1) Linearised weighted least squares on a dense grid
(Sanathanan-Koerner iteration with Lawson re-weighting) gives a near-minimax
start; (2) the rational Remez exchange (equioscillation at 2n+2 points, the E*Qd
product linearised with the previous Qd) polishes it to the minimax solution.
Output: ascending coefficients (P then Qd) printed to 30 digits, and the
max relative error of the exact-arithmetic rational on a fine grid.

    python tools/fit_rational.py 12 37       # (12,12) on [0, 37]
    python tools/fit_rational.py 8 74        # (8,8) on [0, 74]
"""
from __future__ import annotations

import sys

import mpmath as mp

mp.mp.dps = 60


def Qexact(v):
    """Q(v) by root-finding on log ncdf (independent of the oracle)."""
    v = mp.mpf(v)
    if v == 0:
        return mp.mpf(0)
    t = mp.exp(-v) / 2
    # start: the tail model for large v, sqrt(pi/2) v for small v
    x0 = mp.sqrt(2 * v - mp.log(mp.pi) - mp.log(max(2 * v - mp.log(mp.pi), mp.mpf(1)))) if v > 2 else mp.sqrt(mp.pi / 2) * v
    return mp.findroot(lambda x: mp.log(mp.ncdf(-x)) - mp.log(t), x0)


def g(v):
    v = mp.mpf(v)
    if v < mp.mpf("1e-30"):
        return mp.sqrt(mp.pi / 2)
    return Qexact(v) / v


def peval(c, x):
    s = mp.mpf(0)
    for a in reversed(c):
        s = s * x + a
    return s


def rel_err(p, q, x, gx):
    return peval(p, x) / (peval(q, x) * gx) - 1


def lawson_sk(n, V, m=None, iters=40):
    """Near-minimax start: min sum w_j ((P - g Qd)/(g Qd_prev))^2 with Lawson weights."""
    m = m or 12 * n + 40
    xs = [V * (1 - mp.cos(mp.pi * (j + mp.mpf(1) / 2) / m)) / 2 for j in range(m)]
    gs = [g(x) for x in xs]
    w = [mp.mpf(1)] * m
    qprev = [mp.mpf(1)] + [mp.mpf(0)] * n
    best = None
    for it in range(iters):
        # unknowns p0..pn, q1..qn; residual r_j = (P(x) - g Qd(x)) / (g Qd_prev(x))
        A = mp.matrix(m, 2 * n + 1)
        b = mp.matrix(m, 1)
        for j, (x, gx) in enumerate(zip(xs, gs)):
            sc = mp.sqrt(w[j]) / (gx * peval(qprev, x))
            xp = mp.mpf(1)
            for k in range(n + 1):
                A[j, k] = xp * sc
                xp *= x
            xp = x
            for k in range(1, n + 1):
                A[j, n + k] = -gx * xp * sc
                xp *= x
            b[j] = gx * sc
        sol = mp.qr_solve(A, b)[0]
        p = [sol[k] for k in range(n + 1)]
        q = [mp.mpf(1)] + [sol[n + k] for k in range(1, n + 1)]
        errs = [rel_err(p, q, x, gx) for x, gx in zip(xs, gs)]
        emax = max(abs(e) for e in errs)
        if best is None or emax < best[0]:
            best = (emax, p, q)
        # Lawson: w_j <- w_j |e_j|, normalised
        w = [wj * abs(e) for wj, e in zip(w, errs)]
        s = sum(w)
        w = [wj / s for wj in w]
        qprev = q
    return best


def extrema(p, q, V, ref, samples=60):
    """Locate the 2n+2 alternating extrema of the relative error near the reference."""
    N = len(ref)
    pts = []
    bounds = [mp.mpf(0)] + [(ref[i] + ref[i + 1]) / 2 for i in range(N - 1)] + [mp.mpf(V)]
    for i in range(N):
        a, b = bounds[i], bounds[i + 1]
        xs = [a + (b - a) * k / samples for k in range(samples + 1)]
        es = [rel_err(p, q, x, g(x)) for x in xs]
        k = max(range(len(xs)), key=lambda j: abs(es[j]))
        # golden refinement around the sampled maximum
        lo, hi = xs[max(k - 1, 0)], xs[min(k + 1, samples)]
        f = lambda x: -abs(rel_err(p, q, x, g(x)))
        for _ in range(40):
            m1, m2 = lo + (hi - lo) * mp.mpf("0.382"), lo + (hi - lo) * mp.mpf("0.618")
            if f(m1) < f(m2):
                hi = m2
            else:
                lo = m1
        x = (lo + hi) / 2
        if abs(rel_err(p, q, xs[k], g(xs[k]))) > abs(rel_err(p, q, x, g(x))):
            x = xs[k]
        pts.append(x)
    return pts


def remez(n, V, start, iters=12, verbose=True):
    _, p, q = start
    N = 2 * n + 2
    # initial reference: extrema of the start's error on a dense grid
    xs = [V * (1 - mp.cos(mp.pi * j / (40 * N))) / 2 for j in range(40 * N + 1)]
    es = [rel_err(p, q, x, g(x)) for x in xs]
    # pick N alternating extrema
    ext = []
    for j in range(len(xs)):
        left = abs(es[j - 1]) if j > 0 else -1
        right = abs(es[j + 1]) if j + 1 < len(xs) else -1
        if abs(es[j]) >= left and abs(es[j]) >= right:
            ext.append(j)
    # merge same-sign neighbours, keep the larger
    alt = []
    for j in ext:
        if alt and mp.sign(es[j]) == mp.sign(es[alt[-1]]):
            if abs(es[j]) > abs(es[alt[-1]]):
                alt[-1] = j
        else:
            alt.append(j)
    while len(alt) > N:   # drop the smallest end
        if abs(es[alt[0]]) < abs(es[alt[-1]]):
            alt.pop(0)
        else:
            alt.pop()
    if len(alt) < N:
        ref = [V * (1 - mp.cos(mp.pi * i / (N - 1))) / 2 for i in range(N)]
    else:
        ref = [xs[j] for j in alt]
    E = mp.mpf(0)
    for it in range(iters):
        gs = [g(x) for x in ref]
        A = mp.matrix(N, N)
        b = mp.matrix(N, 1)
        for i, (x, gx) in enumerate(zip(ref, gs)):
            xp = mp.mpf(1)
            for k in range(n + 1):
                A[i, k] = xp
                xp *= x
            xp = x
            for k in range(1, n + 1):
                A[i, n + k] = -gx * xp
                xp *= x
            A[i, N - 1] = -((-1) ** i) * gx * peval(q, x)
            b[i] = gx
        sol = mp.lu_solve(A, b)
        p = [sol[k] for k in range(n + 1)]
        q = [mp.mpf(1)] + [sol[n + k] for k in range(1, n + 1)]
        E = sol[N - 1]
        ref = extrema(p, q, V, ref)
        emax = max(abs(rel_err(p, q, x, g(x))) for x in ref)
        if verbose:
            print(f"  remez {it}: |E| = {mp.nstr(abs(E), 6)}  max|e| on reference = {mp.nstr(emax, 6)}", flush=True)
        if abs(emax - abs(E)) < mp.mpf("1e-3") * abs(E):
            break
    return p, q, E


def max_error(p, q, V, m=4000):
    worst = (mp.mpf(0), mp.mpf(0))
    for j in range(m + 1):
        x = V * (1 - mp.cos(mp.pi * j / m)) / 2
        e = abs(rel_err(p, q, x, g(x)))
        if e > worst[0]:
            worst = (e, x)
    return worst


def fit(n, V, verbose=True):
    start = lawson_sk(n, V)
    if verbose:
        print(f"({n},{n}) on [0,{V}]: least-squares/Lawson start max|e| = {mp.nstr(start[0], 6)}", flush=True)
    p, q, E = remez(n, V, start, verbose=verbose)
    return p, q, E


if __name__ == "__main__":
    n, V = int(sys.argv[1]), mp.mpf(sys.argv[2])
    p, q, E = fit(n, V)
    e, x = max_error(p, q, V, m=int(sys.argv[3]) if len(sys.argv) > 3 else 2000)
    print(f"# ({n},{n}) on [0,{mp.nstr(V, 6)}]: minimax |E| = {mp.nstr(abs(E), 6)}, "
          f"max rel. error on a fine grid = {mp.nstr(e, 6)} at v = {mp.nstr(x, 6)}")
    print("P", " ".join(mp.nstr(c, 30) for c in p))
    print("Q", " ".join(mp.nstr(c, 30) for c in q))
