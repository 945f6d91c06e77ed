// qm_rode_host.cpp -- per-parameter host setup of the exponential-base
// recycling maps of §4: hyperbolic (§4.1) and
// variance gamma with integer lambda (§4.2; reading R25).
//
// The map Q solves the Recycling ODE with an exponential base (P:104-114,
// P:330-345):   right (v > 0):  Q'' + (a-b) Q' = H(Q) Q'^2
//               left  (v < 0):  Q'' - (a+b) Q' = H(Q) Q'^2
// with Q(0) = 0, Q'(0+-) = f0(0+-)/f(0).  Integrated forward from v = 0 this ODE
// is exponentially ill-conditioned: Q' = 1 is a repelling fixed point
// (d(Q'-1)/dv ~ (a-b)(Q'-1)), so an error e in Q'(0) grows like e^{(a-b)v}
// (reading R26).  We therefore integrate BACKWARD, in the stable direction,
// from an anchor at |v| = V where Q is fixed by its definition
// Fbar(Q(V)) = p+ e^{-(a-b)V} (tail mass by Gauss-Legendre quadrature, Newton),
// down to v = 0 with classical RK4 in long double, recording (Q, Q') at N+1
// equally spaced nodes per side for cubic Hermite interpolation on the GPU.
// Q(0) = 0 and the slope f0(0)/f(0) of P:336/P:344 come out as checks.
//
// Table layout (doubles): see qm_rode.cuh.
#include <cmath>
#include <cstring>
#include <cstdint>

#include "qm_rode_params.h"

namespace qm {

typedef long double ld;

namespace {

struct Target {
    int kind;            // QM_RODE_HYPERBOLIC / QM_RODE_VG
    ld a, b, d;          // alpha, beta, delta (delta unused for VG)
    int m;               // VG: lambda - 1
    ld c[QM_RODE_VG_MAXM + 1];   // VG: polynomial coefficients of S(|x|)

    // log of the unnormalised density
    ld logg(ld x) const
    {
        if (kind == QM_RODE_HYPERBOLIC) return -a * sqrtl(d * d + x * x) + b * x;
        const ld ax = fabsl(x);
        ld s = c[m];
        for (int k = m - 1; k >= 0; --k) s = s * ax + c[k];          // S(|x|) = sum c_j |x|^j
        return b * x - a * ax + logl(s);
    }
    // H(x) = -(log f)'(x) on the side `dir` of the origin
    // (the VG H is discontinuous at 0 for lambda = 1: the side, not sign(x), decides)
    ld H(ld x, int dir) const
    {
        if (kind == QM_RODE_HYPERBOLIC) return a * x / sqrtl(d * d + x * x) - b;
        const ld ax = fabsl(x), sg = (ld)dir;
        ld s = c[m], ds = 0.0L;
        for (int k = m - 1; k >= 0; --k) { ds = ds * ax + s; s = s * ax + c[k]; }
        return -b + sg * (a - ds / s);
    }
};

// 10-point Gauss-Legendre on [lo, hi] of exp(logg(x) - shift)
const ld GLX[5] = {0.148874338981631210884826001129720L, 0.433395394129247190799265943165784L,
                   0.679409568299024406234327365114874L, 0.865063366688984510732096688423493L,
                   0.973906528517171720077964012084452L};
const ld GLW[5] = {0.295524224714752870173892994651338L, 0.269266719309996355091226921569469L,
                   0.219086362515982043995534934228163L, 0.149451349150580593145776339657697L,
                   0.066671344308688137593568809893332L};

ld gl10(const Target &t, ld lo, ld hi, ld shift)
{
    const ld c = 0.5L * (lo + hi), h = 0.5L * (hi - lo);
    ld s = 0.0L;
    for (int j = 0; j < 5; ++j)
        s += GLW[j] * (expl(t.logg(c - h * GLX[j]) - shift) + expl(t.logg(c + h * GLX[j]) - shift));
    return s * h;
}

// integral of g over [x, inf) (dir = +1) or (-inf, x] (dir = -1), in units of e^{shift}
ld tail_mass(const Target &t, ld x, int dir, ld rate, ld shift)
{
    ld w = 0.125L / rate;
    if (t.kind == QM_RODE_HYPERBOLIC && w > 0.25L * t.d) w = 0.25L * t.d;    // resolve sqrt(d^2 + x^2)
    ld s = 0.0L;
    for (int k = 0; k < 400000; ++k) {
        const ld lo = (dir > 0) ? x + k * w : x - (k + 1) * w;
        const ld p = gl10(t, lo, lo + w, shift);
        s += p;
        if (p < 1e-22L * s) break;
    }
    return s;
}

}  // namespace

bool rode_table_build(int kind, const double *params, double *tab)
{
    Target t;
    std::memset(&t, 0, sizeof(t));
    t.kind = kind;
    if (kind == QM_RODE_HYPERBOLIC) {
        t.a = params[0]; t.b = params[1]; t.d = params[2];
        if (!(t.a > 0 && fabsl(t.b) < t.a && t.d > 0)) return false;
    } else if (kind == QM_RODE_VG) {
        const double lam = params[0];
        t.a = params[1]; t.b = params[2];
        if (!(lam >= 1 && lam <= QM_RODE_VG_MAXM + 1 && lam == std::floor(lam) && t.a > 0 && fabsl(t.b) < t.a))
            return false;
        t.m = (int)lam - 1;
        // K_{m+1/2}(z) = sqrt(pi/2z) e^-z sum_k (m+k)!/(k!(m-k)!) (2z)^-k  (A&S 10.2.15), so
        // f ~ e^{bx - a|x|} sum_k (m+k)!/(k!(m-k)!) (2a)^-k |x|^{m-k};  c[j] multiplies |x|^j
        for (int k = 0; k <= t.m; ++k) {
            ld co = 1.0L;
            for (int j = t.m - k + 1; j <= t.m + k; ++j) co *= (ld)j;
            for (int j = 2; j <= k; ++j) co /= (ld)j;
            t.c[t.m - k] = co * powl(2.0L * t.a, -(ld)k);
        }
    } else {
        return false;
    }
    const ld rr = t.a - t.b, rl = t.a + t.b;              // base rates
    const ld shift = t.logg(0.0L);
    const ld Zr = tail_mass(t, 0.0L, +1, rr, shift), Zl = tail_mass(t, 0.0L, -1, rl, shift);
    const ld Z = Zr + Zl, pp = Zr / Z, pm = Zl / Z;
    const int N = QM_RODE_NODES;

    for (int side = 0; side < 2; ++side) {
        const ld rate = side == 0 ? rr : rl, p = side == 0 ? pp : pm;
        const int dir = side == 0 ? +1 : -1;
        const ld V = QM_RODE_VRATE / rate, h = V / N;
        // anchor: tail mass of the target beyond Q(V) equals the base's, p e^{-rate V}
        const ld target = p * expl(-rate * V) * Z;            // in units of e^{shift}
        ld q = dir * (V + 1.0L);                               // Q ~ v + const
        for (int it = 0; it < 100; ++it) {
            const ld g = tail_mass(t, q, dir, rate, shift) - target;
            const ld fq = expl(t.logg(q) - shift);
            const ld step = g / fq;                            // d(tail)/dq = -dir f(q)
            q += dir * step;
            if (fabsl(step) <= 1e-18L * fabsl(q)) break;
        }
        // Q'(V) = f0(V)/f(Q(V)) (first-order quantile ODE), in |v| units
        ld Q = q;
        ld P = dir * (p * rate * expl(-rate * V) * Z) / expl(t.logg(q) - shift);
        // integrate R(w) = Q(dir w), w = |v|, backward from w = V to 0:
        //   R'' = H(R) R'^2 - rate R'   (both sides, with R' = dR/dw)
        double *nodes = tab + QM_RODE_HEADER + side * 2 * (N + 1);
        nodes[2 * N] = (double)Q;
        nodes[2 * N + 1] = (double)P;
        const int sub = QM_RODE_SUBSTEPS;
        const ld s = -h / sub;
        for (int k = N - 1; k >= 0; --k) {
            for (int j = 0; j < sub; ++j) {
                const ld k1q = P, k1p = t.H(Q, dir) * P * P - rate * P;
                const ld q2 = Q + 0.5L * s * k1q, p2 = P + 0.5L * s * k1p;
                const ld k2q = p2, k2p = t.H(q2, dir) * p2 * p2 - rate * p2;
                const ld q3 = Q + 0.5L * s * k2q, p3 = P + 0.5L * s * k2p;
                const ld k3q = p3, k3p = t.H(q3, dir) * p3 * p3 - rate * p3;
                const ld q4 = Q + s * k3q, p4 = P + s * k3p;
                const ld k4q = p4, k4p = t.H(q4, dir) * p4 * p4 - rate * p4;
                Q += s / 6.0L * (k1q + 2.0L * k2q + 2.0L * k3q + k4q);
                P += s / 6.0L * (k1p + 2.0L * k2p + 2.0L * k3p + k4p);
            }
            nodes[2 * k] = (double)Q;
            nodes[2 * k + 1] = (double)P;
        }
        // checks against the centre conditions of P:336 / P:344
        const ld slope0 = dir * p * rate * Z / expl(t.logg(0.0L) - shift);
        tab[12 + side] = (double)Q;                            // residual Q(0)
        tab[14 + side] = (double)(P / slope0 - 1.0L);          // relative slope residual
        nodes[0] = 0.0;                                        // Q(0) = 0 exactly
        tab[2 + side] = (double)h;
        tab[4 + side] = (double)(1.0L / h);
        tab[6 + side] = (double)V;
        tab[8 + side] = (double)p;
        tab[10 + side] = (double)rate;
        const ld lp = logl(p);
        tab[16 + side] = (double)lp;                           // log p_s as a double-double
        tab[18 + side] = (double)(lp - (ld)(double)lp);
        tab[20 + side] = (double)(1.0L / rate);
    }
    tab[0] = kind;
    tab[1] = N;
    return true;
}

}  // namespace qm

// host-side table (diagnostics and the CPU-side tests of the builder)
extern "C" int qm_rode_table_host(int kind, const double *params, double *table)
{
    return qm::rode_table_build(kind, params, table) ? 0 : 1;
}
