// qm_rode_host.cpp -- per-parameter host setup of the exponential-base
// recycling maps of §4: hyperbolic (§4.1) and
// variance gamma with real lambda >= 1 (§4.2; "if lambda > 1 matters
// remain reasonably straightforward ... The recycling ODE may be solved as
// before").  VG density e^{bx} |x|^nu K_nu(a|x|), nu = lambda - 1/2:
// integer lambda <= 9 by the half-integer closed form of K (A&S 10.2.15), any
// other lambda by K_nu of real order (Temme's series for x <= 2, Steed's
// continued fraction CF2 beyond, forward recurrence in the order; reading R29).
//
// The map Q solves the Recycling ODE with an exponential base (P:104-114,
// P:330-345):   right (v > 0):  Q'' + (a-b) Q' = H(Q) Q'^2
//               left  (v < 0):  Q'' - (a+b) Q' = H(Q) Q'^2
// with Q(0) = 0, Q'(0+-) = f0(0+-)/f(0).  Integrated forward from v = 0 this ODE
// is exponentially ill-conditioned: Q' = 1 is a repelling fixed point
// (d(Q'-1)/dv ~ (a-b)(Q'-1)), so an error e in Q'(0) grows like e^{(a-b)v}
// (reading R30).  We therefore integrate BACKWARD, in the stable direction,
// from an anchor at |v| = Vmax (base probability e^-800) where Q is fixed by its
// definition Fbar(Q(Vmax)) = p+ e^{-(a-b)Vmax} (tail mass by Gauss-Legendre
// quadrature, Newton), down to v = 0 with classical RK4 in long double,
// recording (Q, Q', Q'') at the nodes of a coarse (far tail) and a fine segment
// for quintic Hermite interpolation on the GPU.  Q(0) = 0 and the slope
// f0(0)/f(0) of P:336/P:344 come out as checks; the first unit of rate |v| is
// then redone forward from those exact centre conditions (relative accuracy
// where Q -> 0).
//
// Table layout (doubles): see qm_rode.cuh.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdint>

extern "C" {
#include <quadmath.h>
}
#include "qm_rode_params.h"

namespace qm {

typedef long double ld;

namespace {

// ------------------------------------------------ K_nu of real order (VG)
// e^x K_mu(x) and e^x K_{mu+1}(x) for |mu| <= 1/2, x > 0 (scaled by e^x so that
// the far tail, x ~ 10^3, stays in range):
//  x <= 2: Temme's series (J. Comput. Phys. 19, 1975):
//     K_mu = sum_k c_k f_k, K_{mu+1} = (2/x) sum_k c_k (p_k - k f_k), c_k = (x^2/4)^k / k!,
//     f_k = (k f_{k-1} + p_{k-1} + q_{k-1}) / (k^2 - mu^2), p_k = p_{k-1}/(k - mu), q_k = q_{k-1}/(k + mu),
//     f_0 = (mu pi / sin(mu pi)) [cosh(s) G1 + (sinh(s)/s) ln(2/x) G2], s = mu ln(2/x),
//     p_0 = (x/2)^-mu Gamma(1+mu)/2, q_0 = (x/2)^mu Gamma(1-mu)/2,
//     G1 = (1/Gamma(1-mu) - 1/Gamma(1+mu))/(2 mu), G2 = (1/Gamma(1-mu) + 1/Gamma(1+mu))/2
//     (G1, G2 in __float128; G1 -> -Euler gamma as mu -> 0);
//  x > 2: Steed's algorithm for the continued fraction CF2 (Thompson & Barnett,
//     J. Comput. Phys. 64, 1986), which gives K_mu and K_{mu+1}/K_mu together.
struct KTemme { ld mu, gam1, gam2, gampl, gammi; };

KTemme temme_setup(ld mu)
{
    KTemme t;
    t.mu = mu;
    const __float128 m = (__float128)mu;
    const __float128 gp = 1 / tgammaq(1 + m), gm = 1 / tgammaq(1 - m);
    t.gampl = (ld)gp;
    t.gammi = (ld)gm;
    t.gam2 = (ld)((gm + gp) / 2);
    t.gam1 = (fabsq(m) < 1e-12Q) ? -0.57721566490153286060651209008240243L : (ld)((gm - gp) / (2 * m));
    return t;
}

void bessel_k_pair_scaled(const KTemme &T, ld x, ld *kmu, ld *kmu1)
{
    const ld mu = T.mu, EPS = 1e-21L;
    if (x <= 2.0L) {
        const ld x2 = 0.5L * x, pimu = M_PIl * mu;
        const ld fact = (fabsl(pimu) < 1e-18L) ? 1.0L : pimu / sinl(pimu);
        ld d = -logl(x2);
        ld e = mu * d;
        const ld fact2 = (fabsl(e) < 1e-18L) ? 1.0L : sinhl(e) / e;
        ld ff = fact * (T.gam1 * coshl(e) + T.gam2 * fact2 * d);
        ld sum = ff;
        e = expl(e);
        ld p = 0.5L * e / T.gampl, q = 0.5L / (e * T.gammi), c = 1.0L;
        d = x2 * x2;
        ld sum1 = p;
        for (int i = 1; i < 400; ++i) {
            ff = ((ld)i * ff + p + q) / ((ld)i * (ld)i - mu * mu);
            c *= d / (ld)i;
            p /= ((ld)i - mu);
            q /= ((ld)i + mu);
            const ld del = c * ff;
            sum += del;
            sum1 += c * p - (ld)i * del;
            if (fabsl(del) < fabsl(sum) * EPS) break;
        }
        const ld ex = expl(x);
        *kmu = sum * ex;
        *kmu1 = sum1 * (2.0L / x) * ex;
        return;
    }
    ld b = 2.0L * (1.0L + x), d = 1.0L / b, h = d, delh = d, q1 = 0.0L, q2 = 1.0L;
    const ld a1 = 0.25L - mu * mu;
    ld q = a1, c = a1, a = -a1, s = 1.0L + q * delh;
    for (int i = 2; i < 100000; ++i) {
        a -= 2.0L * (ld)(i - 1);
        c = -a * c / (ld)i;
        const ld qnew = (q1 - b * q2) / a;
        q1 = q2;
        q2 = qnew;
        q += c * qnew;
        b += 2.0L;
        d = 1.0L / (b + a * d);
        delh = (b * d - 1.0L) * delh;
        h += delh;
        const ld dels = q * delh;
        s += dels;
        if (fabsl(dels / s) < EPS) break;
    }
    h = a1 * h;
    *kmu = sqrtl(M_PIl / (2.0L * x)) / s;
    *kmu1 = *kmu * (mu + x + 0.5L - h) / x;
}

// e^x K_{nu-1}(x) and e^x K_nu(x) for nu >= 1/2 (forward recurrence from mu = nu - round(nu))
struct KReal {
    ld nu = 0.5L;
    int nl = 1;
    KTemme T{};
    void setup(ld nu_)
    {
        nu = nu_;
        nl = (int)(nu_ + 0.5L);
        T = temme_setup(nu_ - (ld)nl);
    }
    void pair(ld x, ld *km1, ld *k) const
    {
        ld a, b;                                             // (K_{mu+j}, K_{mu+j+1})
        bessel_k_pair_scaled(T, x, &a, &b);
        for (int j = 0; j < nl - 1; ++j) {
            const ld nx = 2.0L * (T.mu + (ld)(j + 1)) / x * b + a;
            a = b;
            b = nx;
        }
        *km1 = a;
        *k = b;
    }
};

struct Target {
    int kind;            // QM_RODE_HYPERBOLIC / QM_RODE_VG
    ld a, b, d;          // alpha, beta, delta (delta unused for VG)
    int m;               // VG with integer lambda <= 9: lambda - 1; -1: real lambda (Bessel path)
    ld c[QM_RODE_VG_MAXM + 1];   // VG: polynomial coefficients of S(|x|)
    ld nu = 0.5L, log_f0 = 0.0L; // VG real lambda: nu = lambda - 1/2, log of the x -> 0 limit of |x|^nu K_nu(a|x|)
    KReal K;

    // log of the unnormalised density
    ld logg(ld x) const
    {
        if (kind == QM_RODE_HYPERBOLIC) return -a * sqrtl(d * d + x * x) + b * x;
        if (m < 0) {                                         // e^{bx} |x|^nu K_nu(a|x|)
            const ld ax = fabsl(x);
            if (ax == 0.0L) return log_f0;
            ld km1, k;
            K.pair(a * ax, &km1, &k);
            return b * x + nu * logl(ax) + logl(k) - a * ax;
        }
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
        if (m < 0) {   // -(log f)' = -b + sign a K_{nu-1}(a|x|)/K_nu(a|x|); the ratio -> 0 at x = 0 (nu > 1/2)
            const ld ax = fabsl(x);
            if (ax == 0.0L) return -b;
            ld km1, k;
            K.pair(a * ax, &km1, &k);
            return -b + (ld)dir * a * (km1 / k);
        }
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
    int k0 = 0;
    if (x == 0.0L && t.kind == QM_RODE_VG && t.m < 0) {
        // real-order VG: |x|^nu K_nu(a|x|) = A(x^2) + |x|^(2 nu) B(x^2) (+ a log for integer
        // nu) is not smooth at 0, so the first panel is cut geometrically towards 0
        // (each sub-panel is smooth on its own scale; 2^-64 w is below the ld floor)
        for (int j = 64; j >= 0; --j) {
            const ld a0 = ldexpl(w, -j - 1), a1 = ldexpl(w, -j);
            s += (dir > 0) ? gl10(t, a0, a1, shift) : gl10(t, -a1, -a0, shift);
        }
        k0 = 1;
    }
    for (int k = k0; k < 400000; ++k) {
        const ld lo = (dir > 0) ? x + k * w : x - (k + 1) * w;
        const ld p = gl10(t, lo, lo + w, shift);
        s += p;
        if (p < 1e-22L * s) break;
    }
    return s;
}

// centre nodes on octave levels (qm_rode_params.h): level 0 = [0, Wc 2^-L] and level
// l = [Wc 2^(l-L-1), Wc 2^(l-L)], each cut into QM_RODE_OCT_NODES uniform intervals, so
// that the spacing follows w (relative accuracy where Q -> 0) and the kernel finds the
// level and the local coordinate from the exponent and mantissa bits of w/Wc
ld oct_node(ld Wc, int k)
{
    const int L = QM_RODE_OCT_LEVELS - 1, n = QM_RODE_OCT_NODES;
    const int l = k / n, i = k - l * n;
    if (l == 0) return Wc * ldexpl((ld)i / n, -L);
    return Wc * ldexpl(1.0L + (ld)i / n, l - L - 1);
}
// first node index with w > wf (nodes below it come from the forward sweep)
int oct_first_above(ld Wc, ld wf)
{
    int k = 0;
    while (k < QM_RODE_CENTRE_NODES && oct_node(Wc, k) <= wf) ++k;
    return k;
}

}  // namespace

bool rode_table_build(int kind, const double *params, double *tab)
{
    Target t{};
    t.kind = kind;
    if (kind == QM_RODE_HYPERBOLIC) {
        t.a = params[0]; t.b = params[1]; t.d = params[2];
        if (!(t.a > 0 && fabsl(t.b) < t.a && t.d > 0)) return false;
    } else if (kind == QM_RODE_VG) {
        const double lam = params[0];
        t.a = params[1]; t.b = params[2];
        if (!(lam >= 1 && lam <= QM_RODE_VG_LAMBDA_MAX && t.a > 0 && fabsl(t.b) < t.a)) return false;
        if (lam != std::floor(lam) || lam > QM_RODE_VG_MAXM + 1) {
            if (lam < QM_RODE_VG_LAMBDA_MIN_REAL) return false;
            t.m = -1;
            t.nu = (ld)lam - 0.5L;
            t.K.setup(t.nu);
            // |x|^nu K_nu(a|x|) -> Gamma(nu) 2^(nu-1) a^-nu as x -> 0 (nu > 0)
            t.log_f0 = lgammal(t.nu) + (t.nu - 1.0L) * logl(2.0L) - t.nu * logl(t.a);
        } else {
            t.m = (int)lam - 1;
        }
        // K_{m+1/2}(z) = sqrt(pi/2z) e^-z sum_k (m+k)!/(k!(m-k)!) (2z)^-k  (A&S 10.2.15), so
        // f ~ e^{bx - a|x|} sum_k (m+k)!/(k!(m-k)!) (2a)^-k |x|^{m-k};  c[j] multiplies |x|^j
        for (int k = 0; k <= t.m; ++k) {   // (m < 0, real lambda: no polynomial)
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
    const int Nc = QM_RODE_CENTRE_NODES, N = QM_RODE_NODES, M = QM_RODE_TAIL_NODES, NT = QM_RODE_NT;
    std::memset(tab, 0, QM_RODE_HEADER * sizeof(double));

    // Centre segment: node k at w_k = Wc (k/Nc)^g (qm_rode_params.h).
    // Centre nodes at w_k = Wc (k/Nc)^4 (quartic grading):
    //  - Wc = 10/rate (hyperbolic, integer-lambda VG): the segment holds 99.995 % of
    //    the base samples, so the kernel finds nearly every node in shared memory.  In
    //    the node coordinate s the map is Q'(0) G s^4 + ... (G = Wc/Nc^4 = 7e-14/rate):
    //    fine where Q -> 0 needs relative accuracy (a quadratic grading, G = Wc/Nc^2,
    //    left the s^6 term's interpolation error at 2e-13 of Q in the first interval),
    //    and 4 Wc/Nc = 0.01/rate apart at the far end.
    //  - Wc = 2/rate (real-order VG): the density is A(x^2) + |x|^(2 nu) B(x^2) at
    //    the origin (R29), so the map has a v^(2 lambda) term there; in s it becomes
    //    s^(8 lambda) (smooth to the 6th order), the regular w^2 term s^8.
    const bool real_order = (t.kind == QM_RODE_VG && t.m < 0);
    for (int side = 0; side < 2; ++side) {
        const ld rate = side == 0 ? rr : rl, p = side == 0 ? pp : pm;
        const int dir = side == 0 ? +1 : -1;
        // segments: centre [0, Wc], fine [Wc, V], coarse [V, Vmax] (qm_rode_params.h)
        const ld Wc = (real_order ? QM_RODE_VRATE_C : QM_RODE_VRATE_CQ) / rate, V = QM_RODE_VRATE / rate,
                 Vmax = QM_RODE_VRATE2 / rate;
        const ld w0[3] = {0.0L, Wc, V}, w1[3] = {Wc, V, Vmax};
        const int k0[3] = {0, Nc, Nc + N}, nseg[3] = {Nc, N, M};
        ld hs[3];
        for (int j = 0; j < 3; ++j) {
            hs[j] = (w1[j] - w0[j]) / nseg[j];
            double *rec = tab + QM_RODE_SEG + 8 * (3 * side + j);
            rec[0] = (double)w0[j];
            rec[1] = (double)hs[j];
            rec[2] = (double)(1.0L / hs[j]);
            rec[3] = k0[j];
            rec[4] = nseg[j];
            rec[5] = (double)w1[j];
            if (j == 0) {
                rec[2] = (double)(1.0L / Wc);
                if (real_order) {                 // kernel: s = n (w / Wc)^(1/4), w_s = 4 G s^3, G = Wc/n^4
                    rec[6] = (double)(Wc / ((ld)Nc * Nc * Nc * Nc));
                    rec[7] = 4.0;
                } else {                          // octave levels
                    rec[7] = 1.0;
                }
            }
        }
        auto wnode = [&](int k) {                 // centre node positions
            if (!real_order) return oct_node(Wc, k);
            const ld x = (ld)k / (ld)Nc;
            return Wc * (x * x) * (x * x);
        };
        // nodes 0..kf-1 come from the forward sweep from the exact centre conditions
        // (error growth e^{rate w} <= e^2 there), nodes kf.. from the backward sweep
        const int kf = real_order ? Nc : oct_first_above(Wc, QM_RODE_VRATE_FWD / rate);
        auto seg_of = [&](int k) { return k >= k0[2] ? 2 : (k >= k0[1] ? 1 : 0); };   // interval [k, k+1]

        // anchor: tail mass of the target beyond Q(Vmax) equals the base's, p e^{-rate Vmax}
        const ld target = p * expl(-rate * Vmax) * Z;         // in units of e^{shift}
        ld q = dir * (Vmax + 1.0L);                            // Q ~ v + const
        for (int it = 0; it < 100; ++it) {
            const ld g = tail_mass(t, q, dir, rate, shift) - target;
            const ld fq = expl(t.logg(q) - shift);
            const ld step = g / fq;                            // d(tail)/dq = -dir f(q)
            q += dir * step;
            if (fabsl(step) <= 1e-18L * fabsl(q)) break;
        }
        // Q'(Vmax) = f0(Vmax)/f(Q(Vmax)) (first-order quantile ODE), in |v| units
        ld Q = q;
        ld P = dir * (p * rate * expl(-rate * Vmax) * Z) / expl(t.logg(q) - shift);
        // integrate R(w) = Q(dir w), w = |v|, backward from w = Vmax to 0:
        //   R'' = H(R) R'^2 - rate R'   (both sides, with R' = dR/dw)
        double *nodes = tab + QM_RODE_HEADER + side * 4 * (NT + 1);
        auto put = [&](int k, ld q, ld p) {
            nodes[4 * k] = (double)q;
            nodes[4 * k + 1] = (double)p;
            nodes[4 * k + 2] = (double)(t.H(q, dir) * p * p - rate * p);   // R'' from the RODE
            nodes[4 * k + 3] = 0.0;
        };
        put(NT, Q, P);
        const int sub = QM_RODE_SUBSTEPS;
        // one classical RK4 step of length s for (R, R'); the state updates are
        // compensated (Kahan): ~10^5 steps with |Q| up to ~800/rate would otherwise
        // accumulate a systematic rounding drift of ~1e-13 in Q
        ld cQ = 0.0L, cP = 0.0L;
        auto acc = [](ld &x, ld &c, ld dx) {
            const ld y = dx - c, tx = x + y;
            c = (tx - x) - y;
            x = tx;
        };
        auto rk4 = [&](ld &Q, ld &P, ld s) {
            const ld k1q = P, k1p = t.H(Q, dir) * P * P - rate * P;
            const ld q2 = Q + 0.5L * s * k1q, p2 = P + 0.5L * s * k1p;
            const ld k2q = p2, k2p = t.H(q2, dir) * p2 * p2 - rate * p2;
            const ld q3 = Q + 0.5L * s * k2q, p3 = P + 0.5L * s * k2p;
            const ld k3q = p3, k3p = t.H(q3, dir) * p3 * p3 - rate * p3;
            const ld q4 = Q + s * k3q, p4 = P + s * k3p;
            const ld k4q = p4, k4p = t.H(q4, dir) * p4 * p4 - rate * p4;
            acc(Q, cQ, s / 6.0L * (k1q + 2.0L * k2q + 2.0L * k3q + k4q));
            acc(P, cP, s / 6.0L * (k1p + 2.0L * k2p + 2.0L * k3p + k4p));
        };
        // backward: coarse, fine, then the centre (stored down to node kf; the rest of
        // the sweep gives the checks at v = 0)
        ld Qc = 0.0L;
        constexpr int NG = 4800;                               // r = 1.005: h0 r^-4800 ~ 4e-11 h0 (r = 1.12 left 1e-13 at lambda = 1.5,
                                                               // 1.02 left 5e-15 at lambda = 1.2; 1.005 converged to 1e-17 at 1.1)
        const ld rg = 1.005L;
        // one centre interval [w_k, w_{k+1}] forward (dir_s = +1) or backward (-1) on
        // geometric substeps (ratio <= rg; at least nmin), the first one down to 4e-11 of
        // w_1 next to v = 0 (real-order VG: H has a |Q|^(2 nu - 1) or Q log Q term there,
        // and RK4's error scales with the local step over the distance to 0)
        auto centre_interval = [&](int k, int dir_s, int nmin) {
            const ld wa = wnode(k), wb = wnode(k + 1);
            if (k == 0) {
                if (dir_s > 0) {
                    ld w = 0.0L;
                    for (int i = NG; i >= 1; --i) { const ld wn = wb * powl(rg, -(ld)i); rk4(Q, P, wn - w); w = wn; }
                    rk4(Q, P, wb - w);
                } else {
                    ld w = wb;
                    for (int i = 1; i <= NG; ++i) { const ld wn = wb * powl(rg, -(ld)i); rk4(Q, P, wn - w); w = wn; }
                    rk4(Q, P, -w);
                }
                return;
            }
            const int ns = std::max(nmin, (int)ceill(logl(wb / wa) / logl(rg)));
            ld w = dir_s > 0 ? wa : wb;
            for (int i = 1; i <= ns; ++i) {
                const ld x = (ld)i / (ld)ns;
                const ld wn = (i == ns) ? (dir_s > 0 ? wb : wa) : (dir_s > 0 ? wa * powl(wb / wa, x) : wb * powl(wa / wb, x));
                rk4(Q, P, wn - w);
                w = wn;
            }
        };
        for (int k = NT - 1; k >= 0; --k) {
            if (k < Nc) {
                centre_interval(k, -1, k >= kf ? 4 * sub : sub);
            } else {
                const ld hk = hs[seg_of(k)];
                for (int j = 0; j < sub; ++j) rk4(Q, P, -hk / sub);
            }
            if (k >= kf) put(k, Q, P);
            if (k == kf) Qc = Q;
        }
        // checks against the centre conditions of P:336 / P:344
        const ld slope0 = dir * p * rate * Z / expl(t.logg(0.0L) - shift);
        tab[12 + side] = (double)Q;                            // residual Q(0)
        tab[14 + side] = (double)(P / slope0 - 1.0L);          // relative slope residual
        // Near the centre the backward sweep's accumulated ABSOLUTE error (~1e-14) is a
        // large RELATIVE error because Q -> 0.  There the forward direction is benign over
        // a short distance (error growth e^{rate w} <= e^2 for rate w <= 2), so nodes
        // 0..kf-1 are integrated forward from the exact conditions Q(0) = 0,
        // Q'(0) = slope0 (node kf keeps the backward value; the mismatch is recorded).
        Q = 0.0L;
        P = slope0;
        cQ = cP = 0.0L;
        put(0, Q, P);
        for (int k = 1; k <= kf; ++k) {
            centre_interval(k - 1, +1, 4 * sub);
            if (k < kf) put(k, Q, P);
        }
        tab[22 + side] = (double)(Q - Qc);                     // joint mismatch at node kf
        tab[8 + side] = (double)p;
        tab[10 + side] = (double)rate;
        const ld lp = logl(p);
        tab[16 + side] = (double)lp;                           // log p_s as a double-double
        tab[18 + side] = (double)(lp - (ld)(double)lp);
        tab[20 + side] = (double)(1.0L / rate);
        tab[28 + side] = (double)Vmax;
    }
    tab[0] = kind;
    tab[1] = NT;
    if (t.kind == QM_RODE_HYPERBOLIC) {   // the kernel's R'' = H(R) R'^2 - rate R' (rode_hyp_d2)
        tab[3] = (double)t.a;
        tab[4] = (double)t.b;
        tab[5] = (double)(t.d * t.d);
    }
    tab[30] = 3;
    return true;
}

// ------------------------------------------------ Gaussian base: Student t (§3.6)
// The "purely numerical method" of P:282-283: the Student Recycling ODE
// with the Gaussian base (H^(v) = v), solved numerically once per nu
// and sampled by interpolation.  On the right side (w = v >= 0):
//     R'' = H(R) R'^2 - w R',   H(R) = (1 + 1/n) R / (1 + R^2/n)
// and R(-w) = -R(w) (both distributions are symmetric).  Forward from the centre
// conditions R(0) = 0, R'(0) = gamma the error grows like e^{w^2/2}:
// the tail equation's neighbours R^-n = A + B erfc(w/sqrt2) saturate,
// so a relative error e at w leaves e e^{w^2/2}/... at the far tail (the paper's
// own claim stops at |z| < 6).  As for the exponential base (R30) the table is
// integrated BACKWARD from an anchor in the far tail, w = 38.5 (beyond the
// largest |z| a double uniform can give, 38.47), where R is fixed by its
// definition Fbar_n(R) = Phibar(w): Fbar_n by its convergent large-t series
//     Fbar_n(t) = k_n n^((n+1)/2) sum_j binom(-(n+1)/2, j) n^j t^-(n+2j) / (n+2j),
//     k_n = Gamma((n+1)/2) / (sqrt(n pi) Gamma(n/2))     (t^2 > n; Newton in log t),
// and R' = phi(w)/f_n(R) (the quantile ODE).  In the tail the sweep runs
// in G = log R (R reaches 1e324 at nu = 1):
//     G'' = G'^2 n (1 - e^-2G) / (1 + n e^-2G) - w G',
// which is nearly quadratic (G ~ w^2/(2n)).  Segments: centre [0, 4.5] with nodes at
// 4.5 (k/Nc)^4 (R; the nodes with w <= 2 forward from the exact centre conditions;
// 1 - 7e-6 of the samples), fine [4.5, 9] (R), coarse [9, 38.5] in LOG values (G, G',
// G''), which the kernel exponentiates (table[31] = 1; 2e-19 of the samples);
// beyond 38.5 log-linear extrapolation.
namespace {
typedef __float128 f128;

struct StudentRode {
    ld n;
    // log k_n, gamma = sqrt(n/2) Gamma(n/2)/Gamma((n+1)/2) (in __float128: lgamma
    // differences lose the digits of lgamma's size in long double at large n)
    ld logk, gam;
    explicit StudentRode(ld nn) : n(nn)
    {
        const f128 q = (f128)nn;
        const f128 lr = lgammaq(q / 2) - lgammaq((q + 1) / 2);           // log Gamma(n/2)/Gamma((n+1)/2)
        gam = (ld)(sqrtq(q / 2) * expq(lr));
        logk = (ld)(-lr - 0.5Q * logq(q * M_PIq));
    }
    ld H(ld r) const { return (1.0L + 1.0L / n) * r / (1.0L + r * r / n); }
    // log f_n(t) and log Fbar_n(t) for t^2 >> n
    ld log_pdf(ld t) const { return logk - 0.5L * (n + 1.0L) * log1pl(t * t / n); }
    ld log_sf_tail(ld t) const
    {
        const ld x = n / (t * t);
        ld s = 0.0L, c = 1.0L, xp = 1.0L;                                // c = binom(-(n+1)/2, j)
        for (int j = 0; j < 200; ++j) {
            const ld term = c * xp / (n + 2.0L * j);
            s += term;
            if (fabsl(term) < 1e-22L * fabsl(s)) break;
            c *= (-(n + 1.0L) / 2.0L - (ld)j) / (ld)(j + 1);
            xp *= x;
        }
        return logk + 0.5L * (n + 1.0L) * logl(n) - n * logl(t) + logl(s);
    }
};
}  // namespace

bool rode_student_table_build(double nu, double *tab)
{
    if (!(nu >= QM_RODE_STUDENT_NU_MIN && nu <= QM_RODE_STUDENT_NU_MAX)) return false;
    const StudentRode T((ld)nu);
    const ld n = (ld)nu;
    const int Nc = QM_RODE_CENTRE_NODES, N = QM_RODE_NODES, M = QM_RODE_TAIL_NODES, NT = QM_RODE_NT;
    const ld Wc = QM_RODE_STUDENT_WC, V = QM_RODE_STUDENT_V, Vmax = QM_RODE_STUDENT_VMAX;
    auto wnode = [&](int k) { return oct_node(Wc, k); };                 // centre nodes (octave levels)
    const int kf = oct_first_above(Wc, QM_RODE_STUDENT_WF);             // forward: nodes < kf
    std::memset(tab, 0, QM_RODE_HEADER * sizeof(double));
    // node layout: centre 0..Nc and fine Nc..Nc+N in R (sharing node Nc), coarse
    // Nc+N+1..NT in log |R| (M - 1 intervals; its first node repeats w = V in log form,
    // so that no interval mixes linear and log values)
    const ld w0[3] = {0.0L, Wc, V}, w1[3] = {Wc, V, Vmax};
    const int k0[3] = {0, Nc, Nc + N + 1}, nseg[3] = {Nc, N, M - 1};
    ld hs[3];
    for (int j = 0; j < 3; ++j) hs[j] = (w1[j] - w0[j]) / nseg[j];

    // anchor: Fbar_n(R) = Phibar(Vmax) = erfc(Vmax/sqrt2)/2, Newton in x = log R
    const ld lp = logl(0.5L * erfcl(Vmax * 0.707106781186547524400844362104849039L));
    ld x = (T.logk + 0.5L * (n - 1.0L) * logl(n) - lp) / n;             // leading term
    for (int it = 0; it < 60; ++it) {
        const ld t = expl(x);
        const ld g = T.log_sf_tail(t) - lp;
        const ld dg = -expl(x + T.log_pdf(t) - T.log_sf_tail(t));       // d log Fbar / d log t
        const ld dx = g / dg;
        x -= dx;
        if (fabsl(dx) <= 1e-19L * fabsl(x)) break;
    }
    const ld lphi = -0.5L * Vmax * Vmax - 0.918938533204672741780329736405617639L;   // log phi(Vmax)
    ld G = x, Gp = expl(lphi - T.log_pdf(expl(x)) - x);                  // G' = R'/R = phi/(f R)

    double *nodes = tab + QM_RODE_HEADER;                                // side 0; side 1 = -side 0
    auto Gpp = [&](ld w, ld g, ld gp) {
        const ld e = expl(-2.0L * g);
        return gp * gp * n * (1.0L - e) / (1.0L + n * e) - w * gp;
    };
    auto put_log = [&](int k, ld w, ld g, ld gp) {
        nodes[4 * k] = (double)g; nodes[4 * k + 1] = (double)gp; nodes[4 * k + 2] = (double)Gpp(w, g, gp);
        nodes[4 * k + 3] = 0.0;
    };
    auto put_lin = [&](int k, ld w, ld r, ld rp) {
        nodes[4 * k] = (double)r; nodes[4 * k + 1] = (double)rp;
        nodes[4 * k + 2] = (double)(T.H(r) * rp * rp - w * rp); nodes[4 * k + 3] = 0.0;
    };
    // classical RK4 (Kahan-compensated state) on y' = F(w, y) for two components
    ld c0 = 0.0L, c1 = 0.0L;
    auto acc = [](ld &v, ld &c, ld dv) { const ld y = dv - c, t = v + y; c = (t - v) - y; v = t; };
    auto rk4 = [&](auto F, ld &a, ld &b, ld w, ld s) {
        ld k1a, k1b, k2a, k2b, k3a, k3b, k4a, k4b;
        F(w, a, b, k1a, k1b);
        F(w + 0.5L * s, a + 0.5L * s * k1a, b + 0.5L * s * k1b, k2a, k2b);
        F(w + 0.5L * s, a + 0.5L * s * k2a, b + 0.5L * s * k2b, k3a, k3b);
        F(w + s, a + s * k3a, b + s * k3b, k4a, k4b);
        acc(a, c0, s / 6.0L * (k1a + 2.0L * k2a + 2.0L * k3a + k4a));
        acc(b, c1, s / 6.0L * (k1b + 2.0L * k2b + 2.0L * k3b + k4b));
    };
    auto Flog = [&](ld w, ld g, ld gp, ld &dg, ld &dgp) { dg = gp; dgp = Gpp(w, g, gp); };
    auto Flin = [&](ld w, ld r, ld rp, ld &dr, ld &drp) { dr = rp; drp = T.H(r) * rp * rp - w * rp; };
    const int sub = QM_RODE_SUBSTEPS;

    // backward in G from Vmax down to Wc: coarse nodes in log values, fine nodes in R
    put_log(NT, Vmax, G, Gp);
    for (int i = nseg[2] - 1; i >= 0; --i) {
        const ld wa = w0[2] + (ld)(i + 1) * hs[2];
        for (int j = 0; j < sub; ++j) rk4(Flog, G, Gp, wa - (ld)j * hs[2] / sub, -hs[2] / sub);
        put_log(k0[2] + i, w0[2] + (ld)i * hs[2], G, Gp);
    }
    put_lin(k0[1] + nseg[1], V, expl(G), Gp * expl(G));
    for (int i = nseg[1] - 1; i >= 0; --i) {
        const ld wa = w0[1] + (ld)(i + 1) * hs[1];
        for (int j = 0; j < sub; ++j) rk4(Flog, G, Gp, wa - (ld)j * hs[1] / sub, -hs[1] / sub);
        put_lin(k0[1] + i, w0[1] + (ld)i * hs[1], expl(G), Gp * expl(G));
    }
    // the centre's outer nodes (w >= 2) still in log variables, node to node
    const int sc = 4 * sub;                                              // centre: 0.0027 apart at w = 2
    for (int k = Nc - 1; k >= kf; --k) {
        const ld wa = wnode(k + 1), hn = wa - wnode(k);
        for (int j = 0; j < sc; ++j) rk4(Flog, G, Gp, wa - (ld)j * hn / sc, -hn / sc);
        put_lin(k, wnode(k), expl(G), Gp * expl(G));
    }
    const ld Rc = expl(G), Rpc = Gp * expl(G);                          // backward value at node kf
    // continue backward in R to w = 0: residual checks Q(0) = 0, Q'(0) = gamma
    {
        ld R = Rc, Rp = Rpc;
        c0 = c1 = 0.0L;
        for (int k = kf - 1; k >= 0; --k) {
            const ld wa = wnode(k + 1), hn = wa - wnode(k);
            for (int i = 0; i < sc; ++i) rk4(Flin, R, Rp, wa - (ld)i * hn / sc, -hn / sc);
        }
        tab[12] = (double)R;
        tab[14] = (double)(Rp / T.gam - 1.0L);
    }
    // centre nodes 0..kf-1 forward from the exact conditions
    {
        ld R = 0.0L, Rp = T.gam;
        c0 = c1 = 0.0L;
        put_lin(0, 0.0L, R, Rp);
        for (int k = 1; k <= kf; ++k) {
            const ld wa = wnode(k - 1), hn = wnode(k) - wa;
            for (int i = 0; i < sc; ++i) rk4(Flin, R, Rp, wa + (ld)i * hn / sc, hn / sc);
            if (k < kf) put_lin(k, wnode(k), R, Rp);
        }
        tab[22] = (double)(R / Rc - 1.0L);                               // relative joint mismatch at node kf
    }
    // side 1: the odd reflection (log values: log |R|, same G', G'')
    double *left = tab + QM_RODE_HEADER + 4 * (NT + 1);
    for (int k = 0; k <= NT; ++k) {
        const bool lg = k >= k0[2];                                      // log |R|: G, G', G'' even
        left[4 * k] = lg ? nodes[4 * k] : -nodes[4 * k];
        left[4 * k + 1] = lg ? nodes[4 * k + 1] : -nodes[4 * k + 1];
        left[4 * k + 2] = lg ? nodes[4 * k + 2] : -nodes[4 * k + 2];
        left[4 * k + 3] = 0.0;
    }
    for (int side = 0; side < 2; ++side) {
        for (int j = 0; j < 3; ++j) {
            double *rec = tab + QM_RODE_SEG + 8 * (3 * side + j);
            rec[0] = (double)w0[j]; rec[1] = (double)hs[j]; rec[2] = (double)(1.0L / hs[j]);
            rec[3] = k0[j]; rec[4] = nseg[j]; rec[5] = (double)w1[j];
            if (j == 0) {                                                // octave levels
                rec[2] = (double)(1.0L / Wc);
                rec[7] = 1.0;
            }
        }
        tab[8 + side] = 0.5;
        tab[10 + side] = 1.0;
        tab[13] = tab[12]; tab[15] = tab[14]; tab[23] = tab[22];
        tab[28 + side] = (double)Vmax;
    }
    tab[0] = QM_RODE_STUDENT;
    tab[1] = NT;
    tab[2] = nu;
    tab[30] = 3;
    tab[31] = 1.0;                                                       // segment 2 holds log |R|
    return true;
}

}  // namespace qm

// host-side table (diagnostics and the CPU-side tests of the builder)
extern "C" int qm_rode_table_host(int kind, const double *params, double *table)
{
    if (kind == QM_RODE_STUDENT) return (params && qm::rode_student_table_build(params[0], table)) ? 0 : 1;
    return qm::rode_table_build(kind, params, table) ? 0 : 1;
}
