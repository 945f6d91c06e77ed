/*
 * orc_rode.c -- ORACLE (test infrastructure only; see orc.h).
 *
 * recycling two-sided exponential samples into
 * hyperbolic (§4.1) and variance-gamma (§4.2) samples.
 * The oracle states the map by its DEFINITION: Q(v) = F^-1(F0(v)), with
 *   base f0(x) = p+ (a-b) e^{-(a-b)x} (x > 0), p- (a+b) e^{(a+b)x} (x < 0)
 *   hyperbolic f(x) ~ exp(-a sqrt(d^2 + x^2) + b x)
 *   VG: f(x) ~ e^{bx} |x|^{nu} K_{nu}(a|x|), nu = lambda - 1/2, lambda >= 1
 *      integer lambda = m+1 <= 9: the half-integer closed form (A&S 10.2.15)
 *      = e^{bx - a|x|} sum_{k=0}^{m} (m+k)!/(k!(m-k)!) (2a)^{-k} |x|^{m-k};
 *      any other lambda (reading R29): K_nu by its integral representation
 *      K_nu(z) = int_0^inf exp(-z cosh t) cosh(nu t) dt (A&S 9.6.24) with the
 *      trapezoidal rule (the integrand is entire and decays double-exponentially,
 *      so the rule converges geometrically in 1/h: error ~ exp(-2 pi^2/(h^2 z))
 *      relative for large z, exp(-pi^2/h) otherwise; h = min(1/8, 1/(2 sqrt z))).
 * p+- = target masses of x > 0 / x < 0, computed here by
 * adaptive Gauss-Kronrod (7-15) quadrature of the unnormalised density; the
 * tail masses by the same quadrature; Q by bracketed bisection on the TAIL
 * probability (never 1 - F):  v >= 0: Fbar(Q) = p+ e^{-(a-b) v};
 *                             v <  0: F(Q)    = p- e^{(a+b) v}.
 * Long double throughout.
 */
#include <math.h>
#include <stdint.h>
#include <float.h>
#include "orc.h"

typedef struct { int kind; ld a, b, d; int m; ld nu; } tgt_t;   /* kind 1 hyperbolic, 2 VG; m < 0: real lambda */

/* K_nu(z), z > 0, by the trapezoidal rule on int_0^inf exp(-z cosh t) cosh(nu t) dt */
static ld besselk_trap(ld nu, ld z)
{
    const ld h = (z > 16.0L) ? 0.5L / sqrtl(z) : 0.125L;
    ld s = 0.5L * expl(-z);                              /* t = 0 (half weight: the integrand is even) */
    for (int k = 1; k < 1000000; ++k) {
        const ld t = (ld)k * h;
        const ld term = expl(-z * coshl(t)) * coshl(nu * t);
        s += term;
        if (z * sinhl(t) > nu && term <= 1e-22L * s) break;   /* past the peak, converged */
    }
    return h * s;
}

double orc_besselk(double nu, double z) { return (double)besselk_trap((ld)nu, (ld)z); }
void orc_besselk_ld(double nu, double z, ld *out) { *out = besselk_trap((ld)nu, (ld)z); }

static ld dens_u(const tgt_t *t, ld x)                   /* unnormalised density */
{
    if (t->kind == 1) return expl(-t->a * sqrtl(t->d * t->d + x * x) + t->b * x);
    if (t->m < 0) {                                      /* real lambda: e^{bx} |x|^nu K_nu(a|x|) */
        const ld ax = fabsl(x);
        if (ax == 0.0L) return tgammal(t->nu) * powl(2.0L, t->nu - 1.0L) * powl(t->a, -t->nu);   /* the limit */
        return expl(t->b * x) * powl(ax, t->nu) * besselk_trap(t->nu, t->a * ax);
    }
    ld ax = fabsl(x), s = 0.0L, fact_mk = 1.0L;
    /* sum_{k=0}^{m} (m+k)!/(k!(m-k)!) (2a)^-k |x|^{m-k} */
    for (int k = 0; k <= t->m; ++k) {
        ld c = 1.0L;
        for (int j = t->m - k + 1; j <= t->m + k; ++j) c *= (ld)j;      /* (m+k)!/(m-k)! */
        for (int j = 2; j <= k; ++j) c /= (ld)j;                          /* /k! */
        s += c * powl(2.0L * t->a, -(ld)k) * powl(ax, (ld)(t->m - k));
    }
    (void)fact_mk;
    return expl(t->b * x - t->a * ax) * s;
}

/* Gauss-Kronrod 7-15 on [lo, hi], adaptive (absolute tolerance relative to the running total) */
static const ld XK[8] = {0.991455371120812639206854697526329L, 0.949107912342758524526189684047851L,
                         0.864864423359769072789712788640926L, 0.741531185599394439863864773280788L,
                         0.586087235467691130294144845693013L, 0.405845151377397166906606412076961L,
                         0.207784955007898467600689403773245L, 0.0L};
static const ld WK[8] = {0.022935322010529224963732008058970L, 0.063092092629978553290700663189204L,
                         0.104790010322250183839876322541518L, 0.140653259715525918745189590510238L,
                         0.169004726639267902826583426598550L, 0.190350578064785409913256402421014L,
                         0.204432940075298892414161999234649L, 0.209482141084727828012999174891714L};
static const ld WG[4] = {0.129484966168869693270611432679082L, 0.279705391489276667901467771423780L,
                         0.381830050505118944950369775488975L, 0.417959183673469387755102040816327L};

static ld gk15(const tgt_t *t, ld lo, ld hi, ld *err)
{
    ld c = 0.5L * (lo + hi), h = 0.5L * (hi - lo);
    ld fc = dens_u(t, c), rk = WK[7] * fc, rg = WG[3] * fc;
    for (int j = 0; j < 7; ++j) {
        ld f1 = dens_u(t, c - h * XK[j]), f2 = dens_u(t, c + h * XK[j]);
        rk += WK[j] * (f1 + f2);
        if (j % 2 == 1) rg += WG[j / 2] * (f1 + f2);
    }
    *err = fabsl((rk - rg) * h);
    return rk * h;
}

static ld integ(const tgt_t *t, ld lo, ld hi, ld tol, int depth)
{
    ld e, r = gk15(t, lo, hi, &e);
    /* stop at the tolerance or at long double's rounding floor of the panel: the
       abscissae c +- h x_j carry an absolute rounding of ~eps |c|, i.e. a relative
       error of ~eps |c| |(log f)'| <= eps |c| (a + |b| + 1) in f, which the
       Kronrod-Gauss difference cannot get below */
    ld floor_rel = 8.0L * LDBL_EPSILON * (1.0L + (fabsl(lo) + fabsl(hi)) * (t->a + fabsl(t->b) + 1.0L));
    if (e <= tol || e <= floor_rel * fabsl(r) || depth > 24) return r;
    ld m = 0.5L * (lo + hi);
    return integ(t, lo, m, 0.5L * tol, depth + 1) + integ(t, m, hi, 0.5L * tol, depth + 1);
}

/* integral over [x, inf) (right) or (-inf, x] (left), panels of 1/rate out to 120/rate */
static ld tail_int(const tgt_t *t, ld x, int right)
{
    ld rate = right ? (t->a - t->b) : (t->a + t->b);
    ld w = 1.0L / rate, s = 0.0L, scale = dens_u(t, x) * w + 1e-4900L;
    for (int k = 0; k < 160; ++k) {
        ld lo = right ? x + k * w : x - (k + 1) * w, hi = lo + w;
        ld p = integ(t, lo, hi, 1e-21L * scale, 0);
        s += p;
        if (p < 1e-24L * s) break;
    }
    return s;
}

static void masses(const tgt_t *t, ld *pm, ld *pp, ld *Z)
{
    ld r = tail_int(t, 0.0L, 1), l = tail_int(t, 0.0L, 0);
    *Z = r + l; *pp = r / *Z; *pm = l / *Z;
}

static int make_tgt(int kind, const double *par, tgt_t *t)
{
    t->kind = kind;
    if (kind == 1) { t->a = par[0]; t->b = par[1]; t->d = par[2]; t->m = 0; return !(par[0] > fabs(par[1]) && par[2] > 0); }
    if (kind == 2) {
        const int integer = par[0] == (int)par[0] && par[0] <= 9;
        t->m = integer ? (int)par[0] - 1 : -1; t->nu = (ld)par[0] - 0.5L; t->a = par[1]; t->b = par[2]; t->d = 0;
        return !(par[0] >= 1 && par[1] > fabs(par[2]));
    }
    return 1;
}

int orc_target_masses(int kind, const double *par, ld *out /* p-, p+, Z */)
{
    tgt_t t;
    if (make_tgt(kind, par, &t)) return -1;
    masses(&t, &out[0], &out[1], &out[2]);
    return 0;
}

/* normalised density (for the slope pins) */
int orc_target_density(int kind, const double *par, const double *x, ld *out, int64_t n)
{
    tgt_t t; ld pm, pp, Z;
    if (make_tgt(kind, par, &t)) return -1;
    masses(&t, &pm, &pp, &Z);
    for (int64_t i = 0; i < n; ++i) out[i] = dens_u(&t, (ld)x[i]) / Z;
    return 0;
}

/* Q(v) = F^-1(F0(v)) for base samples v (two-sided exponential with the target's split) */
int orc_recycle_exp_to_target(int kind, const double *par, const double *v, ld *out, int64_t n)
{
    tgt_t t; ld pm, pp, Z;
    if (make_tgt(kind, par, &t)) return -1;
    masses(&t, &pm, &pp, &Z);
    const ld rr = t.a - t.b, rl = t.a + t.b;
    for (int64_t i = 0; i < n; ++i) {
        ld vi = (ld)v[i];
        if (isnan(vi)) { out[i] = NAN; continue; }
        if (isinf(vi)) { out[i] = vi; continue; }
        if (vi == 0.0L) { out[i] = vi; continue; }
        int right = vi > 0.0L;
        ld rate = right ? rr : rl;
        if (rate * fabsl(vi) < 0.5L) {
            /* near the centre solve for the mass between 0 and Q instead (no cancellation):
               int_0^Q f = p (1 - e^{-rate |v|}) = -p expm1(-rate |v|)                    */
            ld target = -(right ? pp : pm) * expm1l(-rate * fabsl(vi));
            ld lo = 0.0L, hi = 1.0L, q;
            while (integ(&t, right ? 0.0L : -hi, right ? hi : 0.0L, 0.0L, 0) / Z < target && hi < 1e6L) { lo = hi; hi *= 2.0L; }
            q = 0.5L * (lo + hi);
            for (int it = 0; it < 200; ++it) {
                ld x = right ? q : -q;
                ld g = integ(&t, right ? 0.0L : x, right ? x : 0.0L, 0.0L, 0) / Z - target;   /* increasing in q */
                if (g > 0.0L) hi = q; else lo = q;
                ld qn = q - g / (dens_u(&t, x) / Z);
                if (!(qn > lo && qn < hi)) qn = 0.5L * (lo + hi);
                if (fabsl(qn - q) <= 4.0L * LDBL_EPSILON * qn || hi - lo <= 4.0L * LDBL_EPSILON * hi) { q = qn; break; }
                q = qn;
            }
            out[i] = right ? q : -q;
            continue;
        }
        /* target tail mass (normalised) */
        ld target = right ? pp * expl(-rr * vi) : pm * expl(rl * vi);
        /* bracket: |Q| in [0, hi] */
        ld lo = 0.0L, hi = 1.0L;
        while (tail_int(&t, right ? hi : -hi, right) / Z > target && hi < 1e6L) { lo = hi; hi *= 2.0L; }
        /* bracketed Newton on g(q) = log tail(q) - log target, g' = -f(q)/tail(q)
           (the log makes it quadratic from afar; bisection if it leaves the bracket) */
        ld q = 0.5L * (lo + hi);
        for (int it = 0; it < 200; ++it) {
            ld x = right ? q : -q;
            ld T = tail_int(&t, x, right);
            ld g = logl(T / Z) - logl(target);
            if (g > 0.0L) lo = q; else hi = q;
            ld qn = q + g * T / dens_u(&t, x);
            if (!(qn > lo && qn < hi)) qn = 0.5L * (lo + hi);
            if (fabsl(qn - q) <= 4.0L * LDBL_EPSILON * qn || hi - lo <= 4.0L * LDBL_EPSILON * hi) { q = qn; break; }
            q = qn;
        }
        out[i] = right ? q : -q;
    }
    return 0;
}
