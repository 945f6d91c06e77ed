/*
 * orc_student.c -- ORACLE (test infrastructure only; see orc.h).
 *
 * Row a6 of SURVEY.md §8: recycling standard-normal samples z into Student-t
 * samples t = A(z) = F_n^-1(Phi(z)) (§1, §3).
 *   gamma     = sqrt(n/2) Gamma(n/2)/Gamma((n+1)/2)               P:156-160 §3.1
 *   c_0 = gamma and the recurrence
 *     (2i+3)(2i+2) c_{i+1} = -(2i+1) c_i
 *        + sum_{l=0}^{i} sum_{m=0}^{i-l} a_lm(n) c_{i-l-m} c_l c_m
 *        - theta(i)/n sum_{l=0}^{i-1} sum_{m=0}^{i-1-l} (2m+1) c_{i-1-l-m} c_l c_m
 *     a_lm(n) = (1+1/n)(2l+1)(2m+1) - (2/n) m (2m+1),
 *     theta(0) = 0, theta(i>=1) = 1                                P:178-188 §3.2
 *   central series  t = z sum_{k=0}^{K} c_k y^k, y = z^2
 *   two-term tail   w = (1 - Phi(z)) n sqrt(pi) Gamma(n/2)/Gamma((n+1)/2),
 *                   t = sqrt(n) w^(-1/n) (1 - (n+1)/(2(n+2)) w^(2/n))   P:267-272 §3.5
 *   composite: central for |z| < z*, tail for |z| >= z*, odd symmetry (P:281,
 *   readings R13/R14).  orc_student_crossover() finds the first root of
 *   central(z) = tail(z) above z = 1; for n = 4, K = 10 this is the paper's
 *   3.93473.
 * The recurrence is exponentially ill-conditioned (terms of size c_i cancel to
 * c_{i+1}); long double loses 12 digits by c_16 at n = 4 and everything at
 * n = 30.  The oracle therefore runs it in mpmath at 100 digits
 * (oracle/__init__.py: student_coeffs) and the C functions below take the
 * coefficients as input.  orc_student_coeffs_ld is the same recurrence in long
 * double, kept only to document that conditioning (tests).
 * The exact map ("exact representation of the composite function")
 * solves P(T > t) = 1/2 erfc(|z|/sqrt2) with P(T > t) = 1/2 I_{n/(n+t^2)}(n/2, 1/2)
 * (the upper tail, no cancellation), or, near the centre,
 * I_{t^2/(n+t^2)}(1/2, n/2) = erf(|z|/sqrt2); the regularized incomplete beta is
 * the continued fraction of A&S 26.5.8 (Lentz evaluation).
 */
#include <math.h>
#include <stdint.h>
#include <float.h>
#include "orc.h"

static const ld PI_L = 3.14159265358979323846264338327950288L;
static const ld SQRT1_2L = 0.707106781186547524400844362104849039L;

/* Gamma(n/2)/Gamma((n+1)/2) via log-gamma differences */
static ld gamma_ratio_half(ld n)
{
    return expl(lgammal(n / 2.0L) - lgammal((n + 1.0L) / 2.0L));
}

ld orc_student_gamma_ld(double n)
{
    ld nn = (ld)n;
    return sqrtl(nn / 2.0L) * gamma_ratio_half(nn);
}

/* c_0..c_K by the recurrence of P:178-188, exactly as printed (long double) */
int orc_student_coeffs_ld(double n_, int K, ld *c)
{
    if (K < 0 || K > 64 || !(n_ > 0.0)) return -1;
    ld n = (ld)n_;
    c[0] = orc_student_gamma_ld(n_);
    for (int i = 0; i < K; ++i) {
        ld rhs = -(ld)(2 * i + 1) * c[i];
        for (int l = 0; l <= i; ++l)
            for (int m = 0; m <= i - l; ++m) {
                ld alm = (1.0L + 1.0L / n) * (ld)(2 * l + 1) * (ld)(2 * m + 1)
                         - (2.0L / n) * (ld)m * (ld)(2 * m + 1);
                rhs += alm * c[i - l - m] * c[l] * c[m];
            }
        if (i >= 1) {                                  /* theta(i) */
            ld s = 0.0L;
            for (int l = 0; l <= i - 1; ++l)
                for (int m = 0; m <= i - 1 - l; ++m)
                    s += (ld)(2 * m + 1) * c[i - 1 - l - m] * c[l] * c[m];
            rhs -= s / n;
        }
        c[i + 1] = rhs / ((ld)(2 * i + 3) * (ld)(2 * i + 2));
    }
    return 0;
}

/* central series, nested in y = z^2 as printed */
static ld central(const ld *c, int K, ld z)
{
    ld y = z * z, s = c[K];
    for (int k = K - 1; k >= 0; --k) s = c[k] + y * s;
    return z * s;
}

/* two-term tail for z > 0 */
static ld tail(ld n, ld z)
{
    ld Cn = n * sqrtl(PI_L) * gamma_ratio_half(n);
    ld w = 0.5L * erfcl(z * SQRT1_2L) * Cn;             /* (1 - Phi(z)) C_n, never 1 - Phi */
    return sqrtl(n) * powl(w, -1.0L / n) * (1.0L - (n + 1.0L) / (2.0L * (n + 2.0L)) * powl(w, 2.0L / n));
}

/* z*(n,K): first sign change of central - tail on z in (1, 12], refined by bisection */
ld orc_student_crossover_ld(double n_, int K, const ld *c)
{
    ld n = (ld)n_;
    ld h = 1.0L / 256.0L, a = 1.0L;
    ld fa = central(c, K, a) - tail(n, a);
    for (ld b = a + h; b <= 12.0L; b += h) {
        ld fb = central(c, K, b) - tail(n, b);
        if ((fa < 0.0L) != (fb < 0.0L)) {
            for (int it = 0; it < 200; ++it) {
                ld m = 0.5L * (a + b), fm = central(c, K, m) - tail(n, m);
                if ((fm < 0.0L) == (fa < 0.0L)) { a = m; fa = fm; } else b = m;
                if (b - a <= 4.0L * LDBL_EPSILON * b) break;
            }
            return 0.5L * (a + b);
        }
        a = b; fa = fb;
    }
    return NAN;
}

double orc_student_crossover(double n, int K, const ld *c) { return (double)orc_student_crossover_ld(n, K, c); }

/* composite recycling map with coefficients c_0..c_K; zstar <= 0 selects the
 * continuity root orc_student_crossover(n, K, c) */
int orc_student_map(const double *z, ld *out, int64_t cnt, double n_, int K, const ld *c, double zstar)
{
    if (!(n_ > 0.0) || K < 0) return -1;
    ld n = (ld)n_;
    ld zs = (zstar > 0.0) ? (ld)zstar : orc_student_crossover_ld(n_, K, c);
    for (int64_t i = 0; i < cnt; ++i) {
        ld zi = (ld)z[i], a = fabsl(zi), t;
        if (isnan(zi)) t = NAN;
        else if (isinf(zi)) t = INFINITY;
        else if (a < zs) t = central(c, K, a);
        else t = tail(n, a);
        out[i] = signbit(zi) ? -t : t;
    }
    return 0;
}

/* the two branches separately (for the crossover / bound pins) */
int orc_student_branches(const double *z, ld *cen, ld *tl, int64_t cnt, double n_, int K, const ld *c)
{
    for (int64_t i = 0; i < cnt; ++i) {
        ld a = fabsl((ld)z[i]);
        cen[i] = central(c, K, a);
        tl[i] = (a > 0.0L) ? tail((ld)n_, a) : NAN;
    }
    return 0;
}

/* ---------------- exact map via the incomplete beta function ---------------- */

/* continued fraction of A&S 26.5.8 for I_x(a,b), evaluated by the modified
 * Lentz method; valid (fast) for x < (a+1)/(a+b+2). */
static ld beta_cf(ld a, ld b, ld x)
{
    const ld tiny = 1e-4000L;
    ld c = 1.0L, d = 1.0L - (a + b) * x / (a + 1.0L);
    if (fabsl(d) < tiny) d = tiny;
    d = 1.0L / d;
    ld h = d;
    for (int m = 1; m <= 100000; ++m) {
        ld mm = (ld)m;
        ld num = mm * (b - mm) * x / ((a + 2.0L * mm - 1.0L) * (a + 2.0L * mm));   /* d_{2m} */
        d = 1.0L + num * d; if (fabsl(d) < tiny) d = tiny;
        c = 1.0L + num / c; if (fabsl(c) < tiny) c = tiny;
        d = 1.0L / d; h *= d * c;
        num = -(a + mm) * (a + b + mm) * x / ((a + 2.0L * mm) * (a + 2.0L * mm + 1.0L));   /* d_{2m+1} */
        d = 1.0L + num * d; if (fabsl(d) < tiny) d = tiny;
        c = 1.0L + num / c; if (fabsl(c) < tiny) c = tiny;
        d = 1.0L / d;
        ld del = d * c;
        h *= del;
        if (fabsl(del - 1.0L) <= LDBL_EPSILON) break;
    }
    return h;
}

/* I_x(a,b) with x and xc = 1 - x supplied separately (both accurate) */
static ld betainc_reg(ld a, ld b, ld x, ld xc)
{
    if (x <= 0.0L) return 0.0L;
    if (xc <= 0.0L) return 1.0L;
    ld lbeta = lgammal(a) + lgammal(b) - lgammal(a + b);
    if (x < (a + 1.0L) / (a + b + 2.0L)) {
        ld front = expl(a * logl(x) + b * logl(xc) - lbeta);
        return front * beta_cf(a, b, x) / a;
    }
    ld front = expl(b * logl(xc) + a * logl(x) - lbeta);
    return 1.0L - front * beta_cf(b, a, xc) / b;
}

ld orc_student_cdf_upper(ld n, ld t)        /* P(T > t), t >= 0 */
{
    ld d = n + t * t;
    return 0.5L * betainc_reg(n / 2.0L, 0.5L, n / d, t * t / d);
}

static ld student_pdf(ld n, ld t)
{
    ld lc = lgammal((n + 1.0L) / 2.0L) - lgammal(n / 2.0L) - 0.5L * logl(n * PI_L);
    return expl(lc - 0.5L * (n + 1.0L) * log1pl(t * t / n));
}

/* exact A(|z|) >= 0 */
static ld student_exact_pos(ld n, ld a)
{
    if (a == 0.0L) return 0.0L;
    int centre = (erfl(a * SQRT1_2L) <= 0.5L);
    ld target = centre ? erfl(a * SQRT1_2L) : erfcl(a * SQRT1_2L);
    /* g(t) increasing in t */
#define G(tt) (centre ? (betainc_reg(0.5L, n / 2.0L, (tt) * (tt) / (n + (tt) * (tt)), n / (n + (tt) * (tt))) - target) \
                      : (target - betainc_reg(n / 2.0L, 0.5L, n / (n + (tt) * (tt)), (tt) * (tt) / (n + (tt) * (tt)))))
    ld lo = 0.0L, hi = 1.0L;
    while (G(hi) < 0.0L && hi < 1e4000L) { lo = hi; hi *= 2.0L; }
    ld t = (lo > 0.0L) ? sqrtl(lo * hi) : 0.5L * hi;
    for (int it = 0; it < 2000; ++it) {
        ld g = G(t);
        if (g == 0.0L) return t;
        if (g > 0.0L) hi = t; else lo = t;
        ld tn = t - g / (2.0L * student_pdf(n, t));    /* dG/dt = 2 f(t) in both forms */
        if (!(tn > lo && tn < hi)) tn = (lo > 0.0L && hi / lo > 4.0L) ? sqrtl(lo * hi) : 0.5L * (lo + hi);
        if (fabsl(tn - t) <= 2.0L * LDBL_EPSILON * t || hi - lo <= 2.0L * LDBL_EPSILON * hi) return tn;
        t = tn;
    }
#undef G
    return t;
}

int orc_student_exact(const double *z, ld *out, int64_t cnt, double n_)
{
    if (!(n_ > 0.0)) return -1;
    for (int64_t i = 0; i < cnt; ++i) {
        ld zi = (ld)z[i], t;
        if (isnan(zi)) t = NAN;
        else if (isinf(zi)) t = INFINITY;
        else t = student_exact_pos((ld)n_, fabsl(zi));
        out[i] = signbit(zi) ? -t : t;
    }
    return 0;
}

void orc_student_cdf_upper_v(const ld *t, ld *out, int64_t cnt, double n)
{
    for (int64_t i = 0; i < cnt; ++i) out[i] = orc_student_cdf_upper((ld)n, t[i]);
}

/* tail constant C_n = n sqrt(pi) Gamma(n/2)/Gamma((n+1)/2) */
void orc_student_tail_const(double n, ld *out)
{
    *out = (ld)n * sqrtl(PI_L) * gamma_ratio_half((ld)n);
}

/* ---------------- purely numerical method (§3.6) ----------------
 * "The direct numerical solution of the RODE can be done using standard
 * methods ... explicit Runge-Kutta ... a precision of better than 5e-8 on the
 * range |z| < 6."  The Student Recycling ODE
 *     (1 + Q^2/n)(Q'' + v Q') = (1 + 1/n) Q (Q')^2
 * with the centre conditions Q(0) = 0, Q'(0) = gamma, written as the
 * first-order system (Q, P = Q'):  Q' = P,  P' = (1 + 1/n) Q P^2 / (1 + Q^2/n) - v P,
 * integrated FORWARD from v = 0 to |z| by the classical explicit Runge-Kutta
 * method of order 4 in ceil(|z|/h) equal steps; odd symmetry for z < 0.
 * Forward is the paper's direction; its error grows like e^{v^2/2} (the
 * neighbouring solutions Q^-n = A + B erfc(v/sqrt2) of the tail equation
 * saturate), so this is an oracle for |z| up to ~8, not for the far tail. */
static void student_rode_rhs(ld n, ld v, ld q, ld p, ld *dq, ld *dp)
{
    *dq = p;
    *dp = (1.0L + 1.0L / n) * q * p * p / (1.0L + q * q / n) - v * p;
}

int orc_student_rode(const double *z, ld *out, int64_t cnt, double n_, double h)
{
    if (!(n_ > 0.0) || !(h > 0.0)) return -1;
    const ld n = (ld)n_;
    for (int64_t i = 0; i < cnt; ++i) {
        const ld zi = (ld)z[i], a = fabsl(zi);
        if (isnan(zi)) { out[i] = NAN; continue; }
        if (isinf(zi)) { out[i] = zi; continue; }
        const int64_t N = (int64_t)ceill(a / (ld)h);
        const ld s = (N > 0) ? a / (ld)N : 0.0L;
        ld q = 0.0L, p = orc_student_gamma_ld(n_), v = 0.0L;
        for (int64_t k = 0; k < N; ++k) {
            ld k1q, k1p, k2q, k2p, k3q, k3p, k4q, k4p;
            student_rode_rhs(n, v, q, p, &k1q, &k1p);
            student_rode_rhs(n, v + 0.5L * s, q + 0.5L * s * k1q, p + 0.5L * s * k1p, &k2q, &k2p);
            student_rode_rhs(n, v + 0.5L * s, q + 0.5L * s * k2q, p + 0.5L * s * k2p, &k3q, &k3p);
            student_rode_rhs(n, v + s, q + s * k3q, p + s * k3p, &k4q, &k4p);
            q += s / 6.0L * (k1q + 2.0L * k2q + 2.0L * k3q + k4q);
            p += s / 6.0L * (k1p + 2.0L * k2p + 2.0L * k3p + k4p);
            v = (ld)(k + 1) * s;
        }
        out[i] = signbit(zi) ? -q : q;
    }
    return 0;
}
