// qm_dd.cuh -- double-double helpers for the fp64 paths that must stay within
// 2 ulp of the exactly evaluated formula (baselines, Student tail).
#pragma once
#include "qm_math.cuh"

namespace qm {

QM_DEV dd dd_from(double a) { return dd{a, 0.0}; }

QM_DEV dd two_sum(double a, double b)
{
    const double s = __dadd_rn(a, b);
    const double bb = __dadd_rn(s, -a);
    return dd{s, __dadd_rn(__dadd_rn(a, -__dadd_rn(s, -bb)), __dadd_rn(b, -bb))};
}

QM_DEV dd dd_norm(double hi, double lo)
{
    const double s = __dadd_rn(hi, lo);
    return dd{s, __dadd_rn(lo, -__dadd_rn(s, -hi))};
}

QM_DEV dd dd_add(dd a, dd b)
{
    const dd s = two_sum(a.hi, b.hi);
    return dd_norm(s.hi, __dadd_rn(s.lo, __dadd_rn(a.lo, b.lo)));
}

QM_DEV dd dd_add_d(dd a, double b)
{
    const dd s = two_sum(a.hi, b);
    return dd_norm(s.hi, __dadd_rn(s.lo, a.lo));
}

QM_DEV dd dd_mul(dd a, dd b)
{
    const double p = __dmul_rn(a.hi, b.hi);
    const double e = __fma_rn(a.hi, b.hi, -p);
    return dd_norm(p, __fma_rn(a.hi, b.lo, __fma_rn(a.lo, b.hi, e)));
}

QM_DEV dd dd_mul_d(dd a, double b)
{
    const double p = __dmul_rn(a.hi, b);
    const double e = __fma_rn(a.hi, b, -p);
    return dd_norm(p, __fma_rn(a.lo, b, e));
}

QM_DEV double rcp_refined(double b)
{
    double r = rcp_approx_f64(b);
    r = __fma_rn(r, __fma_rn(-b, r, 1.0), r);
    return __fma_rn(r, __fma_rn(-b, r, 1.0), r);     // ~2^-88 relative for |b| in normal range
}

// a / b as a double-double (|b| normal, nonzero)
QM_DEV dd dd_div(dd a, dd b)
{
    const double r = rcp_refined(b.hi);
    const double q0 = __dmul_rn(a.hi, r);
    double e = __fma_rn(-b.hi, q0, a.hi);
    e = __fma_rn(-q0, b.lo, __dadd_rn(e, a.lo));
    return dd_norm(q0, __dmul_rn(e, r));
}

// sqrt of a double-double a > 0
QM_DEV dd dd_sqrt(dd a)
{
    const double s = sqrt(a.hi);                       // correctly rounded
    const double e = __fma_rn(-s, s, a.hi);            // exact remainder
    const double c = __dmul_rn(__dadd_rn(e, a.lo), __dmul_rn(0.5, rcp_refined(s)));
    return dd_norm(s, c);
}

// exp of a double-double: k = round(x/ln2), r = x - k ln2 (dd),
// exp(r) = 1 + r + r^2/2 + ... (Taylor to r^17, |r| <= 0.347) in dd for the
// first terms; one final 2^k scaling.  The argument is first clamped to
// [-746, 710]: beyond, exp overflows to +inf / underflows to +0 through the
// scaling (|k| <= 1077 keeps both exponent halves in range).
QM_DEV dd dd_exp(dd x)
{
    if (x.hi > 710.0) x = dd{710.0, 0.0};           // +inf after scaling
    if (x.hi < -746.0) x = dd{-746.0, 0.0};         // +0 after scaling
    const double k = rint(__dmul_rn(x.hi, 1.4426950408889634));
    // ln2 as a triple for an exact-enough reduction
    const double L1 = 6.93147180369123816490e-01, L2 = 1.90821492927058770002e-10, L3 = 1.1612227229362531851e-26;
    dd r = dd_add_d(x, -k * L1);                       // k*L1 exact (|k| < 2^11)
    r = dd_add_d(r, -k * L2);
    r = dd_add_d(r, -k * L3);
    // Taylor with Horner in dd for the leading terms, double for the tail
    double t = 1.0 / 355687428096000.0;                // 1/17!
    const double inv_fact[17] = {1.0, 1.0, 0.5, 1.0 / 6, 1.0 / 24, 1.0 / 120, 1.0 / 720, 1.0 / 5040,
                                 1.0 / 40320, 1.0 / 362880, 1.0 / 3628800, 1.0 / 39916800,
                                 1.0 / 479001600, 1.0 / 6227020800.0, 1.0 / 87178291200.0,
                                 1.0 / 1307674368000.0, 1.0 / 20922789888000.0};
#pragma unroll
    for (int i = 16; i >= 6; --i) t = __fma_rn(t, r.hi, inv_fact[i]);
    dd s = dd{t, 0.0};
#pragma unroll
    for (int i = 5; i >= 0; --i) {
        s = dd_mul(s, r);
        // exact-enough 1/i! as dd for i <= 5 (1/3!, 1/5! are not exact)
        const dd c = (i == 3) ? dd{1.0 / 6, 9.25185853854297e-18} : (i == 5) ? dd{1.0 / 120, 1.1564823173178713963e-19} : (i == 4) ? dd{1.0 / 24, 2.3129646346357427925e-18} : dd{inv_fact[i], 0.0};
        s = dd_add(s, c);
    }
    // 2^k as two exact powers of two built from exponent bits (no branches;
    // |k| <= 2044 keeps both halves in the normal range)
    const int ki = (int)k, k1 = ki / 2, k2 = ki - k1;
    const double sc1 = __longlong_as_double((long long)(k1 + 1023) << 52);
    const double sc2 = __longlong_as_double((long long)(k2 + 1023) << 52);
    return dd{s.hi * sc1 * sc2, s.lo * sc1 * sc2};
}

// -log(x) as dd for any positive finite x (subnormals pre-scaled by 2^54)
QM_DEV dd neg_log_dd(double x)
{
    const bool sub = x < 2.2250738585072014e-308;
    return neg_log2x_dd(sub ? __dmul_rn(x, 18014398509481984.0) : x, sub ? -55 : -1);
}

// natural log of a positive finite double as dd
QM_DEV dd dd_log(double x)
{
    const dd m = neg_log_dd(x);
    return dd{-m.hi, -m.lo};
}

// §5.1 supplementary tail model (reading R1): Q(v) = sqrt(2 q(a,b)),
// a = v - 1/2 log pi, b = log a,
// q = a - b/2 + (b/4 - 1/2)/a + (b^2 - 6b + 14)/(16 a^2) + (2b^3 - 21b^2 + 102b - 214)/(96 a^3)
//       + (3b^4 - 46b^3 + 348b^2 - 1488b + 2978)/(384 a^4).
// a - b/2 in double-double, the small corrections in double, dd sqrt.
QM_DEV double tail_model_q_dd(dd v)
{
    const double C_HI = 0.5723649429247001, C_LO = 5.1329755813539131214e-18;   // log(pi)/2
    dd a = two_sum(v.hi, -C_HI);
    a = dd_norm(a.hi, __dadd_rn(a.lo, __dadd_rn(v.lo, -C_LO)));
    dd b = dd_log(a.hi);
    b = dd_add_d(b, a.lo / a.hi);                                   // log(a_hi + a_lo)
    const double bh = b.hi, ia = 1.0 / a.hi;
    const double t1 = (0.25 * bh - 0.5) * ia;
    const double t2 = ((bh - 6.0) * bh + 14.0) * (1.0 / 16.0) * ia * ia;
    const double t3 = (((2.0 * bh - 21.0) * bh + 102.0) * bh - 214.0) * (1.0 / 96.0) * ia * ia * ia;
    const double t4 = ((((3.0 * bh - 46.0) * bh + 348.0) * bh - 1488.0) * bh + 2978.0) * (1.0 / 384.0) * ia * ia * ia * ia;
    dd q = dd_add(a, dd{-0.5 * b.hi, -0.5 * b.lo});
    q = dd_add_d(q, t1 + t2 + t3 + t4);
    const dd s = dd_sqrt(dd{2.0 * q.hi, 2.0 * q.lo});
    return s.hi + s.lo;
}

QM_DEV double tail_model_q(double v) { return tail_model_q_dd(dd{v, 0.0}); }

// Compensated Horner for arbitrary-sign coefficients at a dd point, fully compensated.
template <int N>
QM_DEV dd horner_dd(const double *a, dd z)
{
    return horner_comp<N, N - 1>(a, z.hi, z.lo);
}

// a / b rounded once to double
QM_DEV double dd_div_round(dd a, dd b)
{
    const double r = rcp_refined(b.hi);
    const double q0 = __dmul_rn(a.hi, r);
    double e = __fma_rn(-b.hi, q0, a.hi);
    e = __fma_rn(-q0, b.lo, __dadd_rn(e, a.lo));
    return __fma_rn(e, r, q0);
}

}  // namespace qm
