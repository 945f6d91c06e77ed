// qm_baselines.cuh -- the branching comparison quantiles of the paper's
// Table 3: AS241 (Wichura 1988; "two breaks, at u=0.925 and
// u=1-e^-25"), Acklam level 1 ("breaks at u=0.97575") and the
// refined Acklam (one Halley step).  Coefficients are not in the paper
// (P:601-616 point to external code); they are transcribed from the original
// publications (reading R17).  These kernels branch per element ON
// PURPOSE: they are the divergence foil of the breakless kernels, and their
// branch efficiency is what ncu reports for them.
//
// Arithmetic: region decisions in double (as the oracle takes them); each
// region's formula in double-double (compensated Horner, dd log/sqrt, dd
// quotient) with one final rounding, so that the result stays within 2 ulp of
// the exactly evaluated formula -- the refined step is plain double, as in the
// published code.
#pragma once
#include "qm_dd.cuh"

namespace qm {

enum { ALG_AS241 = 2, ALG_ACKLAM = 3, ALG_ACKLAM_REF = 4, ALG_MORO = 6 };

// AS241 PPND16 in ascending powers
__constant__ double kAS_A[8] = {3.3871328727963666080e0, 1.3314166789178437745e+2, 1.9715909503065514427e+3,
                                1.3731693765509461125e+4, 4.5921953931549871457e+4, 6.7265770927008700853e+4,
                                3.3430575583588128105e+4, 2.5090809287301226727e+3};
__constant__ double kAS_B[8] = {1.0, 4.2313330701600911252e+1, 6.8718700749205790830e+2, 5.3941960214247511077e+3,
                                2.1213794301586595867e+4, 3.9307895800092710610e+4, 2.8729085735721942674e+4,
                                5.2264952788528545610e+3};
__constant__ double kAS_C[8] = {1.42343711074968357734e0, 4.63033784615654529590e0, 5.76949722146069140550e0,
                                3.64784832476320460504e0, 1.27045825245236838258e0, 2.41780725177450611770e-1,
                                2.27238449892691845833e-2, 7.74545014278341407640e-4};
__constant__ double kAS_D[8] = {1.0, 2.05319162663775882187e0, 1.67638483018380384940e0, 6.89767334985100004550e-1,
                                1.48103976427480074590e-1, 1.51986665636164571966e-2, 5.47593808499534494600e-4,
                                1.05075007164441684324e-9};
__constant__ double kAS_E[8] = {6.65790464350110377720e0, 5.46378491116411436990e0, 1.78482653991729133580e0,
                                2.96560571828504891230e-1, 2.65321895265761230930e-2, 1.24266094738807843860e-3,
                                2.71155556874348757815e-5, 2.01033439929228813265e-7};
__constant__ double kAS_F[8] = {1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1, 1.48753612908506148525e-2,
                                7.86869131145613259100e-4, 1.84631831751005468180e-5, 1.42151175831644588870e-7,
                                2.04426310338993978564e-15};

// Acklam level 1, ascending powers: central num a6 + a5 r + ... + a1 r^5 (times q),
// central den 1 + b5 r + ... + b1 r^5, tail num c6 + c5 q + ... + c1 q^5,
// tail den 1 + d4 q + d3 q^2 + d2 q^3 + d1 q^4.
__constant__ double kAK_A[6] = {2.506628277459239e+00, -3.066479806614716e+01, 1.383577518672690e+02,
                                -2.759285104469687e+02, 2.209460984245205e+02, -3.969683028665376e+01};
__constant__ double kAK_B[6] = {1.0, -1.328068155288572e+01, 6.680131188771972e+01, -1.556989798598866e+02,
                                1.615858368580409e+02, -5.447609879822406e+01};
__constant__ double kAK_C[6] = {2.938163982698783e+00, 4.374664141464968e+00, -2.549732539343734e+00,
                                -2.400758277161838e+00, -3.223964580411365e-01, -7.784894002430293e-03};
__constant__ double kAK_D[5] = {1.0, 3.754408661907416e+00, 2.445134137142996e+00, 3.224671290700398e-01,
                                7.784695709041462e-03};

QM_DEV double nan_d() { return __longlong_as_double(0x7fffffffffffffffLL); }
QM_DEV double inf_d() { return __longlong_as_double(0x7ff0000000000000LL); }

QM_DEV double as241(double u)
{
    if (!(u >= 0.0 && u <= 1.0)) return nan_d();
    if (u == 0.0) return -inf_d();
    if (u == 1.0) return inf_d();
    const double qd = __dadd_rn(u, -0.5);
    if (fabs(qd) <= 0.425) {
        const dd q = two_sum(u, -0.5);                             // exact q
        const dd r = dd_add_d(dd{-dd_mul(q, q).hi, -dd_mul(q, q).lo}, 0.180625);
        const dd num = dd_mul(q, horner_dd<8>(kAS_A, r));
        return dd_div_round(num, horner_dd<8>(kAS_B, r));
    }
    const double t = (qd < 0.0) ? u : __dadd_rn(1.0, -u);         // exact
    const dd R = dd_sqrt(neg_log_dd(t));                           // sqrt(-log t)
    double x;
    if (R.hi <= 5.0) {
        const dd r = dd_add_d(R, -1.6);
        x = dd_div_round(horner_dd<8>(kAS_C, r), horner_dd<8>(kAS_D, r));
    } else {
        const dd r = dd_add_d(R, -5.0);
        x = dd_div_round(horner_dd<8>(kAS_E, r), horner_dd<8>(kAS_F, r));
    }
    return (qd < 0.0) ? -x : x;
}

// Acklam level 1 on the lower half t = min(p, 1-p) (reading R19), x <= 0
QM_DEV double acklam_lower(double t)
{
    if (t < 0.02425) {
        const dd L = neg_log_dd(t);                                 // -log t
        const dd q = dd_sqrt(dd{2.0 * L.hi, 2.0 * L.lo});
        return dd_div_round(horner_dd<6>(kAK_C, q), horner_dd<5>(kAK_D, q));
    }
    const dd q = two_sum(t, -0.5);
    const dd r = dd_mul(q, q);
    return dd_div_round(dd_mul(q, horner_dd<6>(kAK_A, r)), horner_dd<6>(kAK_B, r));
}

template <bool REFINE>
QM_DEV double acklam(double p)
{
    if (!(p >= 0.0 && p <= 1.0)) return nan_d();
    if (p == 0.0) return -inf_d();
    if (p == 1.0) return inf_d();
    const double t = (p < 0.5) ? p : __dadd_rn(1.0, -p);
    double x = acklam_lower(t);
    if (REFINE && t >= 2.2250738585072014e-308) {   // R20: exp(x^2/2) overflows for subnormal t; keep level 1
        // Halley step of the published refinement (plain double, as published)
        const double e = 0.5 * erfc(-x * 0.70710678118654752440) - t;
        const double uu = e * 2.50662827463100050242 * exp(0.5 * x * x);
        x = x - uu / (1.0 + 0.5 * x * uu);
    }
    return (p < 0.5) ? x : 0.0 - x;
}

// Moro (1995): Beasley-Springer central rational y A(y^2)/B(y^2) for
// |y| = |u - 1/2| < 0.42 ("Moro: breaks at u = 0.92"), Moro's series in
// s = log(-log r), r = min(u, 1-u), beyond ("a log(log()) operation is carried
// out in the tail region").  Coefficients external (R17), ascending.
__constant__ double kMO_A[4] = {2.50662823884, -18.61500062529, 41.39119773534, -25.44106049637};
__constant__ double kMO_B[5] = {1.0, -8.47351093090, 23.08336743743, -21.06224101826, 3.13082909833};
__constant__ double kMO_C[9] = {0.3374754822726147, 0.9761690190917186, 0.1607979714918209,
                                0.0276438810333863, 0.0038405729373609, 0.0003951896511919,
                                0.0000321767881768, 0.0000002888167364, 0.0000003960315187};

QM_DEV double moro(double u)
{
    if (!(u >= 0.0 && u <= 1.0)) return nan_d();
    if (u == 0.0) return -inf_d();
    if (u == 1.0) return inf_d();
    const double yd = __dadd_rn(u, -0.5);
    if (fabs(yd) < 0.42) {
        const dd y = two_sum(u, -0.5);                              // exact y
        const dd r = dd_mul(y, y);
        return dd_div_round(dd_mul(y, horner_dd<4>(kMO_A, r)), horner_dd<5>(kMO_B, r));
    }
    const double t = (yd < 0.0) ? u : __dadd_rn(1.0, -u);          // exact
    const dd L = neg_log_dd(t);                                     // -log t > 0
    const dd sl = dd_add_d(dd_log(L.hi), L.lo / L.hi);              // log(L_hi + L_lo)
    const dd x = horner_dd<9>(kMO_C, sl);
    const double xr = __dadd_rn(x.hi, x.lo);
    return (yd < 0.0) ? -xr : xr;
}

// ------------------------------------------------------------------------
// Plain-double versions (config 1 like-for-like with the paper's Table 3, whose
// codes are all plain double: "Acklam single coded as double", Lea's refined
// Acklam, App D, AS241 -- P:634-662): the same formulas and region breaks,
// every operation one IEEE double operation (FMA Horner, CUDA log/sqrt/erfc/exp,
// IEEE division), no compensation.  Their accuracy is that of plain double
// evaluation (bounded by ~(2 N + 3) ulp for N-term polynomials; measured by the
// tests), not the 2-ulp contract of the kernels above.
template <int N>
QM_DEV double horner_plain(const double *a, double x)
{
    double s = a[N - 1];
#pragma unroll
    for (int i = N - 2; i >= 0; --i) s = __fma_rn(s, x, a[i]);
    return s;
}

QM_DEV double specials_or(double u, double x)
{
    x = (u == 0.0) ? -inf_d() : x;
    x = (u == 1.0) ? inf_d() : x;
    return (u >= 0.0 && u <= 1.0) ? x : nan_d();
}

// App D and the (7,7) of App A, as printed: vv, z = -log(2 vv), z P(z)/Q(z), sign
template <int ALG>
QM_DEV double breakless_plain(double u)
{
    const double omu = 1.0 - u;
    const double vv = fmin(u, omu);
    const double z = -log(2.0 * vv);
    const double r = (ALG == ALG_BREAKLESS77) ? z * horner_plain<8>(kA77P_d, z) / horner_plain<8>(kA77Q_d, z)
                                              : z * horner_plain<14>(kD13P, z) / horner_plain<14>(kD13Q, z);
    return specials_or(u, (u < 0.5) ? -fabs(r) : fabs(r));   // sgn = +1 at u = 1/2 (z = -0 there)
}

QM_DEV double as241_plain(double u)
{
    const double q = u - 0.5;
    double x;
    if (fabs(q) <= 0.425) {
        const double r = 0.180625 - q * q;
        x = q * horner_plain<8>(kAS_A, r) / horner_plain<8>(kAS_B, r);
    } else {
        const double t = (q < 0.0) ? u : 1.0 - u;
        double r = sqrt(-log(t));
        if (r <= 5.0) {
            r -= 1.6;
            x = horner_plain<8>(kAS_C, r) / horner_plain<8>(kAS_D, r);
        } else {
            r -= 5.0;
            x = horner_plain<8>(kAS_E, r) / horner_plain<8>(kAS_F, r);
        }
        x = (q < 0.0) ? -x : x;
    }
    return specials_or(u, x);
}

template <bool REFINE>
QM_DEV double acklam_plain(double p)
{
    const double t = (p < 0.5) ? p : 1.0 - p;
    double x;
    if (t < 0.02425) {
        const double q = sqrt(-2.0 * log(t));
        x = horner_plain<6>(kAK_C, q) / horner_plain<5>(kAK_D, q);
    } else {
        const double q = t - 0.5, r = q * q;
        x = q * horner_plain<6>(kAK_A, r) / horner_plain<6>(kAK_B, r);
    }
    if (REFINE && t >= 2.2250738585072014e-308) {
        const double e = 0.5 * erfc(-x * 0.70710678118654752440) - t;
        const double uu = e * 2.50662827463100050242 * exp(0.5 * x * x);
        x = x - uu / (1.0 + 0.5 * x * uu);
    }
    return specials_or(p, (p < 0.5) ? x : -x);
}

QM_DEV double moro_plain(double u)
{
    const double y = u - 0.5;
    double x;
    if (fabs(y) < 0.42) {
        const double r = y * y;
        x = y * horner_plain<4>(kMO_A, r) / horner_plain<5>(kMO_B, r);
    } else {
        const double t = (y < 0.0) ? u : 1.0 - u;
        x = horner_plain<9>(kMO_C, log(-log(t)));
        x = (y < 0.0) ? -x : x;
    }
    return specials_or(u, x);
}

template <int ALG>
__global__ void __launch_bounds__(256)
k_plain_f64(const double *__restrict__ u, double *__restrict__ z, int64_t n)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double x = u[i];
        double r;
        if (ALG == ALG_BREAKLESS || ALG == ALG_BREAKLESS77) r = breakless_plain<ALG>(x);
        else if (ALG == ALG_AS241) r = as241_plain(x);
        else if (ALG == ALG_ACKLAM) r = acklam_plain<false>(x);
        else if (ALG == ALG_ACKLAM_REF) r = acklam_plain<true>(x);
        else r = moro_plain(x);
        z[i] = r;
    }
}

template <int ALG>
QM_DEV double branchy(double u)
{
    if (ALG == ALG_MORO) return moro(u);
    if (ALG == ALG_AS241) return as241(u);
    if (ALG == ALG_ACKLAM) return acklam<false>(u);
    return acklam<true>(u);
}

template <int ALG>
__global__ void __launch_bounds__(256)
k_branchy_f64(const double *__restrict__ u, double *__restrict__ z, int64_t n)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        z[i] = branchy<ALG>(u[i]);
}

}  // namespace qm
