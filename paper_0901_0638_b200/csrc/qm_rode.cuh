// qm_rode.cuh -- exponential-base recycling into hyperbolic / variance-gamma
// samples (§4 of the paper).
//
// The map Q(v) is the numerically solved Recycling ODE (built on the host by
// qm_rode_host.cpp into a table of (Q, Q', Q'') at the nodes of a centre, a fine
// (out to base probability e^-40) and a coarse segment (out to e^-800), per
// side; see qm_rode_params.h).  Per sample the kernel does a quintic Hermite interpolation
// between two nodes (four 16-byte gathers from the table, which stays in L2/L1;
// the error is O(h^6), needed for relative accuracy near v = 0).  Past e^-800
// (no double uniform reaches it) linear extrapolation with the end slope
// (Q' -> 1 in the tails).  Side and segment are selects, not branches.
// The fused sampler draws u from Philox and applies the base quantile Q0 of
// P:322-329 first.
#pragma once
#include "qm_dd.cuh"
#include "qm_rode_params.h"

namespace qm {

QM_DEV double rode_eval(const double *__restrict__ tab, double v)
{
    const int side = (v < 0.0) ? 1 : 0;
    const double a = fabs(v);
    const double *sg = tab + QM_RODE_SEG + 24 * side;          // 3 segment records of 8 doubles
    const double Vmax = __ldg(tab + 28 + side);
    const double2 *nd = reinterpret_cast<const double2 *>(tab + QM_RODE_HEADER + side * 4 * (QM_RODE_NT + 1));
    // segment j = [a >= Wc] + [a >= V] (selects; NaN lands in j = 0 and is replaced later)
    const int j = (a >= __ldg(sg + 8)) + (a >= __ldg(sg + 16));
    const double2 r01 = __ldg(reinterpret_cast<const double2 *>(sg + 8 * j));       // w0, h
    const double2 r23 = __ldg(reinterpret_cast<const double2 *>(sg + 8 * j + 2));   // 1/h, k0
    const double2 r45 = __ldg(reinterpret_cast<const double2 *>(sg + 8 * j + 4));   // n, w1
    const double h = r01.y;
    const double s = fmin((a - r01.x) * r23.x, r45.x);        // local coordinate in [0, n]
    const double fk = fmin(floor(s), r45.x - 1.0);
    const int k = (int)r23.y + (int)fk;
    const double t = s - fk;
    // node k: (R, R') at nd[2k], (R'', 0) at nd[2k+1]
    const double2 n0 = __ldg(nd + 2 * k), c0 = __ldg(nd + 2 * k + 1);
    const double2 n1 = __ldg(nd + 2 * k + 2), c1 = __ldg(nd + 2 * k + 3);
    // quintic Hermite in monomial form: R(k h + t h) = p0 + m0 t + a0/2 t^2 + c3 t^3 + c4 t^4 + c5 t^5
    const double m0 = h * n0.y, m1 = h * n1.y, h2 = h * h;
    const double a0 = h2 * c0.x, a1 = h2 * c1.x, dp = n1.x - n0.x;
    const double c3 = 10.0 * dp - 6.0 * m0 - 4.0 * m1 - 1.5 * a0 + 0.5 * a1;
    const double c4 = -15.0 * dp + 8.0 * m0 + 7.0 * m1 + 1.5 * a0 - a1;
    const double c5 = 6.0 * dp - 3.0 * m0 - 3.0 * m1 - 0.5 * a0 + 0.5 * a1;
    const double q = n0.x + t * (m0 + t * (0.5 * a0 + t * (c3 + t * (c4 + t * c5))));
    const double qx = n1.x + (a - Vmax) * n1.y;              // beyond Vmax: n1 = node NT
    return (a <= Vmax) ? q : qx;
}

// x = Q(v) with IEEE semantics: +-0 -> +-0, +-inf -> +-inf, NaN -> NaN
QM_DEV double rode_map(const double *__restrict__ tab, double v)
{
    const double q = rode_eval(tab, v);
    const double r = (v == 0.0) ? v : q;
    return (fabs(v) < __longlong_as_double(0x7ff0000000000000LL)) ? r : v;
}

template <typename T>
__global__ void __launch_bounds__(256)
k_rode_map(const T *__restrict__ v, T *__restrict__ x, int64_t n, const double *__restrict__ tab)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        x[i] = (T)rode_map(tab, (double)v[i]);
}

// base quantile Q0: u < p- -> log(u/p-)/(a+b); u > p- -> -log((1-u)/p+)/(a-b).
// |v| = (-log t + log p_s)/rate_s with t = u (left) or 1-u (right), exact on the odd grid.
QM_DEV double exp_base_quantile(const double *__restrict__ tab, double u)
{
    const int side = (u < __ldg(tab + 9)) ? 1 : 0;             // tab[9] = p-
    const double t = side ? u : __dadd_rn(1.0, -u);
    const dd L = neg_log_dd(t);                                 // -log t
    const dd m = dd_add(L, dd{__ldg(tab + 16 + side), __ldg(tab + 18 + side)});
    const double av = (m.hi + m.lo) * __ldg(tab + 20 + side);
    return side ? -av : av;
}

template <typename T>
__global__ void __launch_bounds__(256)
k_exp_base_quantile(const T *__restrict__ u, T *__restrict__ v, int64_t n, const double *__restrict__ tab)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double ui = (double)u[i];
        const double r = exp_base_quantile(tab, ui);
        v[i] = (T)((ui > 0.0 && ui < 1.0) ? r : (ui == 0.0 ? -__longlong_as_double(0x7ff0000000000000LL)
                                                  : (ui == 1.0 ? __longlong_as_double(0x7ff0000000000000LL)
                                                               : __longlong_as_double(0x7fffffffffffffffLL))));
    }
}

// fused: Philox uniforms (qm_philox_uniform layout) -> Q0 -> Q
template <typename T>
__global__ void __launch_bounds__(256)
k_rode_philox(T *__restrict__ x, int64_t n, unsigned long long seed, unsigned long long c0,
              const double *__restrict__ tab)
{
    constexpr int W = (sizeof(T) == 4) ? 4 : 2;                 // samples per Philox block
    const int64_t nb = (n + W - 1) / W;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += stride) {
        const uint4 w = philox_block(c0 + (unsigned long long)b, seed);
        double u[4];
        if (W == 4) { u[0] = u01_f32(w.x); u[1] = u01_f32(w.y); u[2] = u01_f32(w.z); u[3] = u01_f32(w.w); }
        else { u[0] = u01_f64(w.x, w.y); u[1] = u01_f64(w.z, w.w); }
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const int64_t i = b * W + k;
            if (i < n) x[i] = (T)rode_eval(tab, exp_base_quantile(tab, u[k]));
        }
    }
}

}  // namespace qm
