// qm_rode.cuh -- exponential-base recycling into hyperbolic / variance-gamma
// samples (§4 of the paper).
//
// The map Q(v) is the numerically solved Recycling ODE (built on the host by
// qm_rode_host.cpp into a table of (Q, Q') at equally spaced |v| nodes per
// side).  Per sample the kernel does a cubic Hermite interpolation between two
// nodes (two 16-byte gathers from the table, which stays in L2/L1) and, past
// |v| = V (base probability e^-40), linear extrapolation with the end slope
// (Q' -> 1 in the tails).  The side is a select, not a branch.
// The fused sampler draws u from Philox and applies the base quantile Q0 of
// P:322-329 first.
#pragma once
#include "qm_dd.cuh"
#include "qm_rode_params.h"

namespace qm {

QM_DEV double rode_eval(const double *__restrict__ tab, double v)
{
    const int side = (v < 0.0) ? 1 : 0;
    const int N = QM_RODE_NODES;
    const double a = fabs(v);
    const double h = __ldg(tab + 2 + side), ih = __ldg(tab + 4 + side), V = __ldg(tab + 6 + side);
    const double2 *nd = reinterpret_cast<const double2 *>(tab + QM_RODE_HEADER + side * 2 * (N + 1));
    const double s = fmin(a * ih, (double)N);
    int k = (int)s;
    k = (k > N - 1) ? N - 1 : k;
    const double t = s - (double)k;
    const double2 n0 = __ldg(nd + k), n1 = __ldg(nd + k + 1);
    const double t2 = t * t, t3 = t2 * t;
    const double h00 = 2.0 * t3 - 3.0 * t2 + 1.0, h10 = t3 - 2.0 * t2 + t;
    const double h01 = -2.0 * t3 + 3.0 * t2, h11 = t3 - t2;
    const double q = h00 * n0.x + h * (h10 * n0.y + h11 * n1.y) + h01 * n1.x;
    const double qx = n1.x + (a - V) * n1.y;                 // beyond V: k = N-1, n1 = node N
    return (a <= V) ? q : qx;
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
