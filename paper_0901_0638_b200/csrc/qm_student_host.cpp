// qm_student_host.cpp -- per-call host setup of the normal -> Student-t map:
// gamma, the coefficient recurrence of P:178-188 and the tail
// constants of P:270-272.  Runs once per (nu, K, zstar) in __float128 (113-bit)
// because the recurrence is ill-conditioned: each step cancels terms of size
// c_i down to c_{i+1}; 113 bits keep c_0..c_24 exact to double for nu <= 20
// (tests/test_gpu_student.py compares them with an independent 100-digit run).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <map>
#include <tuple>
extern "C" {
#include <quadmath.h>
}
#include "qm_student_params.h"

namespace qm {

static void split_dd(__float128 x, double *hi, double *lo)
{
    *hi = (double)x;
    *lo = (double)(x - (__float128)(*hi));
}

bool student_params(double nu_d, int K, double zstar, StudentParams *out)
{
    if (!(nu_d >= 1.0 && nu_d <= 20.0) || K < 1 || K > QM_STUDENT_KMAX || !(zstar > 0.0)) return false;
    static std::mutex mu;
    static std::map<std::tuple<double, int, double>, StudentParams> cache;
    std::lock_guard<std::mutex> g(mu);
    auto key = std::make_tuple(nu_d, K, zstar);
    auto it = cache.find(key);
    if (it != cache.end()) { *out = it->second; return true; }

    const __float128 n = nu_d;
    const __float128 lg_ratio = lgammaq(n / 2) - lgammaq((n + 1) / 2);     // log G(n/2)/G((n+1)/2)
    __float128 c[QM_STUDENT_KMAX + 1];
    c[0] = sqrtq(n / 2) * expq(lg_ratio);                                  // gamma
    for (int i = 0; i < K; ++i) {
        __float128 rhs = -(__float128)(2 * i + 1) * c[i];
        for (int l = 0; l <= i; ++l)
            for (int m = 0; m <= i - l; ++m) {
                const __float128 alm = (1 + 1 / n) * (__float128)(2 * l + 1) * (__float128)(2 * m + 1)
                                       - (2 / n) * (__float128)m * (__float128)(2 * m + 1);
                rhs += alm * c[i - l - m] * c[l] * c[m];
            }
        if (i >= 1) {
            __float128 s = 0;
            for (int l = 0; l <= i - 1; ++l)
                for (int m = 0; m <= i - 1 - l; ++m)
                    s += (__float128)(2 * m + 1) * c[i - 1 - l - m] * c[l] * c[m];
            rhs -= s / n;
        }
        c[i + 1] = rhs / ((__float128)(2 * i + 3) * (__float128)(2 * i + 2));
    }
    StudentParams sp;
    std::memset(&sp, 0, sizeof(sp));
    for (int k = 0; k <= K; ++k) sp.c[k] = (double)c[k];
    sp.K = K;
    // Compensating the last 2 Horner steps already gives the fully compensated
    // result (emulation over 3.2e5 normals, nu = 3, 4, 10: max 1.43 ulp; none: 3.3);
    // 3 for margin.  QM_STUDENT_KC overrides it (development only).
    const char *kc_env = getenv("QM_STUDENT_KC");
    sp.kc = kc_env ? atoi(kc_env) : 3;
    if (sp.kc > K) sp.kc = K;
    if (sp.kc < 0) sp.kc = 0;
    sp.zstar = zstar;
    split_dd(sqrtq(n), &sp.sqrt_nu, &sp.sqrt_nu_lo);
    split_dd(1 / n, &sp.inv_nu, &sp.inv_nu_lo);
    split_dd(2 / n, &sp.two_over_nu, &sp.two_over_nu_lo);
    sp.acoef = (double)((n + 1) / (2 * (n + 2)));
    // log(C_n / 2) = log(n) + log(pi)/2 + lg_ratio - log 2
    const __float128 logC2 = logq(n) + logq(M_PIq) / 2 + lg_ratio - logq((__float128)2);
    split_dd(logC2, &sp.logC_hi, &sp.logC_lo);
    cache[key] = sp;
    *out = sp;
    return true;
}

}  // namespace qm

// test hook: the coefficients as the kernel receives them
extern "C" int qm_student_coefficients(double nu, int K, double *c_out)
{
    qm::StudentParams sp;
    if (!qm::student_params(nu, K, 1.0, &sp)) return 1;
    for (int k = 0; k <= K; ++k) c_out[k] = sp.c[k];
    return 0;
}
