/*
 * orc_mc.c -- ORACLE (test infrastructure only; see orc.h).
 *
 * Config 5 of BASELINE.json: a Monte-Carlo European-call sweep
 * whose normal innovations come from the EXPONENTIAL base (P:397-405, P:505:
 * "If an exponential base is used we are essentially employing the last two
 * steps"; "the overhead of converting to normal is then the evaluation of
 * a simple rational function").  Per sample:
 *   w  = Philox word (stream layout of orc_philox.c, fp32 grid),
 *   v  = -log u,  u = (2 (w >> 9) + 1) 2^-24     (one-sided unit exponential)
 *   s  = +1 if bit 8 of w is set, else -1        (two-sided / Laplace base)
 *   Z  = s Q(v),  Q = App C (5,5) rational with float-rounded coefficients
 *   S_T = S0 exp((r - sigma^2/2) T + sigma sqrt(T) Z)
 *   sums over samples of (S_T - K_j)^+ and ((S_T - K_j)^+)^2 for each strike.
 * Long double throughout; the price is exp(-rT) * mean payoff.
 */
#include <math.h>
#include <stdint.h>
#include "orc.h"

ld orc_Q_C55_f32coef(ld v);   /* orc_normal.c */

void orc_mc_call(int64_t n, uint64_t seed, uint64_t c0, double S0, double r, double sigma, double T,
                 const double *K, int nk, ld *sums /* 2*nk */)
{
    uint32_t ctr[4], key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) }, w[4];
    for (int j = 0; j < 2 * nk; ++j) sums[j] = 0.0L;
    const ld a = logl((ld)S0) + ((ld)r - 0.5L * (ld)sigma * (ld)sigma) * (ld)T;
    const ld b = (ld)sigma * sqrtl((ld)T);
    for (int64_t i = 0; i < n; ++i) {
        if (i % 4 == 0) {
            uint64_t c = c0 + (uint64_t)(i / 4);
            ctr[0] = (uint32_t)c; ctr[1] = (uint32_t)(c >> 32); ctr[2] = 0; ctr[3] = 0;
            orc_philox4x32_10(ctr, key, w);
        }
        uint32_t word = w[i % 4];
        ld u = ldexpl(2.0L * (ld)(word >> 9) + 1.0L, -24);
        ld v = 0.0L - logl(u);
        ld z = orc_Q_C55_f32coef(v);
        if (((word >> 8) & 1u) == 0u) z = -z;
        ld ST = expl(a + b * z);
        for (int j = 0; j < nk; ++j) {
            ld p = ST - (ld)K[j];
            if (p < 0.0L) p = 0.0L;
            sums[2 * j] += p;
            sums[2 * j + 1] += p * p;
        }
    }
}
