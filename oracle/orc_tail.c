/*
 * orc_tail.c -- ORACLE (test infrastructure only; see orc.h).
 *
 * precision in the deep tail.  The paper proposes to
 * "sample the tail interval completely separately and apply a transformed
 * quantile to that region by itself" with the supplementary model
 * Q(v) = sqrt(2 q(a,b)) of §5.1 (reading R1: a = v - 1/2 log pi,
 * b = log a), "precision better than 1.06e-9 ... in the region v >= 37".
 * Composite: Q(v) = rational(v) for v < vc, tail model for v >= vc, with
 * vc = 37 for the single-precision rationals and vc = 86.75 for App D
 * (reading R23: where the tail model's error drops below App D's).
 */
#include <math.h>
#include <stdint.h>
#include "orc.h"

ld orc_Q_tail_ld(ld v, int groups);                    /* orc_normal.c */
int orc_rational(const ld *v, ld *out, int64_t n, int formula, int prec);

static ld composite(ld v, int formula, int prec, double vc)
{
    if (v < (ld)vc) {
        ld o;
        orc_rational(&v, &o, 1, formula, prec);
        return o;
    }
    return orc_Q_tail_ld(v, 4);
}

int orc_normal_breakless_tail(const double *u, ld *out, int64_t n, int formula, int prec, double vc)
{
    for (int64_t i = 0; i < n; ++i) {
        ld ui = (ld)u[i], r;
        if (isnan(ui) || ui < 0.0L || ui > 1.0L) r = NAN;
        else if (ui == 0.0L) r = -INFINITY;
        else if (ui == 1.0L) r = INFINITY;
        else {
            ld vv = (ui < 0.5L) ? ui : 1.0L - ui;
            ld z = 0.0L - logl(2.0L * vv);
            ld q = composite(z, formula, prec, vc);
            r = (ui >= 0.5L) ? q : -q;
        }
        out[i] = r;
    }
    return 0;
}

int orc_exp_to_normal_tail(const double *v, ld *out, int64_t n, int formula, int prec, double vc)
{
    for (int64_t i = 0; i < n; ++i) {
        ld vi = (ld)v[i], a = fabsl(vi), q;
        if (isnan(vi)) q = NAN;
        else if (isinf(vi)) q = INFINITY;
        else q = composite(a, formula, prec, vc);
        out[i] = signbit(vi) ? -q : q;
    }
    return 0;
}
