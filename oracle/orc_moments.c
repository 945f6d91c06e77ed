/*
 * orc_moments.c -- ORACLE (test infrastructure only; see orc.h).
 *
 * Row a8 of SURVEY.md §8 (not in the paper; the north star's "moment and Monte
 * Carlo price sums"): S_k = sum_i x_i^k, k = 1..kmax, accumulated in long
 * double in index order.
 */
#include <stdint.h>
#include "orc.h"

void orc_moments_f64(const double *x, int64_t n, int kmax, ld *S)
{
    for (int k = 0; k < kmax; ++k) S[k] = 0.0L;
    for (int64_t i = 0; i < n; ++i) {
        ld xi = (ld)x[i], p = 1.0L;
        for (int k = 0; k < kmax; ++k) { p *= xi; S[k] += p; }
    }
}

void orc_moments_f32(const float *x, int64_t n, int kmax, ld *S)
{
    for (int k = 0; k < kmax; ++k) S[k] = 0.0L;
    for (int64_t i = 0; i < n; ++i) {
        ld xi = (ld)x[i], p = 1.0L;
        for (int k = 0; k < kmax; ++k) { p *= xi; S[k] += p; }
    }
}
