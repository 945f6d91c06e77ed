/*
 * orc_philox.c -- ORACLE (test infrastructure only; see orc.h).
 *
 * Row a1 of SURVEY.md §8: the uniform source.  The paper samples "u in 0<u<1"
 * (§5 algorithm) and uses a placeholder rnd() that it calls "completely
 * unsuitable for real-world use" (P:551 footnote).  The north star asks for a
 * counter-based Philox generator fused into the kernel, bit-exact against the
 * oracle.  Philox4x32-10 is Salmon, Moraes, Dror & Shaw, "Parallel random
 * numbers: as easy as 1, 2, 3" (SC'11): 10 rounds of
 *     (hi0,lo0) = mulhilo(M0, x0); (hi1,lo1) = mulhilo(M1, x2)
 *     x' = (hi1 ^ x1 ^ k0, lo1, hi0 ^ x3 ^ k1, lo0)
 * with the key bumped by the Weyl constants (W0, W1) between rounds.
 * Pinned by the Random123 known-answer tests in tests/test_oracle_philox.py.
 *
 * Stream layout: key = (lo32(seed), hi32(seed));
 * block counter c -> ctr = (lo32(c), hi32(c), 0, 0).
 *   fp32: sample i of a call uses block c0 + i/4, word i%4, and
 *         u = (2*(w >> 9) + 1) * 2^-24           (odd 24-bit grid, never 0 or 1)
 *   fp64: sample i uses block c0 + i/2, words 2(i%2) (high) and 2(i%2)+1 (low):
 *         x = ((w_hi << 32) | w_lo) >> 12;  u = (2x + 1) * 2^-53
 * Both grids are symmetric (u on the grid <=> 1-u on the grid).
 */
#include <stdint.h>
#include <string.h>
#include <math.h>
#include "orc.h"

#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += PHILOX_W0; k1 += PHILOX_W1; }
        uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)x0;
        uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)x2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t y0 = hi1 ^ x1 ^ k0;
        uint32_t y1 = lo1;
        uint32_t y2 = hi0 ^ x3 ^ k1;
        uint32_t y3 = lo0;
        x0 = y0; x1 = y1; x2 = y2; x3 = y3;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

static void block_words(uint64_t seed, uint64_t c, uint32_t w[4])
{
    uint32_t ctr[4] = { (uint32_t)c, (uint32_t)(c >> 32), 0u, 0u };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    orc_philox4x32_10(ctr, key, w);
}

/* raw words: nblocks x 4 words starting at block counter c0 */
void orc_philox_raw(uint32_t *out, int64_t nblocks, uint64_t seed, uint64_t c0)
{
    for (int64_t b = 0; b < nblocks; ++b)
        block_words(seed, c0 + (uint64_t)b, out + 4 * b);
}

void orc_philox_uniform_f32(float *u, int64_t n, uint64_t seed, uint64_t c0)
{
    uint32_t w[4];
    for (int64_t i = 0; i < n; ++i) {
        if (i % 4 == 0) block_words(seed, c0 + (uint64_t)(i / 4), w);
        uint32_t k = w[i % 4] >> 9;                       /* 23 bits */
        double num = 2.0 * (double)k + 1.0;               /* odd, < 2^24: exact */
        u[i] = (float)ldexp(num, -24);                    /* exact in float */
    }
}

void orc_philox_uniform_f64(double *u, int64_t n, uint64_t seed, uint64_t c0)
{
    uint32_t w[4];
    for (int64_t i = 0; i < n; ++i) {
        if (i % 2 == 0) block_words(seed, c0 + (uint64_t)(i / 2), w);
        int j = (int)(i % 2);
        uint64_t x = (((uint64_t)w[2 * j] << 32) | (uint64_t)w[2 * j + 1]) >> 12;   /* 52 bits */
        ld num = 2.0L * (ld)x + 1.0L;                     /* odd, < 2^53: exact */
        u[i] = (double)ldexpl(num, -53);                  /* exact in double */
    }
}

/* uniforms at arbitrary sample indices idx[j] of the stream (same layout) */
void orc_philox_uniform_f32_at(const int64_t *idx, float *u, int64_t n, uint64_t seed, uint64_t c0)
{
    uint32_t w[4];
    for (int64_t j = 0; j < n; ++j) {
        block_words(seed, c0 + (uint64_t)(idx[j] / 4), w);
        uint32_t k = w[idx[j] % 4] >> 9;
        u[j] = (float)ldexp(2.0 * (double)k + 1.0, -24);
    }
}

void orc_philox_uniform_f64_at(const int64_t *idx, double *u, int64_t n, uint64_t seed, uint64_t c0)
{
    uint32_t w[4];
    for (int64_t j = 0; j < n; ++j) {
        block_words(seed, c0 + (uint64_t)(idx[j] / 2), w);
        int h = (int)(idx[j] % 2);
        uint64_t x = (((uint64_t)w[2 * h] << 32) | (uint64_t)w[2 * h + 1]) >> 12;
        u[j] = (double)ldexpl(2.0L * (ld)x + 1.0L, -53);
    }
}
