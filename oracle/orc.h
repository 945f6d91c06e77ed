/*
 * orc.h -- internal header of the CPU ORACLE (test infrastructure only).
 *
 * The oracle is a plain, slow, obviously-correct CPU program that states what
 * the hot path of Shaw & Brickman, "Quantile Mechanics II" (arXiv 0901.0638)
 * computes.  It is used ONLY by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py.  It shares no code, header,
 * table or constant with the CUDA product path (paper_0901_0638_b200/), and the
 * product never links, imports or calls it.
 *
 * Arithmetic: x87 80-bit `long double` (64-bit significand) throughout; libm's
 * long-double special functions (logl, erfl, erfcl, lgammal, expl, powl).
 * Citations "P:n" are PAPER.md line numbers (section in brackets).
 */
#ifndef ORC_H
#define ORC_H
#include <stdint.h>

typedef long double ld;

/* ---- orc_philox.c ---- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* ---- orc_normal.c ---- */
ld orc_ndtri_exact_ld(ld u);
ld orc_Qexact_ld(ld v);

#endif
