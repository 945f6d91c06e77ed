"""Min-max crossover z* of the composite normal -> Student-t map (reading R13).

Calls only oracle/ (test infrastructure).  For each (n, K): evaluate the central
series and the two-term tail and the exact map
F_n^-1(Phi(z)) on a 0.002 grid of z in (0, 12]; pick the split that minimises
max(central error below, tail error above).  Output: the rows of
tests/golden/student_crossover.txt.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402


def minmax_crossover(n, K):
    z = np.linspace(1e-3, 12.0, 6001)
    ex = O.student_exact(z, n).astype(np.float64)
    c, t = O.student_branches(z, n, K)
    ec = np.abs(c.astype(np.float64) / ex - 1)
    et = np.abs(t.astype(np.float64) / ex - 1)
    pre = np.concatenate([[0.0], np.maximum.accumulate(ec)[:-1]])
    suf = np.maximum.accumulate(et[::-1])[::-1]
    tot = np.maximum(pre, suf)
    s = int(np.argmin(tot))
    return z[s], tot[s]


# caller-supplied crossovers tested beside the shipped table (qm.h): nu x K grid
CALLER_GRID = [(n, K) for n in (2.0, 2.5, 7.0, 20.0) for K in (10, 16, 24)]

if __name__ == "__main__":
    for n, K in [(3.0, 16), (5.0, 16), (10.0, 16)]:
        zs, e = minmax_crossover(n, K)
        print(f"{int(n):<5d} {K:<4d} {zs:.4f}   {e:.3e}")
    for n, K in CALLER_GRID:
        zs, e = minmax_crossover(n, K)
        print(f"caller {n:<5g} {K:<4d} {zs:.4f}   {e:.3e}")
