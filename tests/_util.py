"""Small helpers shared by the tests (no method arithmetic)."""
import mpmath as mp
import numpy as np


def ld2mp(x):
    """Exact conversion of an x87 long double to mpmath (hi + lo doubles)."""
    x = np.longdouble(x)
    hi = float(x)
    lo = float(x - np.longdouble(hi))
    return mp.mpf(hi) + mp.mpf(lo)
