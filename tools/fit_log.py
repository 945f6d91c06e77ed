"""Design-time fits for the kernels' log polynomials (product constants in csrc/qm_math.cuh).

fp32: R(f) = (log1p(f) - f)/f^2 on f in [-1/3, 1/3], degree 7 (Chebyshev fit, mpmath).
fp64: T(w) = (2 atanh(s) - 2 s)/s^3, w = s^2 in [0, 1/25], degree 7.
Prints the coefficients (ascending powers) and the fit errors.
"""
import mpmath as mp
import numpy as np

mp.mp.dps = 40


def R(f):
    if abs(f) < mp.mpf("1e-12"):
        return mp.mpf(-0.5) + f / 3 - f * f / 4
    return (mp.log1p(f) - f) / (f * f)


def T(w):
    if w < mp.mpf("1e-30"):
        return mp.mpf(2) / 3
    s = mp.sqrt(w)
    return (2 * mp.atanh(s) - 2 * s) / (s ** 3)


if __name__ == "__main__":
    poly, err = mp.chebyfit(R, [-mp.mpf(1) / 3, mp.mpf(1) / 3], 8, error=True)
    print("fp32 R, err", mp.nstr(err, 5), [repr(float(np.float32(float(x)))) for x in poly[::-1]])
    pol, e = mp.chebyfit(T, [0, mp.mpf(1) / 25], 8, error=True)
    print("fp64 T, err", mp.nstr(e, 5), [repr(float(x)) for x in pol[::-1]])
