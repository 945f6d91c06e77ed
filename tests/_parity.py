"""ULP comparison of a GPU result with the oracle's long-double value (no method arithmetic)."""
import math

import numpy as np


def ulp_errors(got: np.ndarray, ref_ld: np.ndarray, dtype) -> np.ndarray:
    """|got - ref| in ulps of ref rounded to `dtype`; specials must match exactly
    (inf with the same sign, NaN with NaN, zero with the same sign) -> 0, else inf."""
    got = np.asarray(got, dtype=dtype)
    ref_ld = np.asarray(ref_ld, dtype=np.longdouble)
    ref_t = ref_ld.astype(dtype)
    err = np.zeros(got.shape, dtype=np.float64)
    if got.size == 0:
        return err
    fin = np.isfinite(ref_t) & (ref_t != 0)
    spacing = np.spacing(np.abs(ref_t[fin])).astype(np.longdouble)
    e = (np.abs(got[fin].astype(np.longdouble) - ref_ld[fin]) / spacing).astype(np.float64)
    err[fin] = np.where(np.isnan(e), np.inf, e)
    # a finite reference beyond the target type's range must round to +-inf
    ovf = np.isfinite(ref_ld) & np.isinf(ref_t)
    err[ovf] = np.where(got[ovf] == ref_t[ovf], 0.0, np.inf)
    nan_ref = np.isnan(ref_ld)
    err[nan_ref] = np.where(np.isnan(got[nan_ref]), 0.0, np.inf)
    inf_ref = np.isinf(ref_ld)
    err[inf_ref] = np.where(got[inf_ref] == ref_t[inf_ref], 0.0, np.inf)
    zero_ref = (ref_t == 0) & ~nan_ref
    ok0 = (got[zero_ref] == 0) & (np.signbit(got[zero_ref]) == np.signbit(ref_t[zero_ref]))
    # a nonzero ref that rounds to 0 in the target type is compared absolutely
    tiny = zero_ref & (ref_ld != 0)
    err[zero_ref] = np.where(ok0, 0.0, np.inf)
    if np.any(tiny):
        err[tiny] = np.where(np.abs(got[tiny].astype(np.longdouble) - ref_ld[tiny]) <=
                             np.finfo(dtype).smallest_subnormal, 0.0, np.inf)
    return err


def summary(err: np.ndarray) -> dict:
    if err.size == 0:
        return {"max_ulp": 0.0, "hist": []}
    h = np.histogram(np.minimum(err, 8.0), bins=[0, 0.5, 1, 1.5, 2, 3, 4, 8, 9])[0]
    return {"max_ulp": float(err.max()) if err.size else 0.0, "hist": h.tolist()}


def student_rode_bar(z, t, nu):
    """Accuracy bar of the interpolated Student map (qm.h): 4e-15 + 16 eps (1 + kappa),
    kappa = |z t'(z) / t(z)| the map's condition number, t' = phi(z) / f_nu(t) (the
    quantile ODE).  The kernel's node coordinate s = n (|z|/Wc)^(1/4) and, in
    the tail, the interpolated log|t| carry roundings of a few ulp of z, which kappa
    amplifies (kappa ~ 20 at |z| = 4.5 for nu = 1, ~ z^2/nu in the tail)."""
    z = np.abs(np.asarray(z, np.float64))
    t = np.abs(np.asarray(t, np.float64))
    x = t / math.sqrt(nu)
    with np.errstate(over="ignore", divide="ignore"):
        l1p = np.where(x > 1e100, 2 * np.log(x), np.log1p(np.minimum(x, 1e100) ** 2))    # log(1 + x^2)
    lf = math.lgamma((nu + 1) / 2) - math.lgamma(nu / 2) - 0.5 * math.log(nu * math.pi) - 0.5 * (nu + 1) * l1p
    lphi = -0.5 * z * z - 0.5 * math.log(2 * math.pi)
    kappa = z * np.exp(lphi - lf - np.log(t))
    return 4e-15 + 16 * 2.0 ** -53 * (1 + kappa)
