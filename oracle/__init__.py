"""CPU ORACLE for the bulk inverse-CDF sampling hot path -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct long-double C (``orc_*.c``) that states what the
hot path of Shaw & Brickman, *Quantile Mechanics II* (arXiv 0901.0638) computes,
with a thin ctypes/numpy wrapper.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
It shares no code, header, table or constant with the CUDA product
(``paper_0901_0638_b200/``), which never imports it.

Pins (``tests/test_oracle_*.py``) tie every function to the paper or to
mathematics independent of this code (printed values, closed forms, mpmath at
40+ digits, Random123 known answers).  Functions without such a pin are marked
"parity unpinned" below and in DESIGN.md.  Unpinned: none at present; the refined
Acklam formula is pinned only away from u = 1/2 (the paper itself reports a
loss of precision at the centre).

Citations ``P:n`` are PAPER.md line numbers.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "liboracle.so"
_SRCS = ["orc_philox.c", "orc_normal.c", "orc_student.c", "orc_moments.c", "orc_mc.c", "orc_tail.c", "orc_rode.c"]

# formula ids of the oracle (local to the oracle; the product has its own enum)
C55, A77, D13 = 55, 77, 13
F1212, F88, F44, TWO_REGION = 1212, 88, 44, 410   # our fits (row f3) and the two-region variant (f4)


def build(force: bool = False) -> Path:
    """Compile liboracle.so with gcc (plain -O2, no fast-math, no contraction)."""
    srcs = [_HERE / s for s in _SRCS]
    if not force and _SO.exists():
        newest = max(os.path.getmtime(s) for s in srcs + [_HERE / "orc.h"])
        if os.path.getmtime(_SO) >= newest:
            return _SO
    cmd = ["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-ffp-contract=off",
           "-fno-fast-math", "-Wall", "-o", str(_SO)] + [str(s) for s in srcs] + ["-lm"]
    subprocess.run(cmd, check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_SO))
        P = ctypes.c_void_p
        i64, i32, dbl, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint64
        sig = {
            "orc_philox4x32_10": (None, [P, P, P]),
            "orc_philox_raw": (None, [P, i64, u64, u64]),
            "orc_philox_uniform_f32": (None, [P, i64, u64, u64]),
            "orc_philox_uniform_f64": (None, [P, i64, u64, u64]),
            "orc_philox_uniform_f32_at": (None, [P, P, i64, u64, u64]),
            "orc_philox_uniform_f64_at": (None, [P, P, i64, u64, u64]),
            "orc_ndtri_exact": (None, [P, P, i64]),
            "orc_Qexact": (None, [P, P, i64]),
            "orc_rational": (i32, [P, P, i64, i32, i32]),
            "orc_coeffs": (i32, [i32, i32, P, P]),
            "orc_normal_breakless": (i32, [P, P, i64, i32, i32]),
            "orc_normal_antithetic": (i32, [P, P, i64, i32, i32]),
            "orc_exp_to_normal": (i32, [P, P, i64, i32, i32]),
            "orc_Q_taylor": (None, [P, P, i64, i32]),
            "orc_Q_tail": (None, [P, P, i64, i32]),
            "orc_Q_taylor_coeffs": (None, [P]),
            "orc_normal_as241": (i32, [P, P, i64, i32]),
            "orc_normal_acklam": (i32, [P, P, i64, i32, i32]),
            "orc_normal_moro": (i32, [P, P, i64, i32]),
            "orc_student_coeffs_ld": (i32, [dbl, i32, P]),
            "orc_student_tail_const": (None, [dbl, P]),
            "orc_student_crossover": (dbl, [dbl, i32, P]),
            "orc_student_map": (i32, [P, P, i64, dbl, i32, P, dbl]),
            "orc_student_branches": (i32, [P, P, P, i64, dbl, i32, P]),
            "orc_student_exact": (i32, [P, P, i64, dbl]),
            "orc_student_cdf_upper_v": (None, [P, P, i64, dbl]),
            "orc_student_rode": (i32, [P, P, i64, dbl, dbl]),
            "orc_moments_f64": (None, [P, i64, i32, P]),
            "orc_moments_f32": (None, [P, i64, i32, P]),
            "orc_mc_call": (None, [i64, u64, u64, dbl, dbl, dbl, dbl, P, i32, P]),
            "orc_normal_breakless_tail": (i32, [P, P, i64, i32, i32, dbl]),
            "orc_target_masses": (i32, [i32, P, P]),
            "orc_target_density": (i32, [i32, P, P, P, i64]),
            "orc_recycle_exp_to_target": (i32, [i32, P, P, P, i64]),
            "orc_exp_to_normal_tail": (i32, [P, P, i64, i32, i32, dbl]),
            "orc_besselk_ld": (None, [dbl, dbl, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _in(x, dtype=np.float64) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=dtype))


def _chk(rc):
    if rc is not None and rc < 0:
        raise ValueError("oracle: invalid formula/argument")


# ---------------------------------------------------------------- Philox (a1)
def philox4x32_10(ctr, key) -> np.ndarray:
    c = _in(ctr, np.uint32); k = _in(key, np.uint32); o = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(o))
    return o


def philox_raw(nblocks: int, seed: int, counter_offset: int = 0) -> np.ndarray:
    o = np.zeros(4 * nblocks, np.uint32)
    lib().orc_philox_raw(_p(o), nblocks, seed, counter_offset)
    return o


def philox_uniform(n: int, seed: int, counter_offset: int = 0, dtype=np.float32) -> np.ndarray:
    """Uniforms on the odd grid, (2k+1) 2^-24 (fp32) or (2k+1) 2^-53 (fp64)."""
    o = np.zeros(n, dtype)
    if dtype == np.float32:
        lib().orc_philox_uniform_f32(_p(o), n, seed, counter_offset)
    else:
        lib().orc_philox_uniform_f64(_p(o), n, seed, counter_offset)
    return o


def philox_uniform_at(idx, seed: int, counter_offset: int = 0, dtype=np.float32) -> np.ndarray:
    """The uniforms at sample indices idx of the stream (for sampled full-size checks)."""
    idx = _in(idx, np.int64)
    o = np.zeros(idx.size, dtype)
    f = lib().orc_philox_uniform_f32_at if dtype == np.float32 else lib().orc_philox_uniform_f64_at
    f(_p(idx), _p(o), idx.size, seed, counter_offset)
    return o


# ------------------------------------------------------- normal quantile (a2-a5, a7)
def ndtri_exact(u) -> np.ndarray:
    """w(u) with Phi(w(u)) = u, long double."""
    u = _in(u); o = np.empty(u.shape, np.longdouble)
    lib().orc_ndtri_exact(_p(u), _p(o), u.size)
    return o


def Q_exact(v) -> np.ndarray:
    """Q(v) = Phi^-1(1 - e^-v/2)."""
    v = _in(v, np.longdouble); o = np.empty(v.shape, np.longdouble)
    lib().orc_Qexact(_p(v), _p(o), v.size)
    return o


def rational(v, formula: int, prec: int) -> np.ndarray:
    """v P(v)/Q(v) of formula C55/A77/D13/F1212/F88/F44/TWO_REGION; prec 32/64 rounds the
    coefficients, 0 keeps decimals."""
    v = _in(v, np.longdouble); o = np.empty(v.shape, np.longdouble)
    _chk(lib().orc_rational(_p(v), _p(o), v.size, formula, prec))
    return o


def coeffs(formula: int, prec: int):
    p = np.zeros(14, np.longdouble); q = np.zeros(14, np.longdouble)
    n = lib().orc_coeffs(formula, prec, _p(p), _p(q))
    _chk(n)
    return p[:n].copy(), q[:n].copy()


def normal_breakless(u, formula: int, prec: int) -> np.ndarray:
    u = _in(u); o = np.empty(u.shape, np.longdouble)
    _chk(lib().orc_normal_breakless(_p(u), _p(o), u.size, formula, prec))
    return o


def normal_antithetic(u, formula: int, prec: int) -> np.ndarray:
    u = _in(u); o = np.empty(2 * u.size, np.longdouble)
    _chk(lib().orc_normal_antithetic(_p(u), _p(o), u.size, formula, prec))
    return o


def exp_to_normal(v, formula: int, prec: int) -> np.ndarray:
    v = _in(v); o = np.empty(v.shape, np.longdouble)
    _chk(lib().orc_exp_to_normal(_p(v), _p(o), v.size, formula, prec))
    return o


def normal_breakless_tail(u, formula: int, prec: int, vc: float) -> np.ndarray:
    """Composite of row f2: rational for v < vc, the §5.1 tail model beyond (orc_tail.c)."""
    u = _in(u); o = np.empty(u.shape, np.longdouble)
    _chk(lib().orc_normal_breakless_tail(_p(u), _p(o), u.size, formula, prec, vc))
    return o


HYPERBOLIC, VG = 1, 2


def target_masses(kind: int, params):
    """(p-, p+, Z) of the hyperbolic (params alpha, beta, delta) or VG (lambda, alpha, beta) target
    (VG: any real lambda >= 1; P:395 puts lambda < 1 out of scope)."""
    p = _in(params); o = np.zeros(3, np.longdouble)
    _chk(lib().orc_target_masses(kind, _p(p), _p(o)))
    return o


def target_density(kind: int, params, x) -> np.ndarray:
    p = _in(params); x = _in(x); o = np.empty(x.shape, np.longdouble)
    _chk(lib().orc_target_density(kind, _p(p), _p(x), _p(o), x.size))
    return o


def besselk(nu: float, z: float):
    """K_nu(z) (long double) by the trapezoidal rule on its integral representation
    (A&S 9.6.24) -- the VG density's Bessel function for non-integer lambda."""
    o = np.zeros(1, np.longdouble)
    lib().orc_besselk_ld(nu, z, _p(o))
    return o[0]


def recycle_exp_to_target(kind: int, params, v) -> np.ndarray:
    """Q(v) = F^-1(F0(v)) by definition (quadrature + bracketed Newton on the tail mass)."""
    p = _in(params); v = _in(v); o = np.empty(v.shape, np.longdouble)
    _chk(lib().orc_recycle_exp_to_target(kind, _p(p), _p(v), _p(o), v.size))
    return o


def exp_to_normal_tail(v, formula: int, prec: int, vc: float) -> np.ndarray:
    v = _in(v); o = np.empty(v.shape, np.longdouble)
    _chk(lib().orc_exp_to_normal_tail(_p(v), _p(o), v.size, formula, prec, vc))
    return o


def Q_taylor(v, terms: int = 10) -> np.ndarray:
    v = _in(v, np.longdouble); o = np.empty(v.shape, np.longdouble)
    lib().orc_Q_taylor(_p(v), _p(o), v.size, terms)
    return o


def Q_taylor_coeffs() -> np.ndarray:
    """c_0..c_10 of the printed series Q(v) = sum c_k v^k."""
    c = np.zeros(11, np.longdouble)
    lib().orc_Q_taylor_coeffs(_p(c))
    return c


def Q_tail(v, groups: int = 4) -> np.ndarray:
    v = _in(v, np.longdouble); o = np.empty(v.shape, np.longdouble)
    lib().orc_Q_tail(_p(v), _p(o), v.size, groups)
    return o


def normal_as241(u, prec: int = 64) -> np.ndarray:
    u = _in(u); o = np.empty(u.shape, np.longdouble)
    _chk(lib().orc_normal_as241(_p(u), _p(o), u.size, prec))
    return o


def normal_acklam(u, prec: int = 64, refine: bool = False) -> np.ndarray:
    u = _in(u); o = np.empty(u.shape, np.longdouble)
    _chk(lib().orc_normal_acklam(_p(u), _p(o), u.size, prec, int(refine)))
    return o


def normal_moro(u, prec: int = 64) -> np.ndarray:
    """Moro (1995) quantile (row f4), same formula, long double."""
    u = _in(u); o = np.empty(u.shape, np.longdouble)
    _chk(lib().orc_normal_moro(_p(u), _p(o), u.size, prec))
    return o


# ------------------------------------------------------------- Student (a6)
def _mp_coeffs(n: float, K: int, dps: int = 100):
    """gamma and the recurrence of P:178-188 in mpmath at `dps` digits.

    The recurrence cancels terms of size c_i down to c_{i+1}; at 100 digits the
    result is exact to long double for n <= 100, K <= 24 (tests)."""
    import mpmath as mp
    with mp.workdps(dps):
        nn = mp.mpf(n)
        c = [mp.sqrt(nn / 2) * mp.gamma(nn / 2) / mp.gamma((nn + 1) / 2)]
        for i in range(K):
            rhs = -(2 * i + 1) * c[i]
            for l in range(i + 1):
                for m in range(i - l + 1):
                    alm = (1 + 1 / nn) * (2 * l + 1) * (2 * m + 1) - (2 / nn) * m * (2 * m + 1)
                    rhs += alm * c[i - l - m] * c[l] * c[m]
            if i >= 1:
                s = 0
                for l in range(i):
                    for m in range(i - l):
                        s += (2 * m + 1) * c[i - 1 - l - m] * c[l] * c[m]
                rhs -= s / nn
            c.append(rhs / ((2 * i + 3) * (2 * i + 2)))
        return [mp.nstr(x, 40, strip_zeros=False) for x in c]


_coef_cache = {}


def student_coeffs(n: float, K: int) -> np.ndarray:
    """c_0..c_K (long double, correctly rounded from 100-digit arithmetic)."""
    key = (float(n), int(K))
    if key not in _coef_cache:
        _coef_cache[key] = np.array([np.longdouble(s) for s in _mp_coeffs(n, K)], dtype=np.longdouble)
    return _coef_cache[key].copy()


def student_coeffs_ld(n: float, K: int) -> np.ndarray:
    """The same recurrence run in long double (documents its ill-conditioning)."""
    c = np.zeros(K + 1, np.longdouble)
    _chk(lib().orc_student_coeffs_ld(n, K, _p(c)))
    return c


def student_gamma(n: float):
    return student_coeffs(n, 0)[0]


def student_tail_const(n: float):
    o = np.zeros(1, np.longdouble)
    lib().orc_student_tail_const(n, _p(o))
    return o[0]


def student_crossover(n: float, K: int) -> float:
    c = student_coeffs(n, K)
    return lib().orc_student_crossover(n, K, _p(c))


def student_map(z, n: float, K: int, zstar: float = 0.0) -> np.ndarray:
    z = _in(z); o = np.empty(z.shape, np.longdouble); c = student_coeffs(n, K)
    _chk(lib().orc_student_map(_p(z), _p(o), z.size, n, K, _p(c), zstar))
    return o


def student_branches(z, n: float, K: int):
    z = _in(z); cc = np.empty(z.shape, np.longdouble); t = np.empty(z.shape, np.longdouble)
    c = student_coeffs(n, K)
    _chk(lib().orc_student_branches(_p(z), _p(cc), _p(t), z.size, n, K, _p(c)))
    return cc, t


def student_exact(z, n: float) -> np.ndarray:
    z = _in(z); o = np.empty(z.shape, np.longdouble)
    _chk(lib().orc_student_exact(_p(z), _p(o), z.size, n))
    return o


def student_rode(z, n: float, h: float = 1e-3) -> np.ndarray:
    """Student map by the forward RK4 solution of the Recycling ODE."""
    z = _in(z); o = np.empty(z.shape, np.longdouble)
    _chk(lib().orc_student_rode(_p(z), _p(o), z.size, n, h))
    return o


def student_cdf_upper(t, n: float) -> np.ndarray:
    t = _in(t, np.longdouble); o = np.empty(t.shape, np.longdouble)
    lib().orc_student_cdf_upper_v(_p(t), _p(o), t.size, n)
    return o


# ------------------------------------------------------------- moments (a8)
def moments(x, kmax: int = 4) -> np.ndarray:
    x = np.ascontiguousarray(x)
    S = np.zeros(kmax, np.longdouble)
    if x.dtype == np.float32:
        lib().orc_moments_f32(_p(x), x.size, kmax, _p(S))
    else:
        x = _in(x)
        lib().orc_moments_f64(_p(x), x.size, kmax, _p(S))
    return S


# -------------------------------------------------------- Monte Carlo (config 5)
def mc_call(n: int, seed: int, counter_offset: int, S0: float, r: float, sigma: float, T: float, strikes):
    """Sums of (S_T - K)^+ and its square per strike over n exponential-base samples (orc_mc.c)."""
    K = _in(strikes)
    out = np.zeros(2 * K.size, np.longdouble)
    lib().orc_mc_call(n, seed, counter_offset, S0, r, sigma, T, _p(K), K.size, _p(out))
    return out.reshape(-1, 2)


def black_scholes_call(S0: float, K, r: float, sigma: float, T: float) -> np.ndarray:
    """Closed-form European call (the pin of the Monte-Carlo sweep), via mpmath."""
    import mpmath as mp
    out = []
    for k in np.atleast_1d(K):
        d1 = (mp.log(S0 / k) + (r + sigma * sigma / 2) * T) / (sigma * mp.sqrt(T))
        d2 = d1 - sigma * mp.sqrt(T)
        out.append(float(S0 * mp.ncdf(d1) - k * mp.exp(-r * T) * mp.ncdf(d2)))
    return np.array(out)
