"""Python binding of libqm.so -- argument marshalling only.

Each function has the name of the C entry point it calls (include/qm.h) and
takes torch tensors: CUDA tensors for the device entry points, CPU tensors for
qm_normal_quantile_host.  Outputs are allocated with torch when not given.
PyTorch is used for device memory and streams only; every element is computed
by the sm_100a kernels in csrc/.
"""
from __future__ import annotations

import torch

from . import _lib as L
from ._lib import QMError  # noqa: F401

BREAKLESS, BREAKLESS77, AS241, ACKLAM, ACKLAM_REFINED, BREAKLESS_TAIL, MORO = (
    L.QM_BREAKLESS, L.QM_BREAKLESS77, L.QM_AS241, L.QM_ACKLAM, L.QM_ACKLAM_REFINED, L.QM_BREAKLESS_TAIL, L.QM_MORO)
BREAKLESS1212, BREAKLESS88, TWO_REGION = L.QM_BREAKLESS1212, L.QM_BREAKLESS88, L.QM_TWO_REGION


def _prec(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return L.QM_F32
    if t.dtype == torch.float64:
        return L.QM_F64
    raise TypeError(f"unsupported dtype {t.dtype} (float32 or float64)")


def _dev(t: torch.Tensor, name: str) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _buf(t: torch.Tensor, name: str, dtype, numel: int | None = None, min_numel: int | None = None) -> torch.Tensor:
    """The one validator of every caller-supplied device buffer (out, rows, table):
    a contiguous CUDA tensor of `dtype` with exactly `numel` (or at least
    `min_numel`) elements -- the kernels write or read that many."""
    _dev(t, name)
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} must have {numel} elements, got {t.numel()}")
    if min_numel is not None and t.numel() < min_numel:
        raise ValueError(f"{name} must have at least {min_numel} elements, got {t.numel()}")
    return t


def _out(x: torch.Tensor, out, numel: int | None = None, dtype=None) -> torch.Tensor:
    n = x.numel() if numel is None else numel
    if out is None:
        return torch.empty(n, dtype=dtype or x.dtype, device=x.device)
    _buf(out, "out", dtype or x.dtype, numel=n)
    if out.device != x.device:
        raise ValueError("out must be on the input's device")
    return out


def _gen_out(out, n: int, dtype, device) -> torch.Tensor:
    """Output of a generator entry point (no input tensor): n elements of dtype."""
    if n < 0:
        raise ValueError("n must be >= 0")
    if out is None:
        return torch.empty(n, dtype=dtype, device=device or "cuda")
    return _buf(out, "out", out.dtype if dtype is None else dtype, numel=n)


def qm_normal_quantile(u: torch.Tensor, out=None, alg: int = BREAKLESS, stream=None) -> torch.Tensor:
    _dev(u, "u")
    z = _out(u, out)
    L.check("qm_normal_quantile", L.load().qm_normal_quantile(
        u.data_ptr(), z.data_ptr(), u.numel(), _prec(u), alg, _stream(stream)))
    return z


def qm_normal_quantile_plain(u: torch.Tensor, out=None, alg: int = BREAKLESS, stream=None) -> torch.Tensor:
    """Plain-double version of the formula (config 1 like-for-like timing, Table 3)."""
    _dev(u, "u")
    if u.dtype != torch.float64:
        raise ValueError("qm_normal_quantile_plain is fp64 only")
    z = _out(u, out)
    L.check("qm_normal_quantile_plain", L.load().qm_normal_quantile_plain(
        u.data_ptr(), z.data_ptr(), u.numel(), alg, _stream(stream)))
    return z


def qm_normal_antithetic(u: torch.Tensor, out=None, alg: int = BREAKLESS, stream=None) -> torch.Tensor:
    _dev(u, "u")
    z = _out(u, out, 2 * u.numel())
    L.check("qm_normal_antithetic", L.load().qm_normal_antithetic(
        u.data_ptr(), z.data_ptr(), u.numel(), _prec(u), alg, _stream(stream)))
    return z


def qm_philox_uniform(n: int, seed: int, counter_offset: int = 0, dtype=torch.float32,
                      out=None, device=None, stream=None) -> torch.Tensor:
    u = _gen_out(out, n, None if out is not None else dtype, device)
    L.check("qm_philox_uniform", L.load().qm_philox_uniform(
        u.data_ptr(), n, _prec(u), seed, counter_offset, _stream(stream)))
    return u


def qm_normal_philox(n: int, seed: int, counter_offset: int = 0, dtype=torch.float32, alg: int = BREAKLESS,
                     out=None, device=None, stream=None) -> torch.Tensor:
    z = _gen_out(out, n, None if out is not None else dtype, device)
    L.check("qm_normal_philox", L.load().qm_normal_philox(
        z.data_ptr(), n, _prec(z), alg, seed, counter_offset, _stream(stream)))
    return z


def _student_K(nu: float, K):
    """K = None: the order of the validated configuration (qm.h): 10 for the paper's
    nu = 4, 16 otherwise."""
    return (10 if float(nu) == 4.0 else 16) if K is None else int(K)


def qm_recycle_normal_to_t(z: torch.Tensor, nu: float, K: int | None = None, zstar: float = 0.0,
                           out=None, stream=None) -> torch.Tensor:
    """zstar <= 0: the library's validated crossover for (nu, K) (qm.h), else
    QMError(QM_EUNSUPPORTED); zstar > 0: the caller's crossover."""
    _dev(z, "z")
    K = _student_K(nu, K)
    t = _out(z, out)
    L.check("qm_recycle_normal_to_t", L.load().qm_recycle_normal_to_t(
        z.data_ptr(), t.data_ptr(), z.numel(), _prec(z), float(nu), int(K), float(zstar), _stream(stream)))
    return t


def qm_recycle_normal_to_t_moments(z: torch.Tensor, nu: float, K: int | None = None, zstar: float = 0.0, out=None,
                                   rows=None, stream=None):
    """t = qm_recycle_normal_to_t(z) and its moment rows ((rows, 4) fp64) in one pass."""
    _dev(z, "z")
    K = _student_K(nu, K)
    t = _out(z, out)
    nr = qm_moment_row_count(z.numel())
    if rows is None:
        rows = torch.empty((nr, 4), dtype=torch.float64, device=z.device)
    _buf(rows, "rows", torch.float64, numel=4 * nr)
    L.check("qm_recycle_normal_to_t_moments", L.load().qm_recycle_normal_to_t_moments(
        z.data_ptr(), t.data_ptr(), z.numel(), _prec(z), float(nu), int(K), float(zstar), rows.data_ptr(),
        _stream(stream)))
    return t, rows


def qm_recycle_exp_to_normal(v: torch.Tensor, out=None, alg: int = BREAKLESS, stream=None) -> torch.Tensor:
    _dev(v, "v")
    z = _out(v, out)
    L.check("qm_recycle_exp_to_normal", L.load().qm_recycle_exp_to_normal(
        v.data_ptr(), z.data_ptr(), v.numel(), _prec(v), alg, _stream(stream)))
    return z


HYPERBOLIC, VG, STUDENT = L.QM_TARGET_HYPERBOLIC, L.QM_TARGET_VG, L.QM_TARGET_STUDENT


def _params(p):
    import ctypes
    arr = (ctypes.c_double * 3)(*[float(x) for x in p])
    return arr


def qm_exp_target_table(kind: int, params, device=None) -> torch.Tensor:
    """Device table of the exponential-base recycling map (hyperbolic: alpha, beta, delta;
    VG: lambda, alpha, beta)."""
    tab = torch.empty(L.QM_RODE_TABLE_DOUBLES, dtype=torch.float64, device=device or "cuda")
    L.check("qm_exp_target_table", L.load().qm_exp_target_table(kind, _params(params), tab.data_ptr()))
    return tab


def qm_normal_target_table(kind: int, params, device=None) -> torch.Tensor:
    """Device table of the Gaussian-base recycling map solved from the RODE
    (STUDENT: nu)."""
    tab = torch.empty(L.QM_RODE_TABLE_DOUBLES, dtype=torch.float64, device=device or "cuda")
    L.check("qm_normal_target_table", L.load().qm_normal_target_table(kind, _params(params), tab.data_ptr()))
    return tab


def qm_rode_table_host(kind: int, params):
    """The same table in host memory (numpy), for diagnostics."""
    import ctypes
    import numpy as np
    tab = np.zeros(L.QM_RODE_TABLE_DOUBLES, np.float64)
    if L.load().qm_rode_table_host(kind, _params(params), tab.ctypes.data_as(ctypes.c_void_p)) != 0:
        raise ValueError("bad target parameters")
    return tab


def _table(table: torch.Tensor) -> torch.Tensor:
    return _buf(table, "table", torch.float64, numel=L.QM_RODE_TABLE_DOUBLES)


def _rode_call(name, v, table, out, stream):
    _dev(v, "v")
    _table(table)
    x = _out(v, out)
    L.check(name, getattr(L.load(), name)(v.data_ptr(), x.data_ptr(), v.numel(), _prec(v), table.data_ptr(),
                                          _stream(stream)))
    return x


def qm_recycle_exp_to_hyperbolic(v: torch.Tensor, table: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    return _rode_call("qm_recycle_exp_to_hyperbolic", v, table, out, stream)


def qm_recycle_exp_to_vg(v: torch.Tensor, table: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    return _rode_call("qm_recycle_exp_to_vg", v, table, out, stream)


def qm_recycle_normal_to_t_rode(z: torch.Tensor, table: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    return _rode_call("qm_recycle_normal_to_t_rode", z, table, out, stream)


def qm_exp_base_quantile(u: torch.Tensor, table: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    return _rode_call("qm_exp_base_quantile", u, table, out, stream)


def qm_exp_target_philox(n: int, table: torch.Tensor, seed: int, counter_offset: int = 0, dtype=torch.float64,
                         out=None, stream=None) -> torch.Tensor:
    _table(table)
    x = _gen_out(out, n, None if out is not None else dtype, table.device)
    L.check("qm_exp_target_philox", L.load().qm_exp_target_philox(x.data_ptr(), n, _prec(x), table.data_ptr(), seed,
                                                                  counter_offset, _stream(stream)))
    return x


def qm_mc_row_count(n: int) -> int:
    return L.load().qm_mc_row_count(n)


def qm_mc_european_call(n: int, seed: int, counter_offset: int, S0: float, r: float, sigma: float, T: float,
                        strikes, out=None, device=None, stream=None) -> torch.Tensor:
    """Config-5 Monte-Carlo call sweep rows, shape (qm_mc_row_count(n), 2 * nstrikes) fp64."""
    import ctypes
    ks = [float(k) for k in strikes]
    if not 1 <= len(ks) <= L.QM_MC_MAX_STRIKES:
        raise ValueError("1..32 strikes")
    p = L.McParams(S0, r, sigma, T, len(ks), (ctypes.c_double * L.QM_MC_MAX_STRIKES)(*ks))
    nr = qm_mc_row_count(n)
    rows = out if out is not None else torch.empty((max(nr, 1), 2 * len(ks)), dtype=torch.float64,
                                                   device=device or "cuda")
    _buf(rows, "out", torch.float64, min_numel=nr * 2 * len(ks))
    L.check("qm_mc_european_call", L.load().qm_mc_european_call(n, seed, counter_offset, ctypes.byref(p),
                                                                rows.data_ptr(), _stream(stream)))
    return rows


def qm_moment_row_count(n: int) -> int:
    return L.load().qm_moment_row_count(n)


def qm_moment_rows(x: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    """Fixed-chunk moment rows, shape (qm_moment_row_count(n), 4) fp64."""
    _dev(x, "x")
    nr = qm_moment_row_count(x.numel())
    rows = out if out is not None else torch.empty((nr, 4), dtype=torch.float64, device=x.device)
    _buf(rows, "out", torch.float64, min_numel=4 * nr)
    L.check("qm_moment_rows", L.load().qm_moment_rows(x.data_ptr(), x.numel(), _prec(x), rows.data_ptr(),
                                                      _stream(stream)))
    return rows


def qm_reduce_rows(rows: torch.Tensor, out=None, stream=None) -> torch.Tensor:
    """Fixed-order column sums of a (nrows, ncol) fp64 matrix."""
    _buf(rows, "rows", torch.float64)
    if rows.dim() != 2:
        raise ValueError("rows must be a (nrows, ncol) matrix")
    nrows, ncol = rows.shape
    o = out if out is not None else torch.empty(ncol, dtype=torch.float64, device=rows.device)
    _buf(o, "out", torch.float64, min_numel=ncol)
    L.check("qm_reduce_rows", L.load().qm_reduce_rows(rows.data_ptr(), nrows, ncol, o.data_ptr(), _stream(stream)))
    return o


def qm_moments(x: torch.Tensor, kmax: int = 4, out=None, rows=None, stream=None) -> torch.Tensor:
    """S_k = sum x^k, k = 1..kmax, fp64 on the device (deterministic)."""
    _dev(x, "x")
    nr = qm_moment_row_count(x.numel())
    ws = rows if rows is not None else torch.empty(max(nr, 1) * 4, dtype=torch.float64, device=x.device)
    _buf(ws, "rows", torch.float64, min_numel=4 * nr)
    o = out if out is not None else torch.empty(kmax, dtype=torch.float64, device=x.device)
    _buf(o, "out", torch.float64, min_numel=kmax)
    L.check("qm_moments", L.load().qm_moments(x.data_ptr(), x.numel(), _prec(x), kmax, o.data_ptr(),
                                              ws.data_ptr(), _stream(stream)))
    return o


def qm_normal_quantile_host(u: torch.Tensor, out=None, alg: int = BREAKLESS) -> torch.Tensor:
    """Host buffers in and out; the copies and the kernels run inside the call."""
    if u.is_cuda or not u.is_contiguous():
        raise ValueError("u must be a contiguous CPU tensor")
    z = out if out is not None else torch.empty_like(u)
    if z.is_cuda or z.numel() != u.numel() or z.dtype != u.dtype:
        raise ValueError("out must be a CPU tensor like u")
    L.check("qm_normal_quantile_host", L.load().qm_normal_quantile_host(
        u.data_ptr(), z.data_ptr(), u.numel(), _prec(u), alg))
    return z


def qm_student_default_crossover(nu: float, K: int) -> float:
    """The shipped crossover of a validated (nu, K) (qm.h), 0.0 if none."""
    return L.load().qm_student_default_crossover(float(nu), int(K))


def qm_student_coefficients(nu: float, K: int):
    import ctypes
    import numpy as np
    c = np.zeros(K + 1, np.float64)
    rc = L.load().qm_student_coefficients(float(nu), int(K), c.ctypes.data_as(ctypes.c_void_p))
    if rc != 0:
        raise ValueError("unsupported nu/K")
    return c


def qm_abi_version() -> int:
    return L.load().qm_abi_version()


def qm_device_sm_count() -> int:
    return L.load().qm_device_sm_count()
