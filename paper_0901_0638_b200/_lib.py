"""ctypes loader for libqm.so (the C ABI of include/qm.h).

There is no fallback: if the shared library is missing or cannot be loaded the
import fails loudly, and every entry point checks its status code.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
# QM_LIB_PATH: load another build of the same sources (A/B experiments only)
LIB_PATH = Path(os.environ.get("QM_LIB_PATH", str(_HERE / "libqm.so")))

QM_OK, QM_EINVAL, QM_EUNSUPPORTED, QM_ECUDA = 0, 1, 2, 3
QM_F32, QM_F64 = 1, 2
QM_BREAKLESS, QM_BREAKLESS77, QM_AS241, QM_ACKLAM, QM_ACKLAM_REFINED, QM_BREAKLESS_TAIL, QM_MORO = 0, 1, 2, 3, 4, 5, 6
QM_BREAKLESS1212, QM_BREAKLESS88, QM_TWO_REGION = 7, 8, 9
QM_MOMENT_CHUNK = 65536
QM_MC_CHUNK = 1 << 20
QM_TARGET_HYPERBOLIC, QM_TARGET_VG, QM_TARGET_STUDENT = 1, 2, 3
QM_RODE_TABLE_DOUBLES = 80 + 8 * (3584 + 16384 + 4096 + 1)
QM_MC_MAX_STRIKES = 32


class McParams(ctypes.Structure):
    """qm_mc_params of include/qm.h"""
    _fields_ = [("S0", ctypes.c_double), ("r", ctypes.c_double), ("sigma", ctypes.c_double),
                ("T", ctypes.c_double), ("nstrikes", ctypes.c_int),
                ("strikes", ctypes.c_double * QM_MC_MAX_STRIKES)]

# every symbol include/qm.h declares, with (restype, argtypes)
_P, _I64, _I32, _U64, _D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_double
SIGNATURES = {
    "qm_abi_version": (_I32, []),
    "qm_status_string": (ctypes.c_char_p, [_I32]),
    "qm_device_sm_count": (_I32, []),
    "qm_normal_quantile": (_I32, [_P, _P, _I64, _I32, _I32, _P]),
    "qm_normal_antithetic": (_I32, [_P, _P, _I64, _I32, _I32, _P]),
    "qm_normal_quantile_plain": (_I32, [_P, _P, _I64, _I32, _P]),
    "qm_philox_uniform": (_I32, [_P, _I64, _I32, _U64, _U64, _P]),
    "qm_normal_philox": (_I32, [_P, _I64, _I32, _I32, _U64, _U64, _P]),
    "qm_recycle_normal_to_t": (_I32, [_P, _P, _I64, _I32, _D, _I32, _D, _P]),
    "qm_recycle_normal_to_t_moments": (_I32, [_P, _P, _I64, _I32, _D, _I32, _D, _P, _P]),
    "qm_recycle_exp_to_normal": (_I32, [_P, _P, _I64, _I32, _I32, _P]),
    "qm_exp_target_table": (_I32, [_I32, _P, _P]),
    "qm_normal_target_table": (_I32, [_I32, _P, _P]),
    "qm_recycle_normal_to_t_rode": (_I32, [_P, _P, _I64, _I32, _P, _P]),
    "qm_recycle_exp_to_hyperbolic": (_I32, [_P, _P, _I64, _I32, _P, _P]),
    "qm_recycle_exp_to_vg": (_I32, [_P, _P, _I64, _I32, _P, _P]),
    "qm_exp_base_quantile": (_I32, [_P, _P, _I64, _I32, _P, _P]),
    "qm_exp_target_philox": (_I32, [_P, _I64, _I32, _P, _U64, _U64, _P]),
    "qm_rode_table_host": (_I32, [_I32, _P, _P]),
    "qm_mc_row_count": (_I64, [_I64]),
    "qm_mc_european_call": (_I32, [_I64, _U64, _U64, _P, _P, _P]),
    "qm_moment_row_count": (_I64, [_I64]),
    "qm_moment_rows": (_I32, [_P, _I64, _I32, _P, _P]),
    "qm_reduce_rows": (_I32, [_P, _I64, _I32, _P, _P]),
    "qm_moments": (_I32, [_P, _I64, _I32, _I32, _P, _P, _P]),
    "qm_normal_quantile_host": (_I32, [_P, _P, _I64, _I32, _I32]),
    "qm_student_coefficients": (_I32, [_D, _I32, _P]),
    "qm_student_default_crossover": (_D, [_D, _I32]),
}

_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_0901_0638_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class QMError(RuntimeError):
    def __init__(self, fn: str, status: int):
        msg = load().qm_status_string(status).decode()
        super().__init__(f"{fn}: {msg} (status {status})")
        self.status = status


def check(fn: str, status: int) -> None:
    if status != QM_OK:
        raise QMError(fn, status)
