"""The C ABI without a GPU: libqm.so builds, loads, exports every symbol that
include/qm.h declares, validates arguments before any launch, and its host-side
Student setup (__float128 recurrence) agrees with the oracle's
independent 100-digit recurrence."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    from paper_0901_0638_b200 import build, _lib
    build.build()
    return _lib.load()


def declared_symbols():
    text = (ROOT / "include" / "qm.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qm_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_north_star_entry_points():
    syms = declared_symbols()
    for name in ["qm_normal_quantile", "qm_recycle_normal_to_t", "qm_recycle_exp_to_normal",
                 "qm_normal_philox", "qm_philox_uniform", "qm_moments", "qm_normal_quantile_host"]:
        assert name in syms


def test_every_declared_symbol_is_exported(lib):
    from paper_0901_0638_b200 import _lib
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"binding lacks {name}"
    assert lib.qm_abi_version() == 1


def test_argument_validation_before_launch(lib):
    from paper_0901_0638_b200 import _lib as L
    p = ctypes.c_void_p(16)
    assert lib.qm_normal_quantile(p, p, -1, L.QM_F32, 0, None) == L.QM_EINVAL
    assert lib.qm_normal_quantile(None, p, 5, L.QM_F32, 0, None) == L.QM_EINVAL
    assert lib.qm_normal_quantile(p, p, 5, 3, 0, None) == L.QM_EINVAL
    assert lib.qm_normal_quantile(p, p, 5, L.QM_F32, L.QM_TWO_REGION + 1, None) == L.QM_EINVAL
    assert lib.qm_normal_quantile(p, p, 5, L.QM_F32, L.QM_AS241, None) == L.QM_EUNSUPPORTED
    assert lib.qm_normal_quantile(p, p, 5, L.QM_F32, L.QM_MORO, None) == L.QM_EUNSUPPORTED
    assert lib.qm_normal_quantile(p, p, 5, L.QM_F32, L.QM_BREAKLESS1212, None) == L.QM_EUNSUPPORTED
    assert lib.qm_normal_quantile(p, p, 5, L.QM_F64, L.QM_TWO_REGION, None) == L.QM_EUNSUPPORTED
    assert lib.qm_normal_quantile(p, p, 5, L.QM_F64, L.QM_TWO_REGION + 1, None) == L.QM_EINVAL
    assert lib.qm_normal_antithetic(p, p, 4, L.QM_F32, L.QM_TWO_REGION, None) == L.QM_EUNSUPPORTED
    assert lib.qm_normal_philox(p, 5, L.QM_F64, L.QM_MORO, 1, 0, None) == L.QM_EUNSUPPORTED
    assert lib.qm_normal_quantile(p, p, 0, L.QM_F32, 0, None) == L.QM_OK       # n = 0: no-op
    assert lib.qm_normal_antithetic(p, p, 4, L.QM_F64, L.QM_ACKLAM, None) == L.QM_EUNSUPPORTED
    assert lib.qm_recycle_normal_to_t(p, p, 4, L.QM_F64, -1.0, 10, 0.0, None) == L.QM_EINVAL
    # zstar <= 0: the validated table (qm.h); (5, 10) is not in it
    assert lib.qm_recycle_normal_to_t(p, p, 4, L.QM_F64, 5.0, 10, 0.0, None) == L.QM_EUNSUPPORTED
    assert lib.qm_recycle_normal_to_t(p, p, 4, L.QM_F64, 7.0, 16, -1.0, None) == L.QM_EUNSUPPORTED
    assert lib.qm_recycle_normal_to_t(p, p, 0, L.QM_F64, 5.0, 16, 0.0, None) == L.QM_OK
    assert lib.qm_recycle_normal_to_t(p, p, 0, L.QM_F64, 7.0, 16, 5.6185, None) == L.QM_OK   # caller zstar
    assert lib.qm_recycle_normal_to_t(p, p, 4, L.QM_F64, 5.0, 16, float("nan"), None) == L.QM_EINVAL
    assert lib.qm_recycle_normal_to_t_moments(p, p, 4, L.QM_F64, 5.0, 10, 0.0, p, None) == L.QM_EUNSUPPORTED
    assert lib.qm_recycle_normal_to_t(p, p, 4, L.QM_F64, 50.0, 16, 5.0, None) == L.QM_EUNSUPPORTED
    assert lib.qm_recycle_normal_to_t(p, p, 4, L.QM_F64, 4.0, 0, 3.9, None) == L.QM_EINVAL
    assert lib.qm_moments(p, 10, L.QM_F64, 5, p, p, None) == L.QM_EINVAL
    assert lib.qm_reduce_rows(p, 4, 65, p, None) == L.QM_EINVAL
    assert lib.qm_moment_row_count(65536 * 3 + 1) == 4
    assert lib.qm_philox_uniform(None, 3, L.QM_F32, 1, 0, None) == L.QM_EINVAL
    assert lib.qm_normal_quantile_host(p, p, -3, L.QM_F32, 0) == L.QM_EINVAL
    assert lib.qm_status_string(L.QM_EUNSUPPORTED).decode() == "unsupported combination"
    # §3.6 Student table (R35): kind, nu range -- all decided before any CUDA call
    nu = (ctypes.c_double * 3)
    assert lib.qm_normal_target_table(L.QM_TARGET_HYPERBOLIC, nu(4.0), p) == L.QM_EINVAL
    assert lib.qm_normal_target_table(L.QM_TARGET_STUDENT, None, p) == L.QM_EINVAL
    assert lib.qm_normal_target_table(L.QM_TARGET_STUDENT, nu(4.0), None) == L.QM_EINVAL
    assert lib.qm_normal_target_table(L.QM_TARGET_STUDENT, nu(0.0), p) == L.QM_EINVAL
    assert lib.qm_normal_target_table(L.QM_TARGET_STUDENT, nu(float("nan")), p) == L.QM_EINVAL
    assert lib.qm_normal_target_table(L.QM_TARGET_STUDENT, nu(0.5), p) == L.QM_EUNSUPPORTED
    assert lib.qm_normal_target_table(L.QM_TARGET_STUDENT, nu(201.0), p) == L.QM_EUNSUPPORTED
    assert lib.qm_recycle_normal_to_t_rode(p, p, 4, L.QM_F64, None, None) == L.QM_EINVAL
    assert lib.qm_recycle_normal_to_t_rode(p, p, 4, 3, p, None) == L.QM_EINVAL
    assert lib.qm_recycle_normal_to_t_rode(p, p, 0, L.QM_F64, p, None) == L.QM_OK


@pytest.mark.parametrize("nu,K", [(4.0, 10), (3.0, 16), (5.0, 16), (10.0, 16), (10.0, 24), (20.0, 16), (1.0, 12)])
def test_student_host_coefficients_match_oracle(lib, nu, K):
    """Product: __float128 recurrence on the host.  Oracle: mpmath at 100 digits.
    Independent implementations; the double coefficients must agree to 1 ulp."""
    import oracle as O
    from paper_0901_0638_b200 import qm_student_coefficients
    got = qm_student_coefficients(nu, K)
    ref = O.student_coeffs(nu, K)
    ref_d = ref.astype(np.float64)
    # 113 bits absorb the recurrence's cancellation up to nu ~ 10; at nu = 20 the
    # last coefficient (weight c_16 z^32 / t < 1e-20 on |z| < z*) may be 2 ulp off
    tol = 1 if nu <= 10 else 2
    assert np.all(np.abs(got - ref_d) <= tol * np.spacing(np.abs(ref_d))), (got - ref_d) / np.spacing(np.abs(ref_d))


def test_student_validated_table_matches_the_golden_crossovers(lib):
    """The crossovers the library ships (zstar <= 0) are the paper's and the
    oracle-computed min-max ones of tests/golden/student_crossover.txt (reading R13)."""
    rows = [l.split() for l in (ROOT / "tests" / "golden" / "student_crossover.txt").read_text().splitlines()
            if l.strip() and not l.startswith("#")]
    shipped = [r for r in rows if len(r) == 4]
    assert len(shipped) == 4
    for nu, K, zs, _ in shipped:
        assert lib.qm_student_default_crossover(float(nu), int(K)) == float(zs)
    assert lib.qm_student_default_crossover(4.0, 10) == 3.93473
    assert lib.qm_student_default_crossover(4.0, 16) == 0.0
    assert lib.qm_student_default_crossover(7.0, 16) == 0.0


def test_binding_validates_buffers_before_the_library():
    """qm.py routes every out/rows/table through one validator: CPU tensors, wrong
    dtypes and wrong sizes are rejected before any call into libqm (no fallback)."""
    import torch
    from paper_0901_0638_b200 import qm
    t = torch.zeros(4)
    with pytest.raises(ValueError, match="CUDA"):
        qm.qm_normal_quantile(t)
    with pytest.raises(ValueError, match="CUDA"):
        qm.qm_normal_philox(4, 1, out=t)
    with pytest.raises(ValueError, match="CUDA"):
        qm.qm_mc_european_call(1 << 20, 1, 0, 100.0, 0.05, 0.2, 1.0, [100.0], out=torch.zeros(2, dtype=torch.float64))
    with pytest.raises(ValueError, match="CUDA"):
        qm._table(torch.zeros(8, dtype=torch.float64))
    assert qm._student_K(4.0, None) == 10 and qm._student_K(5.0, None) == 16 and qm._student_K(5.0, 24) == 24
