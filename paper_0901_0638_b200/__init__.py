"""B200-native bulk inverse-CDF sampling (Shaw & Brickman, Quantile Mechanics II,
arXiv 0901.0638): the C ABI of libqm.so (include/qm.h) and its Python binding.

The package holds only the hot path: csrc/ (sm_100a kernels + C ABI),
qm.py (binding, same names as the C entry points), shard.py (multi-GPU
sharding + the all-reduce of sums), build.py (nvcc build).
"""
from .qm import (  # noqa: F401
    ACKLAM, ACKLAM_REFINED, AS241, BREAKLESS, BREAKLESS77, BREAKLESS88, BREAKLESS1212, BREAKLESS_TAIL, HYPERBOLIC, MORO,
    STUDENT, TWO_REGION, VG, qm_abi_version,
    qm_device_sm_count, qm_exp_base_quantile, qm_exp_target_philox, qm_exp_target_table, qm_moment_row_count,
    qm_moment_rows, qm_moments, qm_normal_target_table, qm_recycle_normal_to_t_rode, qm_normal_antithetic, qm_normal_philox, qm_normal_quantile, qm_normal_quantile_host, qm_normal_quantile_plain,
    qm_mc_european_call, qm_mc_row_count, qm_philox_uniform, qm_recycle_exp_to_hyperbolic, qm_recycle_exp_to_normal,
    qm_recycle_exp_to_vg, qm_recycle_normal_to_t, qm_recycle_normal_to_t_moments, qm_reduce_rows, qm_rode_table_host, qm_student_coefficients,
    qm_student_default_crossover, QMError)
