"""Stress the TMA-ring kernels: repeat each map many times and compare bitwise with
the LDG kernels (misaligned views: no TMA ring).  python tools/stress_tl.py [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0901_0638_b200 as Q  # noqa: E402
from synth import inputs as I  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
n = (1 << 24) + 37


def pair(dtype, gen):
    x = torch.from_numpy(np.concatenate([[dtype(0.5)], gen(n, dtype=dtype)]).astype(dtype)).cuda()
    return x[1:].clone(), x[1:]                      # aligned (ring) / misaligned (LDG)


cases = []
a32, m32 = pair(np.float32, I.mixed_uniforms)
cases.append(("normal_f32", lambda x: Q.qm_normal_quantile(x), a32, m32))
cases.append(("antithetic_f32", lambda x: Q.qm_normal_antithetic(x), a32, m32))
a64, m64 = pair(np.float64, I.mixed_uniforms)
cases.append(("normal_f64", lambda x: Q.qm_normal_quantile(x), a64, m64))
zn, zm = pair(np.float64, I.normals)
cases.append(("student_f64", lambda x: Q.qm_recycle_normal_to_t(x, 5.0, 16, 4.6506), zn, zm))
cases.append(("student_moments_t", lambda x: Q.qm_recycle_normal_to_t_moments(x, 5.0, 16, 4.6506)[0], zn, zm))
lv, lm = pair(np.float32, I.laplace)
cases.append(("exp2n_f32", lambda x: Q.qm_recycle_exp_to_normal(x), lv, lm))
tab = Q.qm_exp_target_table(Q.HYPERBOLIC, [1.0, 0.5, 1.0])
hv, hm = pair(np.float64, I.laplace)
cases.append(("rode_f64", lambda x: Q.qm_recycle_exp_to_hyperbolic(x, tab), hv, hm))
bad = 0
for name, fn, xa, xm in cases:
    ref = fn(xm)
    nbad = 0
    for _ in range(reps):
        g = fn(xa)
        if not (torch.equal(g.nan_to_num(), ref.nan_to_num()) and torch.equal(g.isnan(), ref.isnan())):
            nbad += 1
    bad += nbad
    print(name, "mismatching runs:", nbad, "of", reps, flush=True)
print("stress done, total mismatches", bad)
