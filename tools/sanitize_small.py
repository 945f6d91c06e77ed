"""Kernels outside the TMA ring (LDG maps, staged RODE tables, reductions) for racecheck."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0901_0638_b200 as Q  # noqa: E402
from synth import inputs as I  # noqa: E402

n = (1 << 20) + 37
Q.qm_normal_quantile(torch.from_numpy(I.mixed_uniforms(n, dtype=np.float32)).cuda())
Q.qm_normal_quantile(torch.from_numpy(I.mixed_uniforms(n, dtype=np.float64)).cuda(), alg=Q.AS241)
zn = torch.from_numpy(I.normals(n, dtype=np.float64)).cuda()
t = Q.qm_recycle_normal_to_t(zn, 5.0, 16, 4.6506)
rows = torch.empty(4 * Q.qm_moment_row_count(n), dtype=torch.float64, device="cuda")
Q.qm_moments(t, 4, rows=rows)
tab = Q.qm_exp_target_table(Q.HYPERBOLIC, [1.0, 0.5, 1.0])
Q.qm_recycle_exp_to_hyperbolic(torch.from_numpy(I.laplace(n, dtype=np.float64)).cuda(), tab)
Q.qm_exp_target_philox(1 << 20, tab, 1, 0)
Q.qm_mc_european_call(1 << 21, 1, 0, 100.0, 0.05, 0.2, 1.0, list(np.linspace(50, 150, 17)))
Q.qm_normal_philox(1 << 20, 1, 0)
torch.cuda.synchronize()
print("sanitize small ok")
