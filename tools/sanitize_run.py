"""Small runs of every TMA-pipeline kernel for compute-sanitizer (memcheck / synccheck / racecheck)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0901_0638_b200 as Q  # noqa: E402
from synth import inputs as I  # noqa: E402

n = (1 << 23) + 37
u = torch.from_numpy(I.mixed_uniforms(n, dtype=np.float32)).cuda()
Q.qm_normal_quantile(u)
Q.qm_normal_quantile(u, alg=Q.TWO_REGION)
Q.qm_recycle_exp_to_normal(torch.from_numpy(I.laplace(n, dtype=np.float32)).cuda())
u64 = torch.from_numpy(I.mixed_uniforms(n, dtype=np.float64)).cuda()
Q.qm_normal_quantile(u64)
u64[::97] = 1e-300                                                      # off the grid: d13_full (out of line)
Q.qm_normal_quantile(u64)
Q.qm_normal_quantile(u64[1:])
Q.qm_recycle_exp_to_normal(torch.linspace(-745, 745, n, dtype=torch.float64, device="cuda"))
zn = torch.from_numpy(I.normals(n, dtype=np.float64)).cuda()
Q.qm_recycle_normal_to_t(zn, 5.0, 16, 4.6506)
tab = Q.qm_exp_target_table(Q.HYPERBOLIC, [1.0, 0.5, 1.0])
v = torch.from_numpy(I.laplace(n, dtype=np.float64)).cuda()
Q.qm_recycle_exp_to_hyperbolic(v, tab)
Q.qm_exp_target_philox(1 << 20, tab, 1, 0)
Q.qm_recycle_exp_to_hyperbolic(v[1:], tab)                              # misaligned: the LDG kernel
tr = Q.qm_exp_target_table(Q.VG, [2.7, 1.0, 0.5])                       # real lambda: graded centre
Q.qm_recycle_exp_to_vg(v, tr)
ts = Q.qm_normal_target_table(Q.STUDENT, [3.0])                         # §3.6: odd map, log tail
zs = zn.clone()
zs[:8] = torch.tensor([0.0, -0.0, float("inf"), -float("inf"), float("nan"), 12.0, -30.0, 45.0], dtype=torch.float64)
Q.qm_recycle_normal_to_t_rode(zs, ts)
Q.qm_recycle_normal_to_t_rode(zs[1:], ts)
Q.qm_recycle_normal_to_t_rode(zs.float(), ts)
Q.qm_recycle_normal_to_t_moments(zn, 5.0, 16, 4.6506)
Q.qm_mc_european_call(1 << 22, 1, 0, 100.0, 0.05, 0.2, 1.0, list(np.linspace(50, 150, 17)))
torch.cuda.synchronize()
print("sanitize run ok")
