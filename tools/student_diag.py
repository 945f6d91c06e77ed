"""Worst-ulp inputs of the Student map for one (nu, K, zstar) (diagnostic):
python tools/student_diag.py nu K zstar"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle as O  # noqa: E402
import paper_0901_0638_b200 as Q  # noqa: E402
from _parity import ulp_errors  # noqa: E402
from synth import inputs as I  # noqa: E402

nu, K, zs = float(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
z = np.concatenate([np.linspace(-12.0, 12.0, 12001), I.normals(20000, dtype=np.float64)])
g = Q.qm_recycle_normal_to_t(torch.from_numpy(z).cuda(), nu, K, zs).cpu().numpy()
ref = O.student_map(z, nu, K, zs)
e = ulp_errors(g, ref, np.float64)
idx = np.argsort(-e)[:12]
print(os.environ.get("QM_STUDENT_KC", "kc=default"), "max", e.max())
for i in idx:
    print(f"  z={z[i]:+.6f} |z|>=z*={abs(z[i]) >= zs} ulp={e[i]:.3f} got={g[i]:.17g} ref={float(ref[i]):.17g}")
