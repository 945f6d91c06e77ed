"""Max ulp of the Student map on tail samples (|z| >= z*) vs the oracle (A/B helper)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle as O  # noqa: E402
import paper_0901_0638_b200 as Q  # noqa: E402
from _parity import ulp_errors  # noqa: E402

rng = np.random.default_rng(3)
for nu, K, zs in [(3.0, 16, 3.5667), (4.0, 10, 3.93473), (5.0, 16, 4.6506), (10.0, 16, 6.9584), (20.0, 16, 9.0)]:
    z = np.concatenate([zs + rng.exponential(1.0, 200000), -(zs + rng.exponential(3.0, 100000)), np.linspace(zs, 38, 20001)])
    g = Q.qm_recycle_normal_to_t(torch.from_numpy(z).cuda(), nu, K, zs).cpu().numpy()
    e = ulp_errors(g, O.student_map(z, nu, K, zs), np.float64)
    print(os.environ.get("QM_LIB_PATH", "default"), nu, "tail max ulp", round(float(e.max()), 3), "p99.9", round(float(np.quantile(e, 0.999)), 3))
