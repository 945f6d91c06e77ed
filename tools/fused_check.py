"""Fused fp32 sampler (and the Monte-Carlo sums) of the current build (QM_LIB_PATH):
fused == philox_uniform + quantile bitwise, and max ulp vs the oracle on 2^22 samples."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle as O  # noqa: E402
import paper_0901_0638_b200 as Q  # noqa: E402
from _parity import summary, ulp_errors  # noqa: E402

n = (1 << 22) + 5
z = Q.qm_normal_philox(n, 77, 3)
u = Q.qm_philox_uniform(n, 77, 3)
z2 = Q.qm_normal_quantile(u)
ref = O.normal_breakless(u.cpu().numpy().astype(np.float64), O.C55, 32)
print(os.environ.get("QM_LIB_PATH", "default"), "fused==unfused", bool(torch.equal(z, z2)),
      "fused", summary(ulp_errors(z.cpu().numpy(), ref, np.float32)),
      "unfused", summary(ulp_errors(z2.cpu().numpy(), ref, np.float32)))
