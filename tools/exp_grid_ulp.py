"""Max ulp of the fp32 breakless map over the whole fp32 odd grid (2^24 values)
for the current library build (QM_LIB_PATH) and stream path (experiment helper)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle as O  # noqa: E402
import paper_0901_0638_b200 as Q  # noqa: E402
from _parity import summary, ulp_errors  # noqa: E402

k = np.arange(1 << 23, dtype=np.float64)
lo = np.ldexp(2 * k + 1, -24).astype(np.float32)
u = np.concatenate([lo, (1 - lo.astype(np.float64)).astype(np.float32)])
g = Q.qm_normal_quantile(torch.from_numpy(u).cuda()).cpu().numpy()
ref = O.normal_breakless(u.astype(np.float64), O.C55, 32)
print(os.environ.get("QM_LIB_PATH", "default"), summary(ulp_errors(g, ref, np.float32)))
