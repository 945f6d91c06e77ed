"""e2e host-buffer pipeline A/B: python tools/ab_e2e.py  (env QM_HOST_STREAMS / QM_HOST_CHUNK_LOG2)"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0901_0638_b200 as Q  # noqa: E402

n = 1 << 28
u = Q.qm_philox_uniform(n, 1, 0)
uh = torch.empty(n, dtype=torch.float32, pin_memory=True)
uh.copy_(u.cpu())
zh = torch.empty(n, dtype=torch.float32, pin_memory=True)
Q.qm_normal_quantile_host(uh, out=zh)
t0 = time.perf_counter()
for _ in range(10):
    Q.qm_normal_quantile_host(uh, out=zh)
dt = (time.perf_counter() - t0) / 10
print(os.environ.get("QM_HOST_STREAMS"), os.environ.get("QM_HOST_CHUNK_LOG2"), round(n / dt / 1e9, 2), "Gsamples/s")
