"""The fp32 map's burst rate at 2^20 .. 2^32 (CUDA graphs below ~1 ms, as bench.py's
size_sweep): an A/B helper, e.g. QM_PDL=0 vs 1.   python tools/sweep_quick.py [fused]"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_0901_0638_b200 as Q  # noqa: E402
from bench import SEED, time_steps  # noqa: E402

FUSED = len(sys.argv) > 1 and sys.argv[1] == "fused"
out = {}
for e in ((20, 22, 24, 28, 32) if FUSED else (20, 21, 22, 23, 24, 26, 28, 30, 32)):
    n = 1 << e
    u = torch.empty(n, dtype=torch.float32, device="cuda")
    Q.qm_philox_uniform(n, SEED, 0, out=u)
    z = torch.empty_like(u)
    fn = (lambda: Q.qm_normal_philox(n, SEED, 0, out=z)) if FUSED else (lambda: Q.qm_normal_quantile(u, out=z))
    one = time_steps(fn, 3, 2) / 3
    time.sleep(0.5)
    if one < 1.0:
        reps = max(1, int(8.0 / max(one, 1e-3)) // 5)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                fn()
        ms = time_steps(g.replay, 5, 2) / (5 * reps)
    else:
        k = max(2, int(8.0 / one))
        ms = time_steps(fn, k, 2) / k
    out[f"2^{e}"] = round(n / (ms / 1e3) / 1e9, 1)
    del u, z
    torch.cuda.empty_cache()
print(json.dumps({"pdl": os.environ.get("QM_PDL", "1"), "fused": FUSED, "gsamples_s": out}))
