"""fp32/fp64 streaming map at small sizes (CUDA graphs of 50 launches): A/B helper."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0901_0638_b200 as Q  # noqa: E402

SEED = 0x5EEDC0FFEE123457
for dt in (torch.float32, torch.float64):
    for e in (20, 22, 23, 24, 26):
        n = 1 << e
        u = Q.qm_philox_uniform(n, SEED, 0, dtype=dt)
        z = torch.empty_like(u)
        Q.qm_normal_quantile(u, out=z)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(50):
                Q.qm_normal_quantile(u, out=z)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 250
        print(os.environ.get("QM_STREAM_PATH", "tl"), dt, f"2^{e}", round(n / ms / 1e6, 1), "Gsamples/s")
