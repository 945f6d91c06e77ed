"""Time named hot-path calls with CUDA events (A/B and quick checks; not the bench):
python tools/time_variants.py name1 name2 ...  -> one JSON line per name"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from prof_kernel import make  # noqa: E402

for name in sys.argv[1:]:
    fn, n = make(name)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            fn()
        b.record()
        torch.cuda.synchronize()
        best.append(a.elapsed_time(b) / 10)
    best.sort()
    print(json.dumps({"name": name, "ms_median": best[2], "ms_min": best[0], "gsamples_s": n / best[2] / 1e6}),
          flush=True)
    del fn
    torch.cuda.empty_cache()
