"""Sustained rate of one hot-path call: W windows of L launches each, every
window timed with CUDA events and the SM clock sampled by NVML in it
(experiment helper: does the rate fall as the GPU warms up?).

    python tools/long_run.py [name=stream_f32] [windows=30] [launches=100]
"""
import os
import statistics
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_0901_0638_b200 as Q  # noqa: E402

SEED = 0x5EEDC0FFEE123457
name = sys.argv[1] if len(sys.argv) > 1 else "stream_f32"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 30
L = int(sys.argv[3]) if len(sys.argv) > 3 else 100
n = 1 << 28
if name == "stream_f32":
    u = Q.qm_philox_uniform(n, SEED, 0)
    z = torch.empty_like(u)
    fn = lambda: Q.qm_normal_quantile(u, out=z)
    bps = 8
elif name == "exp2n_f32":
    u = Q.qm_normal_philox(n, SEED, 0)
    z = torch.empty_like(u)
    fn = lambda: Q.qm_recycle_exp_to_normal(u, out=z)
    bps = 8
elif name == "copy_f32":
    u = torch.empty(n, dtype=torch.float32, device="cuda")
    z = torch.empty_like(u)
    fn = lambda: z.copy_(u)
    bps = 8
elif name == "fused_f32":
    n = 1 << 32
    z = torch.empty(n, dtype=torch.float32, device="cuda")
    fn = lambda: Q.qm_normal_philox(n, SEED, 0, out=z)
    bps = 4
    L = max(1, L // 16)
elif name == "mc":
    import numpy as np
    n = 1 << 34
    ks = list(np.linspace(50, 150, 17))
    rows = torch.empty((Q.qm_mc_row_count(n), 34), dtype=torch.float64, device="cuda")
    fn = lambda: Q.qm_mc_european_call(n, SEED, 0, 100.0, 0.05, 0.2, 1.0, ks, out=rows)
    bps = 0
    L = max(1, L // 64)
else:
    raise SystemExit("unknown " + name)

import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
clk, stop = [], threading.Event()


def poll():
    while not stop.is_set():
        clk.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetPowerUsage(h) / 1e3))
        time.sleep(0.002)


th = threading.Thread(target=poll, daemon=True)
th.start()
for _ in range(5):
    fn()
torch.cuda.synchronize()
s = torch.cuda.current_stream()
rows = []
for w in range(W):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(L):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ms = e0.elapsed_time(e1) / L
    cs = [c for t, c, p in clk if t0 <= t <= t1]
    ps = [p for t, c, p in clk if t0 <= t <= t1]
    rows.append((w, n / ms / 1e6, bps * n / ms / 1e6, statistics.median(cs) if cs else None, max(ps) if ps else None))
stop.set()
th.join()
print(f"# {name}: window, Gsamples/s, GB/s, median SM MHz, max W")
for r in rows:
    print(f"{name} {r[0]:3d} {r[1]:8.1f} {r[2]:8.1f} {r[3]} {r[4]}")
