"""Per-launch time series of one hot-path call after a rest (experiment helper:
where, within a run of back-to-back launches, does the rate fall, and with
which clock / power / throttle reason?).  For each window length L: 1 s idle,
then L launches with a CUDA event between every two, NVML polled every ~1 ms.

    python tools/window_curve.py [name=stream_f32] [L1,L2,...]   -> JSON lines
"""
import json
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from prof_kernel import make  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "stream_f32"
lens = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "10,20,50,100,200,400").split(",")]
fn, n = make(name)
import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
samples, stop = [], threading.Event()


def poll():
    while not stop.is_set():
        try:
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1e3, int(r)))
        time.sleep(0.001)


th = threading.Thread(target=poll, daemon=True)
th.start()
for _ in range(3):
    fn()
torch.cuda.synchronize()
s = torch.cuda.current_stream()
for L in lens:
    time.sleep(1.0)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(L + 1)]
    t0 = time.perf_counter()
    ev[0].record(s)
    for i in range(L):
        fn()
        ev[i + 1].record(s)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(L)]
    win = [x for x in samples if t0 <= x[0] <= t1]
    rate = [n / ms / 1e6 for ms in per]
    q = max(1, L // 10)
    print(json.dumps({"name": name, "L": L, "window_gsamples_s": n * L / sum(per) / 1e6,
                      "first_decile": sum(rate[:q]) / q, "last_decile": sum(rate[-q:]) / q,
                      "rate_by_decile": [round(sum(rate[i:i + q]) / len(rate[i:i + q]), 1) for i in range(0, L, q)],
                      "sm_mhz": sorted(x[1] for x in win)[len(win) // 2] if win else None,
                      "sm_mhz_min": min(x[1] for x in win) if win else None,
                      "mem_mhz": sorted(x[2] for x in win)[len(win) // 2] if win else None,
                      "power_w_max": max(x[3] for x in win) if win else None,
                      "reasons": sorted({x[4] for x in win})}), flush=True)
stop.set()
th.join()
