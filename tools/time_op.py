"""Time one hot-path call with CUDA events (A/B helper):  python tools/time_op.py <name> [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0901_0638_b200 as Q  # noqa: E402

SEED = 0x5EEDC0FFEE123457
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
if name == "fused_f32":
    n = 1 << 32
    z = torch.empty(n, dtype=torch.float32, device="cuda")
    fn = lambda: Q.qm_normal_philox(n, SEED, 0, out=z)
elif name.startswith("stream_f32"):
    n = 1 << 28
    alg = {"stream_f32": Q.BREAKLESS, "stream_f32_two": Q.TWO_REGION, "stream_f32_88": Q.BREAKLESS88}[name]
    u = Q.qm_philox_uniform(n, SEED, 0)
    z = torch.empty_like(u)
    fn = lambda: Q.qm_normal_quantile(u, out=z, alg=alg)
elif name == "stream_f64":
    n = 1 << 28
    u = Q.qm_philox_uniform(n, SEED, 0, dtype=torch.float64)
    z = torch.empty_like(u)
    fn = lambda: Q.qm_normal_quantile(u, out=z)
elif name == "fused_f64":
    n = 1 << 31
    z = torch.empty(n, dtype=torch.float64, device="cuda")
    fn = lambda: Q.qm_normal_philox(n, SEED, 0, dtype=torch.float64, out=z)
elif name.startswith("student"):
    n = 1 << 30
    nu, K, zs = {"student4": (4.0, 10, 3.93473), "student5": (5.0, 16, 4.6506), "student3": (3.0, 16, 3.5667),
                 "student10": (10.0, 16, 6.9584)}[name]
    zn = Q.qm_normal_philox(n, SEED, 0, dtype=torch.float64)
    t = torch.empty_like(zn)
    fn = lambda: Q.qm_recycle_normal_to_t(zn, nu, K, zs, out=t)
elif name == "mc":
    import numpy as np
    n = 1 << 34
    ks = list(np.linspace(50, 150, 17))
    rows = torch.empty((Q.qm_mc_row_count(n), 34), dtype=torch.float64, device="cuda")
    fn = lambda: Q.qm_mc_european_call(n, SEED, 0, 100.0, 0.05, 0.2, 1.0, ks, out=rows)
elif name.startswith("rode_hyp"):
    import numpy as np
    from synth import inputs as I
    n = 1 << 28
    tab = Q.qm_exp_target_table(Q.HYPERBOLIC, [1.0, 0.5, 1.0])
    dt = np.float64 if name.endswith("f64") else np.float32
    v = torch.from_numpy(I.laplace(n, dtype=dt)).cuda()
    x = torch.empty_like(v)
    fn = lambda: Q.qm_recycle_exp_to_hyperbolic(v, tab, out=x)
else:
    raise SystemExit("unknown " + name)
for _ in range(3):
    fn()
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(s)
for _ in range(reps):
    fn()
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"{name} {os.environ.get('QM_PHILOX_CFG', '')}{os.environ.get('QM_TL_CFG', '')} {n / ms / 1e6:.1f} Gsamples/s ({ms:.3f} ms)")
