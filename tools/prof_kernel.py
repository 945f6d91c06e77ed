"""Launch one hot-path kernel a few times (for ncu).  python tools/prof_kernel.py <name> [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0901_0638_b200 as Q  # noqa: E402

SEED = 0x5EEDC0FFEE123457


def make(name):
    """(fn, samples per call) of the named hot-path call, inputs resident on the device"""
    n = 1 << 28
    if name in ("stream_f32", "stream_f32_two"):
        u = Q.qm_philox_uniform(n, SEED, 0)
        z = torch.empty_like(u)
        alg = Q.TWO_REGION if name == "stream_f32_two" else Q.BREAKLESS
        fn = lambda: Q.qm_normal_quantile(u, out=z, alg=alg)
    elif name in ("stream_f64", "stream_f64_1212"):
        u = Q.qm_philox_uniform(n, SEED, 0, dtype=torch.float64)
        z = torch.empty_like(u)
        alg = Q.BREAKLESS1212 if name == "stream_f64_1212" else Q.BREAKLESS
        fn = lambda: Q.qm_normal_quantile(u, out=z, alg=alg)
    elif name == "fused_f32":
        z = torch.empty(1 << 32, dtype=torch.float32, device="cuda")
        fn = lambda: Q.qm_normal_philox(1 << 32, SEED, 0, out=z)
    elif name == "fused_f64":
        z = torch.empty(1 << 31, dtype=torch.float64, device="cuda")
        fn = lambda: Q.qm_normal_philox(1 << 31, SEED, 0, dtype=torch.float64, out=z)
    elif name.startswith("config1_") or name.startswith("plain_config1_"):
        import numpy as np
        from synth import inputs as I
        alg = {"breakless": Q.BREAKLESS, "as241": Q.AS241, "acklam": Q.ACKLAM, "refined": Q.ACKLAM_REFINED,
               "moro": Q.MORO, "breakless77": Q.BREAKLESS77}[name.split("config1_")[1]]
        u = torch.from_numpy(I.tail_stratified(1 << 20, dtype=np.float64)).cuda()
        z = torch.empty_like(u)
        call = Q.qm_normal_quantile_plain if name.startswith("plain_") else Q.qm_normal_quantile
        fn = lambda: call(u, out=z, alg=alg)
    elif name == "exp2n_f32":
        import numpy as np
        from synth import inputs as I
        v = torch.from_numpy(I.laplace(n, dtype=np.float32)).cuda()
        z = torch.empty_like(v)
        fn = lambda: Q.qm_recycle_exp_to_normal(v, out=z)
    elif name == "moments":
        x = Q.qm_normal_philox(1 << 30, SEED, 0, dtype=torch.float64)
        rows = torch.empty(4 * Q.qm_moment_row_count(1 << 30), dtype=torch.float64, device="cuda")
        fn = lambda: Q.qm_moments(x, 4, rows=rows)
    elif name == "mc":
        import numpy as np
        ks = list(np.linspace(50, 150, 17))
        rows = torch.empty((Q.qm_mc_row_count(1 << 32), 34), dtype=torch.float64, device="cuda")
        fn = lambda: Q.qm_mc_european_call(1 << 32, SEED, 0, 100.0, 0.05, 0.2, 1.0, ks, out=rows)
    elif name == "student_moments":
        zn = Q.qm_normal_philox(1 << 30, SEED, 0, dtype=torch.float64)
        t = torch.empty_like(zn)
        rows = torch.empty((Q.qm_moment_row_count(1 << 30), 4), dtype=torch.float64, device="cuda")
        fn = lambda: Q.qm_recycle_normal_to_t_moments(zn, 5.0, 16, 4.6506, out=t, rows=rows)
    elif name == "student":
        zn = Q.qm_normal_philox(1 << 30, SEED, 0, dtype=torch.float64)
        t = torch.empty_like(zn)
        fn = lambda: Q.qm_recycle_normal_to_t(zn, 4.0, 10, 3.93473, out=t)
    elif name in ("student_nu3", "student_nu10", "student_nu3_notail"):
        zn = Q.qm_normal_philox(1 << 30, SEED, 0, dtype=torch.float64)
        t = torch.empty_like(zn)
        nu = 10.0 if name == "student_nu10" else 3.0
        zs = 50.0 if name == "student_nu3_notail" else 0.0     # A/B: the series alone (caller z* beyond every sample)
        fn = lambda: Q.qm_recycle_normal_to_t(zn, nu, 16, zs, out=t)
    elif name in ("student_rode", "student_k16"):
        zn = Q.qm_normal_philox(1 << 30, SEED, 0, dtype=torch.float64)
        t = torch.empty_like(zn)
        if name == "student_rode":
            tab = Q.qm_normal_target_table(Q.STUDENT, [5.0])
            fn = lambda: Q.qm_recycle_normal_to_t_rode(zn, tab, out=t)
        else:
            fn = lambda: Q.qm_recycle_normal_to_t(zn, 5.0, 16, out=t)
    elif name == "rode_hyp_f64_ldg":       # misaligned view: the LDG kernel (no TMA input pipeline)
        import numpy as np
        from synth import inputs as I
        tab = Q.qm_exp_target_table(Q.HYPERBOLIC, [1.0, 0.5, 1.0])
        v = torch.from_numpy(I.laplace(n + 1, dtype=np.float64)).cuda()[1:]
        x = torch.empty(n + 1, dtype=torch.float64, device="cuda")[1:]
        fn = lambda: Q.qm_recycle_exp_to_hyperbolic(v, tab, out=x)
    elif name in ("rode_hyp_f64", "rode_philox_f32", "rode_vg_real_f64"):
        if name == "rode_vg_real_f64":
            tab = Q.qm_exp_target_table(Q.VG, [2.7, 1.0, 0.5])
        else:
            tab = Q.qm_exp_target_table(Q.HYPERBOLIC, [1.0, 0.5, 1.0])
        if name != "rode_philox_f32":
            # the table's own exponential base from Philox uniforms
            v = Q.qm_exp_base_quantile(Q.qm_philox_uniform(n, SEED, 0, dtype=torch.float64), tab)
            x = torch.empty_like(v)
            call = Q.qm_recycle_exp_to_vg if name == "rode_vg_real_f64" else Q.qm_recycle_exp_to_hyperbolic
            fn = lambda: call(v, tab, out=x)
        else:
            x = torch.empty(n, dtype=torch.float32, device="cuda")
            fn = lambda: Q.qm_exp_target_philox(n, tab, SEED, 0, dtype=torch.float32, out=x)
    else:
        raise SystemExit(f"unknown {name}")
    return fn, _count(name, n)


def _count(name, n):
    big = {"fused_f32": 1 << 32, "fused_f64": 1 << 31, "moments": 1 << 30, "mc": 1 << 32, "student_moments": 1 << 30,
           "student": 1 << 30, "student_rode": 1 << 30, "student_k16": 1 << 30, "student_nu3": 1 << 30,
           "student_nu10": 1 << 30, "student_nu3_notail": 1 << 30}
    if name.startswith("config1_") or name.startswith("plain_config1_"):
        return 1 << 20
    return big.get(name, n)


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "stream_f32"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    fn, _ = make(name)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print("done", name)
