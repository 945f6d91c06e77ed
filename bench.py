#!/usr/bin/env python
"""Benchmark of the bulk inverse-CDF sampling hot path on B200 (one JSON line).

Default workload (N=1): BASELINE.json configs[1] -- 2^28 fp32 odd-grid uniforms
resident in HBM -> branch-free normal quantile (App C) -> 2^28 fp32
normal samples in HBM.  One step = one launch over the whole batch.  Inputs
(1 GiB) exceed the 126 MB L2, so no flush is needed between steps.
Multi-GPU (torchrun): weak scaling, every rank maps its own 2^28 uniforms
(Philox counter offset rank * 2^26); no collective on the data path; the
elapsed time is the max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gsamples/s per GPU and at 8 GPUs (fp32/fp64); % of HBM BW or FP pipe peak"
UNIT = "Gsamples/s"
SEED = 0x5EEDC0FFEE123457
N_MAIN = 1 << 28
WORKLOAD = ("configs[1]: 2^28 fp32 uniforms streamed from HBM -> branch-free normal quantile "
            "(App C (5,5), QM_BREAKLESS) -> fp32 normal samples in HBM")


# ----------------------------------------------------------------- helpers
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            with open(p) as f:
                d = json.load(f)
            return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)),
                    "source": "MEASURED_PEAKS.json (measured copy bandwidth, burst)"}
        except (OSError, ValueError, KeyError, TypeError):
            pass
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback 6.65 TB/s (B200_PROFILING.md)"}


def load_traffic():
    """Per-element DRAM traffic of each kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


class ClockSampler:
    """Polls NVML (SM clock, clock-event reasons) every ~2 ms during a timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
               0x2: "applications_clocks_setting", 0x10: "sync_boost"}

    def __init__(self, index):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self.samples, self.reasons = [], 0
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(get_reasons(self.h))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1),
                "n_samples": len(self.samples)}


def dist_setup(gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------ reference arm
def oracle_rate(n_sample, threads, seed=SEED, chunk=None):
    """Time the oracle (same formula, long double) over a bounded sample on host
    cores: `threads` workers map chunks of the sample (ctypes releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle as O
    from synth import inputs as I
    if chunk is None:                    # every worker gets work, chunks of <= 4 Mi samples
        chunk = max(1 << 14, min(1 << 22, -(-n_sample // (4 * threads))))
    u = I.uniform_grid(n_sample, seed, np.float32)
    bounds = [(i, min(i + chunk, n_sample)) for i in range(0, n_sample, chunk)]
    O.lib()

    def work(b):
        O.normal_breakless(u[b[0]:b[1]].astype(np.float64), O.C55, 32)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, bounds))
    dt = time.perf_counter() - t0
    return n_sample / dt / 1e9, dt


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args):
    world, rank, _ = dist_setup(args.gpus)
    if rank != 0:
        return
    import oracle as O
    O.build()
    threads = os.cpu_count() or 1
    n_step = 1 << 22                     # bounded sample per step (~15-40 ms on 16 threads)
    for _ in range(args.warmup):
        oracle_rate(n_step, threads)
    ts = []
    for _ in range(args.steps):
        _, dt = oracle_rate(n_step, threads)
        ts.append(dt)
    total = sum(ts)
    value = n_step * args.steps / total / 1e9
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "n": N_MAIN, "reference_sample_per_step": n_step},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": f"{n_step} fp32 odd-grid uniforms per step -> same formula (App C, "
                                       f"float-rounded coefficients) in long double, {threads} threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def time_steps(fn, steps, warmup, dist=None):
    import torch
    for _ in range(warmup):
        fn()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    return e0.elapsed_time(e1)


def max_over_ranks(x, dist):
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def variants(Q, torch, peaks, steps=10, warmup=3):
    """Other §8 rows, each timed alone on one GPU (reported beside the headline)."""
    out = {}
    hbm = peaks["hbm_gbs"]

    facts = load_traffic()
    # issue-slot ceiling: 148 SMs x 4 schedulers x 1 warp-instruction / clock
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    issue_peak = sms * 4 * peaks["sm_max_mhz"] / 1e3          # G warp-instructions / s

    def rec(name, fn, n, bytes_per, extra=None, fact=None):
        ms = time_steps(fn, steps, warmup) / steps
        r = {"gsamples_s": n / (ms / 1e3) / 1e9, "ms": ms, "n": n,
             "hbm_gbs": (bytes_per * n / (ms / 1e3) / 1e9) if bytes_per else 0.0}
        r["hbm_frac"] = r["hbm_gbs"] / hbm
        f = facts.get(fact) if fact else None
        if f and f.get("warp_inst_per_elem"):
            # compute-bound rows: warp-instructions per sample (ncu) x samples/s
            # against the issue ceiling (bench measures the rate, ncu the count)
            ach = f["warp_inst_per_elem"] * r["gsamples_s"]
            r["roofline"] = {"bound": "issue", "achieved": ach, "peak": issue_peak,
                             "unit": "G warp-inst/s", "frac": ach / issue_peak,
                             "warp_inst_per_sample": f["warp_inst_per_elem"], "source": f.get("source")}
        if extra:
            r.update(extra)
        out[name] = r

    n = 1 << 28
    u64 = torch.empty(n, dtype=torch.float64, device="cuda")
    Q.qm_philox_uniform(n, SEED, 0, dtype=torch.float64, out=u64)
    z64 = torch.empty_like(u64)
    rec("stream_f64_D13_2^28", lambda: Q.qm_normal_quantile(u64, out=z64), n, 16, fact="stream_f64")
    # rows f3/f4: (12,12) fp64 on [0, 37], (8,8) fp32 on [0, 74], two-region fp32
    rec("stream_f64_F1212_2^28", lambda: Q.qm_normal_quantile(u64, out=z64, alg=Q.BREAKLESS1212), n, 16)
    u32 = torch.empty(n, dtype=torch.float32, device="cuda")
    Q.qm_philox_uniform(n, SEED, 0, out=u32)
    z32 = torch.empty_like(u32)
    rec("stream_f32_F88_2^28", lambda: Q.qm_normal_quantile(u32, out=z32, alg=Q.BREAKLESS88), n, 8)
    rec("stream_f32_two_region_2^28", lambda: Q.qm_normal_quantile(u32, out=z32, alg=Q.TWO_REGION), n, 8)
    # row f2 (deep-tail composite; its fast path is App C) and row a4 (antithetic pairs:
    # 4 B in, 8 B out per uniform; samples counted = outputs)
    rec("stream_f32_tail_composite_2^28", lambda: Q.qm_normal_quantile(u32, out=z32, alg=Q.BREAKLESS_TAIL), n, 8)
    za = torch.empty(2 * n, dtype=torch.float32, device="cuda")
    rec("antithetic_f32_2^28_uniforms", lambda: Q.qm_normal_antithetic(u32, out=za), 2 * n, 6)
    del u32, z32, za
    zf = torch.empty(1 << 32, dtype=torch.float32, device="cuda")
    rec("philox_fused_f32_2^32", lambda: Q.qm_normal_philox(1 << 32, SEED, 0, out=zf), 1 << 32, 4, fact="fused_f32")
    del zf
    zd = torch.empty(1 << 31, dtype=torch.float64, device="cuda")
    rec("philox_fused_f64_2^31", lambda: Q.qm_normal_philox(1 << 31, SEED, 0, dtype=torch.float64, out=zd),
        1 << 31, 8, fact="fused_f64")
    del zd
    # config 4: Student-t recycling of 2^30 fp64 normals (untimed producer: the fused kernel)
    zn = Q.qm_normal_philox(1 << 30, SEED, 0, dtype=torch.float64)
    tt = torch.empty_like(zn)
    for nu, K, zs in [(4.0, 10, 3.93473), (3.0, 16, 3.5667), (5.0, 16, 4.6506), (10.0, 16, 6.9584)]:
        rec(f"student_f64_nu{int(nu)}_K{K}_2^30",
            lambda nu=nu, K=K, zs=zs: Q.qm_recycle_normal_to_t(zn, nu, K, zs, out=tt), 1 << 30, 16,
            fact="student" if nu == 4.0 else None)
    ws = torch.empty(4 * Q.qm_moment_row_count(1 << 30), dtype=torch.float64, device="cuda")
    rec("moments_f64_2^30", lambda: Q.qm_moments(tt, 4, rows=ws), 1 << 30, 8)
    del zn, tt
    # config 5 building block: Laplace -> normal
    from synth import inputs as I
    v = torch.from_numpy(I.laplace(n, dtype=np.float32)).cuda()
    zo = torch.empty_like(v)
    rec("exp_to_normal_f32_2^28", lambda: Q.qm_recycle_exp_to_normal(v, out=zo), n, 8)
    del v, zo
    # row f1: exponential base -> hyperbolic / VG through the RODE table (fp64 and fp32)
    tab_h = Q.qm_exp_target_table(Q.HYPERBOLIC, [1.0, 0.5, 1.0])
    tab_v = Q.qm_exp_target_table(Q.VG, [2.0, 1.0, 0.5])
    v64 = torch.from_numpy(I.laplace(n, dtype=np.float64)).cuda()
    x64 = torch.empty_like(v64)
    rec("exp_to_hyperbolic_f64_2^28", lambda: Q.qm_recycle_exp_to_hyperbolic(v64, tab_h, out=x64), n, 16)
    rec("exp_to_vg_f64_2^28", lambda: Q.qm_recycle_exp_to_vg(v64, tab_v, out=x64), n, 16)
    del v64, x64
    xf = torch.empty(n, dtype=torch.float32, device="cuda")
    rec("hyperbolic_philox_f32_2^28", lambda: Q.qm_exp_target_philox(n, tab_h, SEED, 0, dtype=torch.float32, out=xf),
        n, 4)
    del xf
    # config 5: 2^34-sample exponential-base Monte-Carlo call sweep, 17 strikes (Philox-fused)
    strikes = list(np.linspace(50, 150, 17))
    rows = torch.empty((Q.qm_mc_row_count(1 << 34), 34), dtype=torch.float64, device="cuda")
    rec("mc_call_sweep_f32_2^34_17K",
        lambda: Q.qm_mc_european_call(1 << 34, SEED, 0, 100.0, 0.05, 0.2, 1.0, strikes, out=rows), 1 << 34, 0,
        fact="mc")
    del rows
    # config 1: 2^20 fp64, breakless vs branching baselines (tail-stratified input)
    u1 = torch.from_numpy(I.tail_stratified(1 << 20, dtype=np.float64)).cuda()
    z1 = torch.empty_like(u1)
    for name, alg in [("breakless_D13", Q.BREAKLESS), ("as241", Q.AS241), ("acklam", Q.ACKLAM),
                      ("acklam_refined", Q.ACKLAM_REFINED), ("moro", Q.MORO), ("breakless77", Q.BREAKLESS77)]:
        # ~25 us of work per launch: time a CUDA graph of 100 launches
        graph = torch.cuda.CUDAGraph()
        Q.qm_normal_quantile(u1, out=z1, alg=alg)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph):
            for _ in range(100):
                Q.qm_normal_quantile(u1, out=z1, alg=alg)
        rec(f"config1_f64_2^20_{name}", graph.replay, 100 << 20, 16,
            extra={"timing": "CUDA graph of 100 launches per step"})
    del u64, z64
    # the paper's Table 3 speed-ups of the breakless App D kernel (context)
    g = lambda k: out[f"config1_f64_2^20_{k}"]["gsamples_s"]
    out["config1_speedups"] = {
        "breakless_vs_as241": g("breakless_D13") / g("as241"),
        "breakless_vs_acklam_refined": g("breakless_D13") / g("acklam_refined"),
        "breakless_vs_acklam_l1": g("breakless_D13") / g("acklam"),
        "paper_table3_vs_as241": {"Quadro FX 4800": 1.44, "GTX 285": 1.45, "GTX 480": 1.41},
        "paper_table3_vs_acklam_lea": {"Quadro FX 4800": 2.69, "GTX 285": 2.71, "GTX 480": 2.61},
        "note": "context only: the paper's timings are for an unstated N on sm_1.x/2.0 hardware (P:647)"}
    out["size_sweep"] = size_sweep(Q, torch)
    return out


def size_sweep(Q, torch):
    """Gsamples/s over 2^20 .. 2^34 samples (north star), 1 GPU: the fp32 streaming
    map (inputs resident in HBM) and the Philox-fused fp32 sampler.  Sizes whose
    launch is shorter than ~1 ms are timed as CUDA graphs of 50 launches."""
    res = {"stream_f32": {}, "fused_f32": {}}

    def timed(fn, n, tag):
        one = time_steps(fn, 3, 2) / 3
        if one < 1.0:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(50):
                    fn()
            ms = time_steps(g.replay, 5, 2) / (5 * 50)
        else:
            ms = time_steps(fn, 5, 2) / 5
        res[tag][f"2^{n.bit_length() - 1}"] = round(n / (ms / 1e3) / 1e9, 2)

    for e in (20, 22, 24, 26, 28, 30, 32):
        n = 1 << e
        u = torch.empty(n, dtype=torch.float32, device="cuda")
        Q.qm_philox_uniform(n, SEED, 0, out=u)
        z = torch.empty_like(u)
        timed(lambda: Q.qm_normal_quantile(u, out=z), n, "stream_f32")
        del u, z
    for e in (20, 24, 28, 32, 34):
        n = 1 << e
        z = torch.empty(n, dtype=torch.float32, device="cuda")
        timed(lambda: Q.qm_normal_philox(n, SEED, 0, out=z), n, "fused_f32")
        del z
    torch.cuda.empty_cache()
    return res


def dist_variants(torch, dist, rank, world, steps=5, warmup=2):
    """Config 4 (2^30 fp64 normals -> Student-t nu=5 -> moments) and config 5
    (2^34-sample exponential-base call sweep) over all ranks, each step ending
    with the NCCL all-reduce of the row matrix and the fixed-order reduction;
    time = max over ranks.  Results are bit-identical for any number of GPUs."""
    from paper_0901_0638_b200 import shard as S
    out = {}
    strikes = list(np.linspace(50, 150, 17))

    def run(name, fn, n_total, collective="all_reduce(SUM) of the fixed-chunk row matrix (NCCL)"):
        ms = max_over_ranks(time_steps(fn, steps, warmup, dist), dist) / steps
        r = fn()
        out[name] = {"gsamples_s": n_total / (ms / 1e3) / 1e9, "ms": ms, "n": n_total, "n_gpus": world,
                     "scaling": "strong", "collective": collective,
                     "result": [float(x) for x in (r[0] if isinstance(r, tuple) else r).flatten()[:4].cpu()]}

    # config 3: Philox-fused 2^32 fp32 normals, fixed total split by counter ranges
    # (no collective: every rank writes its own slice; bit-identical to one GPU)
    nloc = (1 << 32) // world
    zloc = torch.empty(nloc, dtype=torch.float32, device="cuda")
    import paper_0901_0638_b200 as Q
    run("dist_fused_f32_2^32", lambda: (Q.qm_normal_philox(nloc, SEED, rank * (nloc // 4), out=zloc)[:4],), 1 << 32,
        collective="none (counter-range shards)")
    del zloc
    run("dist_student_moments_f64_nu5_2^30",
        lambda: S.student_moments(1 << 30, 5.0, 16, 4.6506, SEED, rank, world)[0], 1 << 30)
    run("dist_mc_call_sweep_2^34_17K",
        lambda: S.mc_call_sweep(1 << 34, SEED, 100.0, 0.05, 0.2, 1.0, strikes, rank, world), 1 << 34)
    return out


def run_ours(args):
    import torch
    world, rank, local = dist_setup(args.gpus)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # QM_DIST_BACKEND=gloo: a validation mode for boxes with fewer GPUs than
        # ranks (ranks share devices; timings meaningless); the product is NCCL
        backend = os.environ.get("QM_DIST_BACKEND", "nccl")
        torch.cuda.set_device(local % torch.cuda.device_count())
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    import paper_0901_0638_b200 as Q
    from paper_0901_0638_b200 import _lib
    _lib.load()
    peaks = load_peaks()
    n = N_MAIN

    # untimed producer: this rank's uniforms (Philox stream, counter offset rank * n/4)
    u = torch.empty(n, dtype=torch.float32, device="cuda")
    Q.qm_philox_uniform(n, SEED, rank * (n // 4), out=u)
    z = torch.empty_like(u)
    step = lambda: Q.qm_normal_quantile(u, out=z)

    sampler = ClockSampler(local)
    with sampler:
        ms = time_steps(step, args.steps, args.warmup, dist)
    ms = max_over_ranks(ms, dist)
    ms_step = ms / args.steps
    value = world * n * args.steps / (ms / 1e3) / 1e9

    # roofline of the (only) kernel of the step: 8 algorithmic bytes per sample
    achieved = 8.0 * n / (ms_step / 1e3) / 1e9
    fact = load_traffic().get("stream_f32", {})
    traffic = fact.get("dram_bytes_per_elem")
    roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "traffic": (traffic * n if traffic else None),
            "kernel": "qm::k_normal_f32_tl<ALG_BREAKLESS, TlCfgL> (TMA bulk loads in, streaming stores out)",
            "algorithmic_bytes_per_launch": 8 * n, "peak_source": peaks["source"],
            "traffic_source": fact.get("source")}

    # e2e through the public C-ABI host entry point: pinned host in, pinned host out
    uh = torch.empty(n, dtype=torch.float32, pin_memory=True)
    uh.copy_(u.cpu())
    zh = torch.empty(n, dtype=torch.float32, pin_memory=True)
    e2e_steps = max(1, min(args.steps, 10))
    Q.qm_normal_quantile_host(uh, out=zh)
    if dist is not None:
        dist.barrier()
    with ClockSampler(local) as s2:
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            Q.qm_normal_quantile_host(uh, out=zh)
        t1 = time.perf_counter()
    e2e_s = max_over_ranks(t1 - t0, dist)
    e2e = {"value": world * n * e2e_steps / e2e_s / 1e9, "unit": UNIT, "h2d_bytes_per_step": 4 * n,
           "d2h_bytes_per_step": 4 * n, "steps": e2e_steps, "api": "qm_normal_quantile_host",
           "gpu_launches": e2e_steps * ((n + (1 << 24) - 1) >> 24), "clocks": s2.summary()}
    assert torch.equal(zh, z.cpu())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        # bounded sample sized for ~10-30 s of CPU work (the oracle runs ~20 M samples/s/thread)
        nsamp = 1 << 28 if threads >= 8 else 1 << 26
        rate, dt = oracle_rate(nsamp, threads)
        rate1, dt1 = oracle_rate(1 << 24, 1)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"2^{nsamp.bit_length() - 1} fp32 odd-grid uniforms (the full configs[1] batch when "
                         f"2^28) -> the same formula (App C, float-rounded coefficients) in long double, "
                         f"{dt:.1f} s wall on {threads} threads",
               "single_thread_value": rate1, "single_thread_sample": f"2^24 samples, {dt1:.1f} s",
               "cpu_model": cpu_model()}

    # configs 4 and 5 across the ranks: fixed global work split by Philox counter
    # ranges, one NCCL all-reduce of the fixed-chunk sum rows (strong scaling)
    dvar = None
    if not args.no_variants:
        dvar = dist_variants(torch, dist, rank, world)

    var = None
    if rank == 0 and not args.no_variants:
        var = variants(Q, torch, peaks)
        var.update(dvar)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": WORKLOAD, "n_per_gpu": n, "global_samples_per_step": world * n,
                           "alg": "QM_BREAKLESS (App C)", "l2": "inputs 1 GiB per GPU > 126 MB L2: no flush",
                           "parallelism": f"dp{world} (counter-offset shards, no data-path collective)"},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": args.steps,
                "clocks": sampler.summary(), "variants": var}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
