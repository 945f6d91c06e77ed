"""GPU parity of the normal-quantile hot path against the oracle (SURVEY §8 rows
a1-a5, a7): every CUDA result is compared element by element with the oracle's
long-double evaluation of the same formula; bar: 4 ulp (fp32), 2 ulp (fp64)
(north star).  Calls go through the C ABI (libqm.so via the ctypes binding)."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import inputs as I
from _parity import summary, ulp_errors

pytestmark = pytest.mark.gpu

Q = pytest.importorskip("paper_0901_0638_b200")
SEED = 0x5EEDC0FFEE123457

CASES = [  # dtype, alg, oracle formula, coefficient precision, ulp bar
    (np.float32, Q.BREAKLESS, O.C55, 32, 4.0),
    (np.float32, Q.BREAKLESS77, O.A77, 32, 4.0),
    (np.float64, Q.BREAKLESS, O.D13, 64, 2.0),
    (np.float64, Q.BREAKLESS77, O.A77, 64, 2.0),
]


def _gpu(fn, x_np, **kw):
    x = torch.from_numpy(np.ascontiguousarray(x_np)).cuda()
    return fn(x, **kw).cpu().numpy()


@pytest.mark.parametrize("n", [(1 << 20) + 37, (1 << 23) + 37])
@pytest.mark.parametrize("dtype,alg,formula,prec,bar", CASES)
def test_normal_quantile_mixed_inputs(dtype, alg, formula, prec, bar, n):
    """Odd-grid uniforms, log-uniform tails, edge values (0, 1, 1/2, subnormals, NaN,
    out of range); several chunks of every warp and a ragged tail.  2^20 + 37 runs
    the LDG kernels, 2^23 + 37 the TMA pipelines (whole tiles) plus the remainder."""
    u = I.mixed_uniforms(n, dtype=dtype)
    g = _gpu(Q.qm_normal_quantile, u, alg=alg)
    ref = O.normal_breakless(u.astype(np.float64), formula, prec)
    err = ulp_errors(g, ref, dtype)
    assert err.max() <= bar, summary(err)


def test_fp32_breakless_exhaustive_grid():
    """Every point of the fp32 odd grid (2^23 values of min(u, 1-u)), both halves."""
    k = np.arange(1 << 23, dtype=np.float64)
    lo = np.ldexp(2 * k + 1, -24).astype(np.float32)          # (0, 1/2)
    u = np.concatenate([lo, (1 - lo.astype(np.float64)).astype(np.float32)])
    g = _gpu(Q.qm_normal_quantile, u, alg=Q.BREAKLESS)
    ref = O.normal_breakless(u.astype(np.float64), O.C55, 32)
    err = ulp_errors(g, ref, np.float32)
    assert err.max() <= 4.0, summary(err)
    # odd symmetry is exact: z(1-u) = -z(u)
    n = lo.size
    assert np.array_equal(g[n:], -g[:n])


@pytest.mark.parametrize("n", [20000, (1 << 22) + 37])          # LDG kernels / TMA pipeline
def test_fp64_off_grid_inputs(n):
    """Uniforms far below the 2^-54 odd grid (u = 10^U(-320, -16): z = 36 .. 736) and
    Laplace |v| up to 745 -- where App D's ten compensated steps are not enough (3.7 ulp
    measured at z = 477) and rat64 switches those lanes to the fully compensated form
    (qm_math.cuh): 2 ulp of the oracle, in warps mixed with on-grid samples."""
    rng = np.random.default_rng(21)
    u = 10.0 ** rng.uniform(-320, -16, n)
    u = np.where(rng.uniform(size=n) < 0.5, u, I.uniform_grid(n, dtype=np.float64))   # mixed warps
    u[1::7] = 1 - u[1::7]
    for alg, form in ((Q.BREAKLESS, O.D13), (Q.BREAKLESS77, O.A77)):
        err = ulp_errors(_gpu(Q.qm_normal_quantile, u, alg=alg), O.normal_breakless(u, form, 64), np.float64)
        assert err.max() <= 2.0, summary(err)
        err = ulp_errors(_gpu(Q.qm_normal_antithetic, u, alg=alg), O.normal_antithetic(u, form, 64), np.float64)
        assert err.max() <= 2.0, summary(err)
    v = rng.uniform(-745, 745, n)
    err = ulp_errors(_gpu(Q.qm_recycle_exp_to_normal, v), O.exp_to_normal(v, O.D13, 64), np.float64)
    assert err.max() <= 2.0, summary(err)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [0, 1, 3, 5, 63, 4097])
@pytest.mark.parametrize("offset", [0, 1])
def test_ragged_and_misaligned(dtype, n, offset):
    u = I.mixed_uniforms(n + offset + 64, dtype=dtype)[:n + offset]
    x = torch.from_numpy(u).cuda()[offset:]                   # offset 1: not 16-byte aligned
    out = torch.empty(n + 1, dtype=x.dtype, device="cuda")[1:] if offset else None
    g = Q.qm_normal_quantile(x, out=out).cpu().numpy()
    ref = O.normal_breakless(u[offset:].astype(np.float64), O.C55 if dtype == np.float32 else O.D13,
                             32 if dtype == np.float32 else 64)
    e = ulp_errors(g, ref, dtype)
    assert (e.max() if e.size else 0.0) <= (4.0 if dtype == np.float32 else 2.0)


@pytest.mark.parametrize("alg", [Q.BREAKLESS, Q.BREAKLESS77, Q.BREAKLESS_TAIL])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_pipeline_equals_ldg_kernel(dtype, alg):
    """qm.h promises results independent of the launch configuration: the TMA
    pipelines (aligned, >= 2^23 samples; vote per 8 / 2 samples per lane) and the
    LDG kernels (a misaligned view) give the same bits, specials included."""
    u = I.mixed_uniforms((1 << 23) + 37, dtype=dtype)
    x = torch.from_numpy(np.concatenate([[dtype(0.5)], u]).astype(dtype)).cuda()
    tiled = Q.qm_normal_quantile(x[1:].clone(), alg=alg)
    ldg = Q.qm_normal_quantile(x[1:], alg=alg)                     # 4/8-byte offset: misaligned
    assert torch.equal(tiled.nan_to_num(), ldg.nan_to_num()) and torch.equal(tiled.isnan(), ldg.isnan())


@pytest.mark.parametrize("n", [10000, (1 << 23) + 37])          # LDG kernels / TMA pipelines
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_in_place(n, dtype):
    """out aliasing the input (qm.h: in-place allowed): every pipeline tile is read
    by TMA before any consumer writes it, and tiles never overlap."""
    u = I.mixed_uniforms(n, dtype=dtype)
    x = torch.from_numpy(u).cuda()
    ref = Q.qm_normal_quantile(x.clone()).cpu().numpy()
    Q.qm_normal_quantile(x, out=x)
    assert np.array_equal(x.cpu().numpy(), ref, equal_nan=True)
    if dtype == np.float32:
        v = torch.from_numpy(I.laplace(n, dtype=np.float32)).cuda()
        ref = Q.qm_recycle_exp_to_normal(v.clone()).cpu().numpy()
        Q.qm_recycle_exp_to_normal(v, out=v)
        assert np.array_equal(v.cpu().numpy(), ref, equal_nan=True)
    else:
        zn = torch.from_numpy(I.normals(n, dtype=np.float64)).cuda()
        ref = Q.qm_recycle_normal_to_t(zn.clone(), 5.0, 16, 4.6506).cpu().numpy()
        Q.qm_recycle_normal_to_t(zn, 5.0, 16, 4.6506, out=zn)
        assert np.array_equal(zn.cpu().numpy(), ref, equal_nan=True)
        tab = Q.qm_exp_target_table(Q.HYPERBOLIC, [1.0, 0.5, 1.0])
        v = torch.from_numpy(I.laplace(n, dtype=np.float64)).cuda()
        ref = Q.qm_recycle_exp_to_hyperbolic(v.clone(), tab).cpu().numpy()
        Q.qm_recycle_exp_to_hyperbolic(v, tab, out=v)
        assert np.array_equal(v.cpu().numpy(), ref, equal_nan=True)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_philox_uniform_bit_exact(dtype):
    """Raw Philox stream bit-exact vs the oracle, including a counter offset and a ragged n."""
    n, c0 = (1 << 20) + 3, 123456789
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    g = Q.qm_philox_uniform(n, SEED, c0, dtype=tdt).cpu().numpy()
    ref = O.philox_uniform(n, SEED, c0, dtype)
    assert np.array_equal(g.view(np.uint32 if dtype == np.float32 else np.uint64),
                          ref.view(np.uint32 if dtype == np.float32 else np.uint64))


@pytest.mark.parametrize("dtype,alg", [(np.float32, Q.BREAKLESS), (np.float64, Q.BREAKLESS), (np.float32, Q.BREAKLESS77)])
def test_fused_equals_unfused_bitwise(dtype, alg):
    n, c0 = (1 << 20) + 5, 99
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    fused = Q.qm_normal_philox(n, SEED, c0, dtype=tdt, alg=alg)
    u = Q.qm_philox_uniform(n, SEED, c0, dtype=tdt)
    unf = Q.qm_normal_quantile(u, alg=alg)
    assert torch.equal(fused, unf)


def test_shards_concatenate_to_one_stream():
    """Counter-offset sharding (SURVEY §8 e): rank r of G generates blocks
    [r B, (r+1) B); the concatenation equals the single-GPU stream."""
    n, G = 1 << 20, 4
    whole = Q.qm_normal_philox(n, SEED, 0)
    parts = [Q.qm_normal_philox(n // G, SEED, r * (n // G) // 4) for r in range(G)]
    assert torch.equal(torch.cat(parts), whole)


@pytest.mark.parametrize("n", [50000, (1 << 23) + 37])          # LDG kernels / fp32 TMA pipeline
@pytest.mark.parametrize("dtype,alg,formula,prec,bar", CASES)
def test_antithetic(dtype, alg, formula, prec, bar, n):
    u = np.concatenate([I.edge_values(dtype), I.uniform_grid(n, dtype=dtype), I.edge_values(dtype)])
    g = _gpu(Q.qm_normal_antithetic, u, alg=alg)
    ref = O.normal_antithetic(u.astype(np.float64), formula, prec)
    err = ulp_errors(g, ref, dtype)
    assert err.max() <= bar, summary(err)


@pytest.mark.parametrize("dtype,alg,formula,prec,bar", CASES)
def test_exp_to_normal(dtype, alg, formula, prec, bar):
    big = [1e3, -1e6, 3e12, -1e30, 1e300] if dtype == np.float64 else [1e3, -1e6, 3e12, -1e30]
    v = np.concatenate([I.laplace(100000, dtype=dtype),
                        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 37.0, -74.0, 1e-30] + big, dtype=dtype)])
    g = _gpu(Q.qm_recycle_exp_to_normal, v, alg=alg)
    ref = O.exp_to_normal(v.astype(np.float64), formula, prec)
    err = ulp_errors(g, ref, dtype)
    assert err.max() <= bar, summary(err)


# -------------------------------------------------- comparison quantiles (a5)
@pytest.mark.parametrize("alg,name", [(Q.AS241, "as241"), (Q.ACKLAM, "acklam"), (Q.MORO, "moro")])
def test_branchy_baselines(alg, name):
    u = I.mixed_uniforms((1 << 18) + 11, dtype=np.float64)
    if name == "moro":   # both sides of Moro's break and its neighbourhood
        u = np.concatenate([u, 0.08 + np.linspace(-1e-9, 1e-9, 101), 0.92 + np.linspace(-1e-9, 1e-9, 101)])
    g = _gpu(Q.qm_normal_quantile, u, alg=alg)
    ref = {"as241": lambda: O.normal_as241(u, 64), "acklam": lambda: O.normal_acklam(u, 64, False),
           "moro": lambda: O.normal_moro(u, 64)}[name]()
    err = ulp_errors(g, ref, np.float64)
    assert err.max() <= 2.0, summary(err)


def test_refined_acklam():
    """Refined Acklam: the Halley step forms Phi(x) - t in double (as published), so
    near the centre its error is |d(Phi - t)|/phi(x) ~ 8 eps t / phi(x) -- the
    paper's 'loss of precision in the middle'.  Bar: 2 ulp + that term."""
    u = I.mixed_uniforms((1 << 18) + 11, dtype=np.float64)
    g = _gpu(Q.qm_normal_quantile, u, alg=Q.ACKLAM_REFINED)
    ref = O.normal_acklam(u, 64, True)
    fin = np.isfinite(ref)
    r = ref[fin].astype(np.float64)
    t = np.minimum(u[fin], 1 - u[fin])
    phi = np.exp(-0.5 * r * r) / np.sqrt(2 * np.pi)
    tol = 2 * np.spacing(np.abs(r)) + 8 * np.finfo(np.float64).eps * t / phi
    assert np.all(np.abs(g[fin] - r) <= tol)
    assert np.array_equal(np.isnan(g), np.isnan(ref.astype(np.float64)))


# ------------------------- config 1 like-for-like: plain double
@pytest.mark.parametrize("alg,name,nterms", [(Q.BREAKLESS, "d13", 14), (Q.BREAKLESS77, "a77", 8), (Q.AS241, "as241", 8)])
def test_plain_double_versions(alg, name, nterms):
    """qm_normal_quantile_plain: the same formulas coded in plain double like the
    paper's Table 3 programs.  For these positive-coefficient rationals the plain
    evaluation error is bounded by (2 N + 5) ulp of the same formula (N = terms of
    the longer polynomial; 2N roundings of two Horner chains, + log/sqrt, division
    and the final product); tail-stratified inputs exercise every region."""
    u = np.concatenate([I.tail_stratified((1 << 18) + 11, dtype=np.float64), I.mixed_uniforms(1 << 16, dtype=np.float64)])
    g = _gpu(Q.qm_normal_quantile_plain, u, alg=alg)
    ref = {"d13": lambda: O.normal_breakless(u, O.D13, 64), "a77": lambda: O.normal_breakless(u, O.A77, 64),
           "as241": lambda: O.normal_as241(u, 64)}[name]()
    err = ulp_errors(g, ref, np.float64)
    print(name, "plain max ulp", summary(err))
    assert err.max() <= 2 * nterms + 5, summary(err)


@pytest.mark.parametrize("alg,name,bound", [(Q.ACKLAM, "acklam", 1.15e-9), (Q.MORO, "moro", 3.1e-9)])
def test_plain_double_mixed_sign_formulas(alg, name, bound):
    """Acklam's and Moro's central rationals have coefficients of both signs, so
    plain double loses digits to cancellation (no ulp bound of the formula); the
    check is the formula's own accuracy against the exact quantile -- Acklam L1
    1.15e-9 relative, Moro 3e-9 absolute for |x| <= 7 (R26) -- plus
    2 ulp."""
    u = np.concatenate([I.tail_stratified((1 << 18) + 11, dtype=np.float64), I.mixed_uniforms(1 << 16, dtype=np.float64)])
    g = _gpu(Q.qm_normal_quantile_plain, u, alg=alg)
    ex = O.ndtri_exact(u).astype(np.float64)
    fin = np.isfinite(ex) & (np.abs(ex) <= 7)
    if name == "acklam":
        ok = np.abs(g[fin] - ex[fin]) <= bound * np.abs(ex[fin]) + 2 * np.spacing(np.abs(ex[fin]))
    else:
        ok = np.abs(g[fin] - ex[fin]) <= bound + 2 * np.spacing(np.abs(ex[fin]))
    assert np.all(ok)
    spec = ~np.isfinite(ex)
    assert np.array_equal(g[spec], ex[spec], equal_nan=True)


def test_plain_refined_acklam():
    u = I.tail_stratified((1 << 18) + 11, dtype=np.float64)
    g = _gpu(Q.qm_normal_quantile_plain, u, alg=Q.ACKLAM_REFINED)
    ref = O.normal_acklam(u, 64, True)
    fin = np.isfinite(ref)
    r = ref[fin].astype(np.float64)
    t = np.minimum(u[fin], 1 - u[fin])
    phi = np.exp(-0.5 * r * r) / np.sqrt(2 * np.pi)
    tol = 4 * np.spacing(np.abs(r)) + 8 * np.finfo(np.float64).eps * t / phi
    assert np.all(np.abs(g[fin] - r) <= tol)


# --------------------------------------- full size, bench launch configuration
def test_full_size_streaming_sampled():
    """configs[1]: 2^28 fp32 uniforms in HBM -> breakless quantile (the bench.py
    launch); 2^20 sampled outputs checked against the oracle one by one."""
    n = 1 << 28
    u = Q.qm_philox_uniform(n, SEED, 0)
    z = Q.qm_normal_quantile(u)
    idx = np.sort(np.random.default_rng(1).choice(n, 1 << 20, replace=False))
    ti = torch.from_numpy(idx).cuda()
    us, zs = u[ti].cpu().numpy(), z[ti].cpu().numpy()
    assert np.array_equal(us, O.philox_uniform_at(idx, SEED, 0, np.float32))
    err = ulp_errors(zs, O.normal_breakless(us.astype(np.float64), O.C55, 32), np.float32)
    assert err.max() <= 4.0, summary(err)
    # whole-array properties: finite, |z| < 5.4 on the fp32 grid, sign matches u - 1/2
    assert bool(torch.isfinite(z).all()) and float(z.abs().max()) < 5.4
    assert int((z > 0).sum()) == int((u > 0.5).sum())
    del u, z


def test_full_size_fused_sampled():
    """configs[2]: Philox-fused 2^32 fp32 normal samples; sampled parity."""
    n = 1 << 32
    z = Q.qm_normal_philox(n, SEED, 0)
    idx = np.sort(np.random.default_rng(2).choice(n, 1 << 18, replace=False))
    zs = z[torch.from_numpy(idx).cuda()].cpu().numpy()
    us = O.philox_uniform_at(idx, SEED, 0, np.float32)
    err = ulp_errors(zs, O.normal_breakless(us.astype(np.float64), O.C55, 32), np.float32)
    assert err.max() <= 4.0, summary(err)
    m = z.double().mean().item()
    assert abs(m) < 6 / np.sqrt(n) * 10
    del z


def test_host_entry_point_equals_device():
    """The e2e C-ABI call on host buffers gives the device path's bits."""
    u = I.mixed_uniforms((1 << 22) + 7, dtype=np.float32)
    dev = _gpu(Q.qm_normal_quantile, u)
    host = Q.qm_normal_quantile_host(torch.from_numpy(u)).numpy()
    assert np.array_equal(dev, host, equal_nan=True)
    u64 = I.mixed_uniforms((1 << 20) + 7, dtype=np.float64)
    assert np.array_equal(_gpu(Q.qm_normal_quantile, u64),
                          Q.qm_normal_quantile_host(torch.from_numpy(u64)).numpy(), equal_nan=True)


def test_determinism_across_launches():
    u = torch.from_numpy(I.mixed_uniforms(1 << 20, dtype=np.float64)).cuda()
    a = Q.qm_normal_quantile(u)
    b = Q.qm_normal_quantile(u)
    assert torch.equal(a.nan_to_num(), b.nan_to_num())


@pytest.mark.parametrize("alg", [Q.BREAKLESS, Q.BREAKLESS77, Q.BREAKLESS_TAIL])
def test_antithetic_pipeline_equals_ldg(alg):
    u = I.mixed_uniforms((1 << 23) + 37, dtype=np.float32)
    x = torch.from_numpy(np.concatenate([[np.float32(0.5)], u])).cuda()
    tiled = Q.qm_normal_antithetic(x[1:].clone(), alg=alg)
    ldg = Q.qm_normal_antithetic(x[1:], alg=alg)                         # misaligned: LDG kernel
    assert torch.equal(tiled.nan_to_num(), ldg.nan_to_num()) and torch.equal(tiled.isnan(), ldg.isnan())


def test_ring_release_race_regression():
    """Regression for the cross-proxy WAR race of the TMA ring: with
    fresh buffers every run, a stage released before its generic reads were
    fenced was sometimes refilled under a warp (one slice of the next tile's
    inputs).  Twelve runs of the antithetic and plain pipelines must all equal the
    LDG kernels bitwise."""
    u = np.concatenate([I.edge_values(np.float32), I.uniform_grid((1 << 23) + 37, dtype=np.float32)])
    x = torch.from_numpy(np.concatenate([[np.float32(0.5)], u])).cuda()
    ref_a = Q.qm_normal_antithetic(x[1:])
    ref_n = Q.qm_normal_quantile(x[1:])
    import time
    for _ in range(12):
        time.sleep(0.1)                                   # an idle GPU between runs made it show
        xa = torch.from_numpy(u).cuda()
        assert torch.equal(Q.qm_normal_antithetic(xa).nan_to_num(), ref_a.nan_to_num())
        assert torch.equal(Q.qm_normal_quantile(xa).nan_to_num(), ref_n.nan_to_num())

