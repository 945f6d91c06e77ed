"""GPU parity of the deep-tail composite QM_BREAKLESS_TAIL:
the breakless rational for v < vc and the §5.1 tail model beyond,
vc = 37 (fp32, App C) / 86.75 (fp64, App D, reading R23)."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import inputs as I
from _parity import summary, ulp_errors

pytestmark = pytest.mark.gpu
Q = pytest.importorskip("paper_0901_0638_b200")

VC = {np.float32: (O.C55, 32, 37.0, 4.0), np.float64: (O.D13, 64, 86.75, 2.0)}


def _deep_uniforms(dtype, nmix=20000):
    rng = np.random.default_rng(11)
    lo = -44 if dtype == np.float32 else -320
    t = 10.0 ** rng.uniform(lo, -15, 20000)                 # v = -log(2t) from ~33 up to the range end
    u = np.concatenate([t, 1 - t[:100], I.mixed_uniforms(nmix, dtype=dtype).astype(np.float64)])
    return u.astype(dtype)


@pytest.mark.parametrize("nmix", [20000, 1 << 23])          # LDG kernels / TMA pipelines
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_tail_composite_quantile(dtype, nmix):
    f, p, vc, bar = VC[dtype]
    u = _deep_uniforms(dtype, nmix)
    g = Q.qm_normal_quantile(torch.from_numpy(u).cuda(), alg=Q.BREAKLESS_TAIL).cpu().numpy()
    ref = O.normal_breakless_tail(u.astype(np.float64), f, p, vc)
    err = ulp_errors(g, ref, dtype)
    assert err.max() <= bar, summary(err)
    # and it is the plain breakless map wherever v < vc
    plain = Q.qm_normal_quantile(torch.from_numpy(u).cuda()).cpu().numpy()
    vv = np.minimum(u.astype(np.float64), 1 - u.astype(np.float64))
    inside = (vv > 2 * np.exp(-vc) / 2) & np.isfinite(u)
    assert np.array_equal(g[inside], plain[inside])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_tail_composite_exp_to_normal_and_antithetic(dtype):
    f, p, vc, bar = VC[dtype]
    v = np.concatenate([I.laplace(20000, dtype=np.float64), np.linspace(30, 700, 5000), -np.linspace(30, 700, 5000),
                        [np.inf, -np.inf, np.nan, 0.0, 1e30]]).astype(dtype)
    g = Q.qm_recycle_exp_to_normal(torch.from_numpy(v).cuda(), alg=Q.BREAKLESS_TAIL).cpu().numpy()
    err = ulp_errors(g, O.exp_to_normal_tail(v.astype(np.float64), f, p, vc), dtype)
    assert err.max() <= bar, summary(err)
    u = _deep_uniforms(dtype)
    u = u[(u > 0) & (u <= 1)]
    g = Q.qm_normal_antithetic(torch.from_numpy(u).cuda(), alg=Q.BREAKLESS_TAIL).cpu().numpy()
    v = np.abs(-np.log(u.astype(np.longdouble)))                         # +0 at u = 1
    ref = np.empty(2 * u.size, np.longdouble)
    ref[0::2] = O.exp_to_normal_tail(v.astype(np.float64), f, p, vc)       # Z = composite(-log u)
    ref[1::2] = -ref[0::2]
    err = ulp_errors(g, ref, dtype)
    # -log u in long double vs the kernel's log: compare through the tail model's
    # condition number (~1/(2v)) -> within the same bar
    assert err.max() <= bar + 0.5, summary(err)
