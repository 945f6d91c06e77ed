"""Seeded synthetic inputs for tests and bench (no method arithmetic here).

This module is the only thing the product tests and the oracle tests share.  It
draws base samples with numpy's generators and places them on exact grids; it
computes nothing the paper's method computes.  Recipes:

* ``uniform_grid``   -- iid uniforms on the odd grid (2k+1) 2^-b (b = 24 for
  fp32, 53 for fp64): "sample u in 0<u<1", never 0 or 1, symmetric.
* ``tail_stratified`` -- half uniform, half log-uniform in min(u, 1-u) over
  [2^-b, 1/2] with a random side: exercises the tails and, for the branching
  baselines, the divergence the paper argues about.
* ``edge_values``    -- 0, 1/2, 1, the smallest grid points, subnormals, NaN,
  out-of-range values and the printed pins (0.975, 0.025, 0.75).
* ``mixed_uniforms`` -- concatenation of the above with a ragged length.
* ``laplace``        -- two-sided unit exponential samples (P:315-329 with
  alpha = 1, beta = 0, p+- = 1/2; the base of P:397-405).
* ``normals``        -- standard normal samples (the Gaussian base of §3).
"""
from __future__ import annotations

import numpy as np

SEED = 0x5EEDC0FFEE123457


def _bits(dtype) -> int:
    return 24 if np.dtype(dtype) == np.float32 else 53


def uniform_grid(n: int, seed: int = SEED, dtype=np.float32) -> np.ndarray:
    b = _bits(dtype)
    rng = np.random.default_rng(seed)
    k = rng.integers(0, 2 ** (b - 1), size=n, dtype=np.int64)
    return np.ldexp((2 * k + 1).astype(np.float64), -b).astype(dtype)


def tail_stratified(n: int, seed: int = SEED, dtype=np.float32) -> np.ndarray:
    b = _bits(dtype)
    rng = np.random.default_rng(seed + 1)
    half = uniform_grid(n // 2, seed + 2, dtype)
    m = n - n // 2
    # log-uniform t in [2^-b, 1/2], rounded to a multiple of 2^-b (exact grid point)
    t = np.exp2(rng.uniform(-b, -1, size=m))
    t = np.maximum(np.round(np.ldexp(t, b)), 1.0)
    t = np.ldexp(t, -b)
    side = rng.uniform(size=m) < 0.5
    u = np.where(side, t, 1.0 - t)          # exact: t is on the grid
    out = np.concatenate([half.astype(np.float64), u])
    rng.shuffle(out)
    return out.astype(dtype)


def edge_values(dtype=np.float32) -> np.ndarray:
    b = _bits(dtype)
    tiny = np.finfo(dtype).smallest_subnormal
    vals = [0.0, 0.5, 1.0, 2.0 ** -b, 1 - 2.0 ** -b, 3 * 2.0 ** -b, 0.975, 0.025, 0.75, 0.25,
            0.5 + 2.0 ** -b, 0.5 - 2.0 ** -b, float(tiny), float(np.finfo(dtype).tiny),
            1e-30, 1e-38, -0.0, np.nan, -0.25, 1.5, np.inf, -np.inf]
    if b == 53:
        vals += [1e-300, 5e-324, 2.0 ** -1022, 1e-100]
    return np.array(vals, dtype=np.float64).astype(dtype)


def mixed_uniforms(n: int, seed: int = SEED, dtype=np.float32) -> np.ndarray:
    e = edge_values(dtype)
    m = max(n - e.size, 0)
    return np.concatenate([uniform_grid(m // 2, seed, dtype), tail_stratified(m - m // 2, seed, dtype), e])


def laplace(n: int, seed: int = SEED, dtype=np.float64) -> np.ndarray:
    rng = np.random.default_rng(seed + 3)
    e = rng.standard_exponential(n)
    s = rng.uniform(size=n) < 0.5
    return np.where(s, e, -e).astype(dtype)


def normals(n: int, seed: int = SEED, dtype=np.float64) -> np.ndarray:
    rng = np.random.default_rng(seed + 4)
    return rng.standard_normal(n).astype(dtype)
