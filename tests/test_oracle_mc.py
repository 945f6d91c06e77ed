"""Pins for the oracle's Monte-Carlo call sweep (config 5 of BASELINE.json;
SURVEY §8 d5, c6): orc_mc_call draws its normal innovations from the
exponential base (v = -log u, a random sign, Z = Q(v)
with the App C rational).  Independent of that code:

* the price exp(-rT) mean (S_T - K)^+ agrees with the Black-Scholes closed form
  (mpmath) within 4 standard errors at every strike (2^22 samples);
* the strike K = 0 gives the forward: E S_T = S0 e^{rT} (martingale), within 4 se;
* sigma = 0 is deterministic: S_T = S0 e^{rT} exactly (to long double rounding);
* T = 0 gives the intrinsic value (S0 - K)^+ exactly.
"""
import numpy as np

import oracle as O

S0, R, SIG, T = 100.0, 0.05, 0.2, 1.0
STRIKES = list(np.linspace(50, 150, 17))
N = 1 << 22


def _price_se(sums, n, r, T):
    s1, s2 = sums[:, 0].astype(np.float64), sums[:, 1].astype(np.float64)
    mean = s1 / n
    var = np.maximum(s2 / n - mean ** 2, 0.0)
    disc = np.exp(-r * T)
    return disc * mean, disc * np.sqrt(var / n)


def test_mc_call_vs_black_scholes():
    sums = O.mc_call(N, 0x5EEDC0FFEE123457, 0, S0, R, SIG, T, STRIKES + [0.0])
    price, se = _price_se(sums, N, R, T)
    bs = O.black_scholes_call(S0, STRIKES, R, SIG, T)
    z = np.abs(price[:-1] - bs) / se[:-1]
    assert z.max() < 4.0, z
    # K = 0: the discounted forward is S0 (E[e^{sigma sqrt(T) Z}] = e^{sigma^2 T/2})
    assert abs(price[-1] - S0) < 4 * se[-1], (price[-1], se[-1])


def test_mc_call_deterministic_limits():
    n = 4097
    sums = O.mc_call(n, 7, 3, S0, R, 0.0, T, [0.0, 90.0, 110.0])
    fwd = S0 * np.exp(np.longdouble(R) * np.longdouble(T))
    assert np.all(np.abs(sums[:, 0] / n - np.array([fwd, fwd - 90, 0.0])) <= 1e-15 * fwd)
    sums = O.mc_call(n, 7, 3, S0, R, SIG, 0.0, [80.0, 100.0, 120.0])
    assert np.all(np.abs(sums[:, 0] / n - np.array([20.0, 0.0, 0.0])) <= 1e-15 * S0)
