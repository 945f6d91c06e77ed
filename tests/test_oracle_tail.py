"""Pins for the deep-tail composite: the breakless rational
for v < vc and the §5.1 supplementary tail model beyond."""
import numpy as np

import oracle as O

VGRID = np.concatenate([np.linspace(0.01, 37, 3000), np.linspace(37, 120, 3000), np.linspace(120, 700, 600)])


def _composite_q(formula, prec, vc):
    # u with v = -log(2 vv): vv = e^-v / 2 (long double), evaluate through the uniform entry point
    v = VGRID.astype(np.longdouble)
    return v, O.exp_to_normal_tail(VGRID, formula, prec, vc)


def test_tail_model_meets_77_at_37():
    """'This again has precision better than 1.06e-9, now in the region v >= 37'
    (P:529): with the (7,7) rational below 37 the composite is within 1.06e-9 on [0, 700]."""
    v, q = _composite_q(O.A77, 0, 37.0)
    e = np.abs(q / O.Q_exact(v) - 1).astype(float)
    assert e.max() < 1.06e-9


def test_composite_D13_and_C55():
    """R23: App D to v = 86.75, then the tail model: < 4e-12 everywhere (App D alone
    reaches 6e-7 at v = 200); App C to v = 37: its own 4e-7 bound everywhere."""
    v, q = _composite_q(O.D13, 0, 86.75)
    e = np.abs(q / O.Q_exact(v) - 1).astype(float)
    assert e.max() < 4.1e-12
    alone = np.abs(O.rational(v, O.D13, 0) / O.Q_exact(v) - 1).astype(float)
    assert alone.max() > 1e-7
    v, q = _composite_q(O.C55, 0, 37.0)
    assert (np.abs(q / O.Q_exact(v) - 1).astype(float)).max() < 4e-7


def test_composite_uniform_entry_and_specials():
    u = np.array([1e-300, 1 - 2.0 ** -53, 0.3, 0.0, 1.0, np.nan, 5e-324])
    r = O.normal_breakless_tail(u, O.D13, 64, 86.75)
    ex = O.ndtri_exact(u[:3])
    assert np.all(np.abs(r[:3] / ex - 1) < 4.1e-12)
    assert r[3] == -np.inf and r[4] == np.inf and np.isnan(r[5])
    assert abs(float(r[6] / O.ndtri_exact([5e-324])[0]) - 1) < 1e-13
    # below vc the composite is the rational itself
    w = np.array([0.2, 1e-10])
    assert np.array_equal(O.normal_breakless_tail(w, O.C55, 32, 37.0), O.normal_breakless(w, O.C55, 32))
