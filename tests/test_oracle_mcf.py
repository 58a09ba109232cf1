"""Pins for the oracle of Dziuk's MCF algorithm:
(M(x^{n-1}) + tau A(x^{n-1})) x^n = M(x^{n-1}) x^{n-1}.

* Sphere: mean curvature flow shrinks a sphere as r(t)^2 = r0^2 - 4t (surface in
  R^3, H = 2/r).  The linearly implicit Euler scheme is first order in tau:
  the radius error at T = 0.04 halves with tau (EOC 1) and is < 1.5e-3 at
  tau = 0.004 on P2 icospheres (spatial error below that).
* Homogeneity: M scales with R^2 and A is scale-free on surfaces, so the
  scheme maps R x with step R^2 tau to R times the unit result (catches a
  misplaced tau).
* Translation: A 1 = 0 and M on both sides make x + c -> x^n + c (catches a
  missing M on the right-hand side).
"""
import numpy as np
import pytest

import lfem_inputs as li
from oracle import mcf


def mean_radius(x):
    return float(np.sqrt(np.mean(np.sum(x * x, axis=1))))


@pytest.mark.parametrize("level", [2, 3])
def test_sphere_radius_law_first_order(level):
    m = li.sphere_mesh(level, 2)
    T = 0.04
    errs = []
    for tau in (0.004, 0.002):
        xs = mcf.mcf(m, tau, int(round(T / tau)))
        errs.append(abs(mean_radius(xs[-1]) - np.sqrt(1.0 - 4.0 * T)))
    assert errs[0] < 1.5e-3
    assert 1.8 < errs[0] / errs[1] < 2.3  # EOC 1 in tau


def test_homogeneity():
    m = li.perturb(li.sphere_mesh(2, 2), 3, 0.02)
    R, tau = 2.5, 0.003
    x1 = mcf.mcf(m, tau, 3)[-1]
    mR = li.Mesh(m.domain, m.order, R * m.coords, m.conn, m.quad)
    xR = mcf.mcf(mR, R * R * tau, 3)[-1]
    assert np.allclose(xR, R * x1, rtol=0, atol=1e-12 * R)


def test_translation():
    m = li.perturb(li.sphere_mesh(2, 1), 4, 0.02)
    c = np.array([0.3, -1.2, 2.0])
    x1 = mcf.mcf(m, 0.002, 2)[-1]
    mc = li.Mesh(m.domain, m.order, m.coords + c, m.conn, m.quad)
    xc = mcf.mcf(mc, 0.002, 2)[-1]
    assert np.allclose(xc, x1 + c, rtol=0, atol=1e-11)


def test_dziuk_surface_shrinks_and_smooths():
    """The paper's initial surface loses area and its radius spread shrinks under the flow."""
    m = li.dziuk_surface(2, 2)
    xs = mcf.mcf(m, 0.005, 4)
    spread = [np.ptp(np.sqrt(np.sum(x * x, axis=1))) for x in xs]
    assert all(b < a for a, b in zip(spread, spread[1:]))
