"""Pins for the oracle's reference data: basis functions and quadrature rules.

The oracle (oracle/lfem_oracle.cpp) builds its own basis (PAPER.md Eq.
form_functions_s2dp2, with the Lagrange vertex functions of
reading G1) and rules (readings G6-G9).  These tests pin them to facts fixed
by mathematics: the Lagrange property phi_j(x_i) = delta_ij,
partition of unity, finite differences, and exact monomial integration
int_T x^a y^b = a! b! / (a+b+2)!  (tetrahedron: a! b! c! / (a+b+c+3)!).
"""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
from lfem_inputs import (BULK_TET, QUAD_TET11_DEG4, QUAD_TET4_DEG2, QUAD_TRI3_DEG2,
                         QUAD_TRI6_DEG4, QUAD_TRI16_DEG8, SURFACE_TRI)

# reference nodes in barycentric coordinates, local order of reading G26
TRI_P2_NODES = [(1, 0, 0), (0, 1, 0), (0, 0, 1), (.5, .5, 0), (0, .5, .5), (.5, 0, .5)]
TET_P2_NODES = [(1, 0, 0, 0), (0, 1, 0, 0), (0, 0, 1, 0), (0, 0, 0, 1),
                (.5, .5, 0, 0), (0, .5, .5, 0), (.5, 0, .5, 0), (.5, 0, 0, .5),
                (0, .5, 0, .5), (0, 0, .5, .5)]


@pytest.mark.parametrize("domain,order,nodes", [
    (SURFACE_TRI, 1, TRI_P2_NODES[:3]), (SURFACE_TRI, 2, TRI_P2_NODES),
    (BULK_TET, 1, TET_P2_NODES[:4]), (BULK_TET, 2, TET_P2_NODES)])
def test_lagrange_property(domain, order, nodes):
    n = len(nodes)
    for i, lam in enumerate(nodes):
        phi, _ = oracle.basis(domain, order, lam)
        e = np.zeros(n)
        e[i] = 1.0
        assert np.array_equal(phi[:n], e), (i, phi[:n])


def _rand_bary(rng, d):
    x = rng.random(d + 1)
    return x / x.sum()


@pytest.mark.parametrize("domain,order", [(SURFACE_TRI, 1), (SURFACE_TRI, 2), (BULK_TET, 1), (BULK_TET, 2)])
def test_partition_of_unity_and_gradients(domain, order):
    d = 2 if domain == SURFACE_TRI else 3
    n = oracle.lib().oracle_nref(domain, order)
    rng = np.random.default_rng(7)
    for _ in range(20):
        lam = _rand_bary(rng, d)
        phi, grad = oracle.basis(domain, order, lam)
        assert abs(phi[:n].sum() - 1.0) < 1e-15
        assert np.abs(grad[:n, :d].sum(axis=0)).max() < 1e-14
        # finite differences along xi_m (lam_0 absorbs the change)
        h = 1e-6
        for m in range(d):
            lp = lam.copy(); lp[m + 1] += h; lp[0] -= h
            lm = lam.copy(); lm[m + 1] -= h; lm[0] += h
            fd = (oracle.basis(domain, order, lp)[0] - oracle.basis(domain, order, lm)[0]) / (2 * h)
            assert np.abs(fd[:n] - grad[:n, m]).max() < 1e-8


def test_printed_p2_basis_is_not_a_partition_of_unity():
    """Reading G1: the P2 vertex functions as printed break sum phi = 1;
    the oracle's Lagrange basis keeps it (tested above)."""
    x, y = 0.2, 0.3
    printed = [1 - x - y, x, y, 4 * x * (1 - x - y), 4 * x * y, 4 * y * (1 - x - y)]
    assert abs(sum(printed) - (1 + 4 * x + 4 * y - 4 * x * x - 4 * x * y - 4 * y * y)) < 1e-15
    assert abs(sum(printed) - 1.0) > 0.1


def _exact_tri(a, b):
    return Fraction(math.factorial(a) * math.factorial(b), math.factorial(a + b + 2))


def _exact_tet(a, b, c):
    return Fraction(math.factorial(a) * math.factorial(b) * math.factorial(c), math.factorial(a + b + c + 3))


@pytest.mark.parametrize("quad,deg,npts", [(QUAD_TRI3_DEG2, 2, 3), (QUAD_TRI6_DEG4, 4, 6), (QUAD_TRI16_DEG8, 8, 16)])
def test_triangle_rule_exactness(quad, deg, npts):
    lam, w = oracle.rule(quad)
    assert lam.shape[0] == npts
    assert np.all(lam >= 0) and np.allclose(lam[:, :3].sum(1), 1.0, atol=1e-15)
    x, y = lam[:, 1], lam[:, 2]
    for a in range(deg + 2):
        for b in range(deg + 2 - a):
            q = float(np.sum(w * x ** a * y ** b))
            ex = float(_exact_tri(a, b))
            if a + b <= deg:
                assert abs(q - ex) < 2e-16 * max(1.0, 50 * ex) + 1e-17, (a, b, q, ex)
    # not exact one degree higher (the rule is exactly of the stated degree)
    errs = [abs(float(np.sum(w * x ** a * y ** (deg + 1 - a))) - float(_exact_tri(a, deg + 1 - a)))
            for a in range(deg + 2)]
    assert max(errs) > 1e-8


@pytest.mark.parametrize("quad,deg,npts", [(QUAD_TET4_DEG2, 2, 4), (QUAD_TET11_DEG4, 4, 11), (8, 7, 35)])
def test_tet_rule_exactness(quad, deg, npts):
    lam, w = oracle.rule(quad)
    assert lam.shape[0] == npts
    assert np.allclose(lam.sum(1), 1.0, atol=1e-15)
    x, y, z = lam[:, 1], lam[:, 2], lam[:, 3]
    for a, b, c in itertools.product(range(deg + 2), repeat=3):
        if a + b + c > deg + 1:
            continue
        q = float(np.sum(w * x ** a * y ** b * z ** c))
        ex = float(_exact_tet(a, b, c))
        if a + b + c <= deg:
            assert abs(q - ex) < 1e-16 + 1e-14 * ex, (a, b, c, q, ex)
    errs = [abs(float(np.sum(w * x ** a * y ** b * z ** (deg + 1 - a - b))) - float(_exact_tet(a, b, deg + 1 - a - b)))
            for a in range(deg + 2) for b in range(deg + 2 - a)]
    assert max(errs) > 1e-8
    if quad == QUAD_TET11_DEG4:
        assert w.min() < 0  # reading G8: Keast's centroid weight is negative


def test_tet35_rule_positive_interior_symmetric():
    """Reading G39 (the paper's degree-7 tet rule): every weight positive, every point
    interior, and the point set invariant under all 24 permutations of the barycentrics
    (a fully symmetric rule), weights equal on each orbit."""
    lam, w = oracle.rule(8)
    assert w.min() > 0 and lam.min() > 0
    key = {tuple(np.round(l, 14)): wi for l, wi in zip(lam, w)}
    for l, wi in zip(lam, w):
        for perm in itertools.permutations(range(4)):
            k = tuple(np.round(l[list(perm)], 14))
            assert k in key and abs(key[k] - wi) < 1e-18
