"""Pins for the oracle's local element matrices against closed forms.

* P1 triangle: M = (area/12)[2 1 1; 1 2 1; 1 1 2] (BASELINE.json north_star)
  and the cotangent stiffness A_ab = -cot(theta_c)/2 (textbook).
* P1 triangle A_a: (1 + (sum u_i^2 + sum_{i<j} u_i u_j)/6) A (exact: a(u_h) is
  degree 2 and the gradients are constant).
* P1 tet: M = (V/20)(1 + delta_ab); A_ab = s_a s_b (n_a . n_b) / (9 V).
* Flat P2 triangle / P2 tet: M and A by EXACT symbolic integration in
  physical coordinates (sympy), with the Lagrange basis obtained by solving
  the Vandermonde system on the physical nodes -- no reference element, no
  quadrature, no Jacobian: an independent computation.  The quadrature rules
  are exact on these integrands (degree <= 4).
* Invariance: rigid motion, scaling (M x s^d, A x s^{d-2}), cyclic relabelling.
* Second formulation (reading G2): Listing 1's L^{-T}[grad; 0]
  equals the metric form J G^{-1} grad on curved P2 elements.
"""
import math

import numpy as np
import pytest
import sympy as sp

import oracle
from lfem_inputs import (BULK_TET, QUAD_TET11_DEG4, QUAD_TET4_DEG2, QUAD_TRI3_DEG2,
                         QUAD_TRI6_DEG4, SURFACE_TRI)

RNG = np.random.default_rng(1234)


def rot(seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((3, 3)))
    return q


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


# ------------------------------------------------------------------ P1 triangle
def _cot_stiffness(P):
    A = np.zeros((3, 3))
    for c in range(3):
        a, b = (c + 1) % 3, (c + 2) % 3
        u = P[a] - P[c]
        v = P[b] - P[c]
        cot = np.dot(u, v) / np.linalg.norm(np.cross(u, v))
        A[a, b] = A[b, a] = -0.5 * cot
    for a in range(3):
        A[a, a] = -A[a].sum()
    return A


@pytest.mark.parametrize("seed", range(5))
def test_p1_triangle_closed_forms(seed):
    rng = np.random.default_rng(seed)
    P = rng.standard_normal((3, 3))
    area = 0.5 * np.linalg.norm(np.cross(P[1] - P[0], P[2] - P[0]))
    u = rng.standard_normal(3)
    M, A, Aa = oracle.element_matrices(SURFACE_TRI, 1, QUAD_TRI3_DEG2, P, u)
    Mex = area / 12.0 * np.array([[2, 1, 1], [1, 2, 1], [1, 1, 2]])
    assert rel(M, Mex) < 1e-14
    assert rel(A, _cot_stiffness(P)) < 1e-13
    fac = 1.0 + (np.sum(u * u) + u[0] * u[1] + u[1] * u[2] + u[0] * u[2]) / 6.0
    assert rel(Aa, fac * A) < 1e-13


def test_p1_reference_triangle_exact():
    P = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], dtype=float)
    M, A, _ = oracle.element_matrices(SURFACE_TRI, 1, QUAD_TRI3_DEG2, P)
    assert rel(M, np.array([[2, 1, 1], [1, 2, 1], [1, 1, 2]]) / 24.0) < 1e-15
    assert rel(A, 0.5 * np.array([[2, -1, -1], [-1, 1, 0], [-1, 0, 1]])) < 1e-15


# ------------------------------------------------------------------ P1 tet
@pytest.mark.parametrize("seed", range(4))
def test_p1_tet_closed_forms(seed):
    rng = np.random.default_rng(100 + seed)
    P = rng.standard_normal((4, 3))
    V = abs(np.linalg.det(np.stack([P[1] - P[0], P[2] - P[0], P[3] - P[0]]))) / 6.0
    M, A, _ = oracle.element_matrices(BULK_TET, 1, QUAD_TET4_DEG2, P)
    assert rel(M, V / 20.0 * (np.ones((4, 4)) + np.eye(4))) < 1e-13
    # face opposite a: area s_a, outward unit normal n_a
    An = np.zeros((4, 4))
    sn = []
    c = P.mean(0)
    for a in range(4):
        f = [i for i in range(4) if i != a]
        nrm = np.cross(P[f[1]] - P[f[0]], P[f[2]] - P[f[0]])
        if np.dot(nrm, P[f[0]] - c) < 0:
            nrm = -nrm
        sn.append(0.5 * nrm)  # s_a n_a
    for a in range(4):
        for b in range(4):
            An[a, b] = np.dot(sn[a], sn[b]) / (9.0 * V)
    assert rel(A, An) < 1e-12


# ------------------------------------------------------------------ exact P2 (sympy)
x, y, z = sp.symbols("x y z")


def _lagrange_basis(nodes, monos, vars_):
    V = sp.Matrix([[m.subs(dict(zip(vars_, p))) for m in monos] for p in nodes])
    Vi = V.inv()
    # phi_j = sum_k monos_k Vi[k, j]
    return [sp.expand(sum(monos[k] * Vi[k, j] for k in range(len(monos)))) for j in range(len(nodes))]


def _exact_p2_triangle(Pv):
    """Pv: 3 rational vertices in the plane.  Returns (M, A) exact."""
    Pv = [sp.Matrix(p) for p in Pv]
    mids = [(Pv[0] + Pv[1]) / 2, (Pv[1] + Pv[2]) / 2, (Pv[2] + Pv[0]) / 2]
    nodes = [tuple(p) for p in Pv + mids]
    monos = [sp.Integer(1), x, y, x * x, x * y, y * y]
    phi = _lagrange_basis(nodes, monos, (x, y))
    # integrate over the triangle: parametrise x = P0 + s(P1-P0) + t(P2-P0)
    s, t = sp.symbols("s t")
    e1, e2 = Pv[1] - Pv[0], Pv[2] - Pv[0]
    jac = abs(e1[0] * e2[1] - e1[1] * e2[0])
    sub = {x: Pv[0][0] + s * e1[0] + t * e2[0], y: Pv[0][1] + s * e1[1] + t * e2[1]}

    def integ(f):
        g = sp.expand(f.subs(sub, simultaneous=True)) * jac
        return sp.integrate(sp.integrate(g, (t, 0, 1 - s)), (s, 0, 1))

    M = sp.zeros(6, 6)
    A = sp.zeros(6, 6)
    grads = [(sp.diff(p, x), sp.diff(p, y)) for p in phi]
    for a in range(6):
        for b in range(a, 6):
            M[a, b] = M[b, a] = integ(phi[a] * phi[b])
            A[a, b] = A[b, a] = integ(grads[a][0] * grads[b][0] + grads[a][1] * grads[b][1])
    return np.array(M, dtype=float), np.array(A, dtype=float)


def test_p2_flat_triangle_exact_sympy():
    Pv = [(sp.Rational(0), sp.Rational(0)), (sp.Rational(3, 2), sp.Rational(1, 4)),
          (sp.Rational(1, 3), sp.Rational(5, 4))]
    Mex, Aex = _exact_p2_triangle(Pv)
    # embed in 3-D, rotate + translate (rigid motion: values unchanged)
    R = rot(5)
    P3 = np.array([[float(a), float(b), 0.0] for a, b in Pv])
    mids = np.array([(P3[0] + P3[1]) / 2, (P3[1] + P3[2]) / 2, (P3[2] + P3[0]) / 2])
    X = np.concatenate([P3, mids]) @ R.T + np.array([0.3, -1.2, 2.0])
    M, A, Aa = oracle.element_matrices(SURFACE_TRI, 2, QUAD_TRI6_DEG4, X, np.zeros(6))
    assert rel(M, Mex) < 1e-14
    assert rel(A, Aex) < 1e-13
    assert rel(Aa, A) < 1e-15  # u == 0  =>  A_a = A
    # closed form M = (area/180) K6 (consistent with sympy)
    area = 0.5 * abs(float((Pv[1][0] - Pv[0][0]) * (Pv[2][1] - Pv[0][1]) - (Pv[1][1] - Pv[0][1]) * (Pv[2][0] - Pv[0][0])))
    K6 = np.array([[6, -1, -1, 0, -4, 0], [-1, 6, -1, 0, 0, -4], [-1, -1, 6, -4, 0, 0],
                   [0, 0, -4, 32, 16, 16], [-4, 0, 0, 16, 32, 16], [0, -4, 0, 16, 16, 32]], float)
    assert rel(M, area / 180.0 * K6) < 1e-14


def _exact_p2_tet(Pv):
    Pv = [sp.Matrix(p) for p in Pv]
    pairs = [(0, 1), (1, 2), (2, 0), (0, 3), (1, 3), (2, 3)]
    nodes = [tuple(p) for p in Pv] + [tuple((Pv[i] + Pv[j]) / 2) for i, j in pairs]
    monos = [sp.Integer(1), x, y, z, x * x, y * y, z * z, x * y, y * z, x * z]
    phi = _lagrange_basis(nodes, monos, (x, y, z))
    r, s, t = sp.symbols("r s t")
    e = [Pv[1] - Pv[0], Pv[2] - Pv[0], Pv[3] - Pv[0]]
    jac = abs(sp.Matrix.hstack(*e).det())
    sub = {v: Pv[0][i] + r * e[0][i] + s * e[1][i] + t * e[2][i] for i, v in enumerate((x, y, z))}

    def integ(f):
        g = sp.Poly(sp.expand(f.subs(sub, simultaneous=True)), r, s, t)
        tot = sp.Integer(0)
        for (a, b, c), coef in g.terms():
            tot += coef * sp.factorial(a) * sp.factorial(b) * sp.factorial(c) / sp.factorial(a + b + c + 3)
        return tot * jac

    M = sp.zeros(10, 10)
    A = sp.zeros(10, 10)
    grads = [[sp.diff(p, v) for v in (x, y, z)] for p in phi]
    for a in range(10):
        for b in range(a, 10):
            M[a, b] = M[b, a] = integ(phi[a] * phi[b])
            A[a, b] = A[b, a] = integ(sum(grads[a][k] * grads[b][k] for k in range(3)))
    return np.array(M, dtype=float), np.array(A, dtype=float), float(jac) / 6.0


@pytest.mark.parametrize("quad", [QUAD_TET11_DEG4, 8], ids=["keast11", "deg7_35"])
def test_p2_flat_tet_exact_sympy(quad):
    """Affine P2 tet: M (degree 4) and A (degree 2) are integrated exactly by the 11-point
    degree-4 rule and by the 35-point degree-7 rule (reading G39) alike."""
    Pv = [(0, 0, 0), (sp.Rational(5, 4), sp.Rational(1, 8), 0), (sp.Rational(1, 4), 1, sp.Rational(1, 8)),
          (sp.Rational(1, 8), sp.Rational(1, 4), sp.Rational(9, 8))]
    Mex, Aex, V = _exact_p2_tet(Pv)
    P = np.array([[float(c) for c in p] for p in Pv])
    pairs = [(0, 1), (1, 2), (2, 0), (0, 3), (1, 3), (2, 3)]
    X = np.concatenate([P, np.array([(P[i] + P[j]) / 2 for i, j in pairs])])
    M, A, _ = oracle.element_matrices(BULK_TET, 2, quad, X)
    assert rel(M, Mex) < 1e-13
    assert rel(A, Aex) < 1e-13
    K10 = np.array([[6, 1, 1, 1, -4, -6, -4, -4, -6, -6], [1, 6, 1, 1, -4, -4, -6, -6, -4, -6],
                    [1, 1, 6, 1, -6, -4, -4, -6, -6, -4], [1, 1, 1, 6, -6, -6, -6, -4, -4, -4],
                    [-4, -4, -6, -6, 32, 16, 16, 16, 16, 8], [-6, -4, -4, -6, 16, 32, 16, 8, 16, 16],
                    [-4, -6, -4, -6, 16, 16, 32, 16, 8, 16], [-4, -6, -6, -4, 16, 8, 16, 32, 16, 16],
                    [-6, -4, -6, -4, 16, 16, 8, 16, 32, 16], [-6, -6, -4, -4, 8, 16, 16, 16, 16, 32]], float)
    assert rel(M, V / 420.0 * K10) < 1e-13


# ------------------------------------------------------------------ invariances
def _curved_p2_tri(seed):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((3, 3))
    v /= np.linalg.norm(v, axis=1)[:, None]
    v = 0.3 * v + np.array([0, 0, 1.0])
    v /= np.linalg.norm(v, axis=1)[:, None]
    m = np.array([(v[0] + v[1]) / 2, (v[1] + v[2]) / 2, (v[2] + v[0]) / 2])
    m /= np.linalg.norm(m, axis=1)[:, None]
    return np.concatenate([v, m])


def _curved_p2_tet(seed):
    rng = np.random.default_rng(seed)
    P = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float) + 0.1 * rng.standard_normal((4, 3))
    pairs = [(0, 1), (1, 2), (2, 0), (0, 3), (1, 3), (2, 3)]
    mid = np.array([(P[i] + P[j]) / 2 for i, j in pairs]) + 0.03 * rng.standard_normal((6, 3))
    return np.concatenate([P, mid])


@pytest.mark.parametrize("kind", ["tri2", "tet2"])
def test_rigid_motion_and_scaling(kind):
    X = _curved_p2_tri(3) if kind == "tri2" else _curved_p2_tet(3)
    dom, quad, d = (SURFACE_TRI, QUAD_TRI6_DEG4, 2) if kind == "tri2" else (BULK_TET, QUAD_TET11_DEG4, 3)
    u = np.random.default_rng(9).standard_normal(X.shape[0])
    M, A, Aa = oracle.element_matrices(dom, 2, quad, X, u)
    Y = X @ rot(11).T + np.array([5.0, -3.0, 1.0])
    M2, A2, Aa2 = oracle.element_matrices(dom, 2, quad, Y, u)
    assert rel(M2, M) < 1e-13 and rel(A2, A) < 1e-12 and rel(Aa2, Aa) < 1e-12
    s = 2.5
    M3, A3, _ = oracle.element_matrices(dom, 2, quad, s * X, u)
    assert rel(M3, M * s ** d) < 1e-13 and rel(A3, A * s ** (d - 2)) < 1e-12


def test_cyclic_relabelling_p2_triangle():
    """Relabel vertices (1,2,3) -> (2,3,1) with edges (12,23,31) -> (23,31,12):
    local matrices permute accordingly (symmetric rule; tests G1/G26)."""
    X = _curved_p2_tri(4)
    u = np.random.default_rng(2).standard_normal(6)
    perm = [1, 2, 0, 4, 5, 3]
    M, A, Aa = oracle.element_matrices(SURFACE_TRI, 2, QUAD_TRI6_DEG4, X, u)
    Mp, Ap, Aap = oracle.element_matrices(SURFACE_TRI, 2, QUAD_TRI6_DEG4, X[perm], u[perm])
    P = np.ix_(perm, perm)
    # a wrong edge order or vertex basis gives O(1) differences
    assert rel(Mp, M[P]) < 1e-12 and rel(Ap, A[P]) < 1e-12 and rel(Aap, Aa[P]) < 1e-12


def test_cyclic_relabelling_p2_tet():
    """Even permutation of the tet vertices (1,2,3) -> (2,3,1), 4 fixed; edges
    (12,23,31,14,24,34) -> (23,31,12,24,34,14)."""
    X = _curved_p2_tet(5)
    perm = [1, 2, 0, 3, 5, 6, 4, 8, 9, 7]
    M, A, _ = oracle.element_matrices(BULK_TET, 2, QUAD_TET11_DEG4, X)
    Mp, Ap, _ = oracle.element_matrices(BULK_TET, 2, QUAD_TET11_DEG4, X[perm])
    P = np.ix_(perm, perm)
    assert rel(Mp, M[P]) < 1e-13 and rel(Ap, A[P]) < 1e-12


@pytest.mark.parametrize("seed", range(4))
def test_listing1_formulation_agrees(seed):
    """Reading G2: Listing 1 builds L from COLUMNS [t1 t2 t1xt2] and uses
    C^T grad; that equals J G^{-1} grad (our metric form)."""
    X = _curved_p2_tri(20 + seed)
    u = np.random.default_rng(seed).standard_normal(6)
    a = oracle.element_matrices(SURFACE_TRI, 2, QUAD_TRI6_DEG4, X, u, formulation=0)
    b = oracle.element_matrices(SURFACE_TRI, 2, QUAD_TRI6_DEG4, X, u, formulation=1)
    for m0, m1 in zip(a, b):
        assert rel(m0, m1) < 1e-13


def test_degenerate_element_rejected():
    X = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float)  # collinear
    with pytest.raises(oracle.OracleError) as ei:
        oracle.element_matrices(SURFACE_TRI, 1, QUAD_TRI3_DEG2, X)
    assert ei.value.code == 4
