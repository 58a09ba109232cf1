"""Pins for the oracle's curve family (Table 4 "surface 1D",
P:646-660): P1/P2 line elements in R^3, Gauss-Legendre rules.

* Rules: exact for xi^k up to degree 3 (2 points) / 5 (3 points), not beyond.
* Straight segments: the textbook element matrices, P1 M = L/6 [2 1; 1 2], A = 1/L [1 -1; -1 1];
  P2 (nodes 1, 2, midpoint) M = L/30 [4 -1 2; -1 4 2; 2 2 16], A = 1/(3L) [7 1 -8; 1 7 -8; -8 -8 16].
* Circle: 1^T M 1 = length; P1: the inscribed polygon 2 n sin(pi/n) exactly; P2 -> 2 pi with EOC 4.
* Kernel A 1 = 0 and the trace identity sum_k x_k^T A x_k = 1^T M 1 (tr P = 1 on curves), which
  pins the tangential gradient t |t|^-2 dphi.
"""
import math

import numpy as np
import pytest

import lfem_inputs as li
import oracle


@pytest.mark.parametrize("quad,deg,npts", [(li.QUAD_LINE2_DEG3, 3, 2), (li.QUAD_LINE3_DEG5, 5, 3),
                                            (li.QUAD_LINE6_DEG11, 11, 6)])
def test_gauss_rules(quad, deg, npts):
    lam, w = oracle.rule(quad)
    assert lam.shape[0] == npts and abs(w.sum() - 1.0) < 1e-15
    xi = lam[:, 1]
    for k in range(deg + 1):
        assert abs(np.sum(w * xi ** k) - 1.0 / (k + 1)) < 1e-15
    assert abs(np.sum(w * xi ** (deg + 1)) - 1.0 / (deg + 2)) > 1e-9


@pytest.mark.parametrize("order", [1, 2])
def test_straight_segment_closed_forms(order):
    p0, p1 = np.array([0.3, -0.2, 0.5]), np.array([1.1, 0.7, -0.4])
    L = np.linalg.norm(p1 - p0)
    X = np.array([p0, p1]) if order == 1 else np.array([p0, p1, 0.5 * (p0 + p1)])
    M, A, _ = oracle.element_matrices(li.SURFACE_LINE, order, li.QUAD_DEFAULT, X)
    if order == 1:
        Me = L / 6 * np.array([[2, 1], [1, 2]])
        Ae = 1 / L * np.array([[1, -1], [-1, 1]])
    else:
        Me = L / 30 * np.array([[4, -1, 2], [-1, 4, 2], [2, 2, 16]])
        Ae = 1 / (3 * L) * np.array([[7, 1, -8], [1, 7, -8], [-8, -8, 16]])
    assert np.allclose(M, Me, rtol=1e-14, atol=1e-15)
    assert np.allclose(A, Ae, rtol=1e-14, atol=1e-14)


def _dense(m, kind):
    c = oracle.assemble_rows(m, ("M", "A"))
    return oracle.to_dense(c, m.n_nodes, kind)


@pytest.mark.parametrize("n", [5, 16, 64])
def test_circle_p1_polygon_length(n):
    m = li.circle_mesh(n, 1)
    M, A = _dense(m, "M"), _dense(m, "A")
    assert abs(M.sum() - 2 * n * math.sin(math.pi / n)) < 1e-13
    assert np.max(np.abs(A.sum(axis=1))) < 1e-12 * np.max(np.abs(A))
    tr = sum(m.coords[:, k] @ A @ m.coords[:, k] for k in range(3))
    assert abs(tr - M.sum()) < 1e-12 * M.sum()


@pytest.mark.parametrize("quad", [li.QUAD_LINE3_DEG5, li.QUAD_LINE6_DEG11], ids=["gauss3", "gauss6"])
def test_circle_p2_length_eoc_and_trace(quad):
    errs = []
    for n in (8, 16, 32):
        m = li.circle_mesh(n, 2)
        m.quad = quad
        M, A = _dense(m, "M"), _dense(m, "A")
        errs.append(abs(M.sum() - 2 * math.pi))
        assert np.max(np.abs(A.sum(axis=1))) < 1e-11 * np.max(np.abs(A))
        tr = sum(m.coords[:, k] @ A @ m.coords[:, k] for k in range(3))
        # curved P2: the trace identity holds for the discrete curve's own tangent, up to rounding
        assert abs(tr - M.sum()) < 1e-11 * M.sum()
    eoc = np.log2(errs[0] / errs[1]), np.log2(errs[1] / errs[2])
    assert all(3.5 < e < 4.5 for e in eoc), eoc


def test_curve_load_vector_is_M_f():
    m = li.circle_mesh(12, 2)
    f = li.random_field(m, 3)
    b = oracle.assemble_rhs_rows(m, f[None, :], "load")[0]
    assert np.allclose(b, _dense(m, "M") @ f, rtol=0, atol=1e-14)
    with pytest.raises(oracle.OracleError):
        oracle.assemble_rhs_rows(m, np.ones((4, m.n_nodes)), "kll")
