"""Pins for the oracle's right-hand sides: the load
vector b and the KLL nonlinear right-hand side f = (f_1; f_2)
(Listing 2).  Every pin comes from the paper or the mathematics,
not from the oracle itself:

* b = M f  (f_h = sum f_j phi_j, the element rule integrates both the
  same way), checked against the oracle's *matrix* path (a different code
  path: std::map CSR of M, then a plain SpMV) on curved P2 spheres, P1
  spheres and displaced P1/P2 cubes.
* f == 1: sum_j b_j = |Gamma_h| -- on the paper's Tables 1-2 mesh
  (tests/golden/table12.json) this is 1 + (4/3)(sqrt2 - 1) exactly; on a
  straight planar square mesh it is 1, on the Kuhn cube the volume 1.
* KLL with nu_h = x_h (nodal positions): the tangential gradient of the
  identity on Gamma_h is the tangential projector P_h, |P_h|_F^2 = 2 at
  every point of any surface mesh, so f_{1,k} = 2 M x_k and f_2 = 2 M H.
* KLL with nu = B x on a (tilted) plane with unit normal n: grad nu_h = B P,
  alpha^2 = |B|_F^2 - |B n|^2 (constant), so f = alpha^2 M u.  |B P|_F and
  |B^T P|_F differ for a generic B, so a transposed gradient fails.
* nu constant  =>  alpha = 0  =>  f = 0.
* The Listing 1 gradient formulation (L^{-T}[grad; 0], reading G2) gives the
  same local vectors as the north star's J G^{-1} grad.
* Row subsets and thread counts do not change a single bit.
"""
import json
import math
import os

import numpy as np
import pytest

import lfem_inputs as li
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def csr_spmv(c, kind, x):
    rows = np.repeat(np.arange(c.rows.size), np.diff(c.row_ptr))
    return np.bincount(rows, weights=c.vals[kind] * x[c.col_idx], minlength=c.rows.size)


def csr_abs_spmv(c, kind, x):
    rows = np.repeat(np.arange(c.rows.size), np.diff(c.row_ptr))
    return np.bincount(rows, weights=np.abs(c.vals[kind] * x[c.col_idx]), minlength=c.rows.size)


def plane_mesh(n: int, order: int) -> li.Mesh:
    """Unit square [0,1]^2 at z = 0, n x n cells, two straight triangles each."""
    g = np.linspace(0.0, 1.0, n + 1)
    X, Y = np.meshgrid(g, g, indexing="ij")
    v = np.stack([X.ravel(), Y.ravel(), np.zeros(X.size)], axis=1)
    idx = lambda i, j: i * (n + 1) + j  # noqa: E731
    f = []
    for i in range(n):
        for j in range(n):
            f.append([idx(i, j), idx(i + 1, j), idx(i + 1, j + 1)])
            f.append([idx(i, j), idx(i + 1, j + 1), idx(i, j + 1)])
    f = np.array(f, dtype=np.int32)
    if order == 1:
        return li._finish(li.Mesh(li.SURFACE_TRI, 1, v, f, li.QUAD_TRI3_DEG2))
    v2, f2 = li.p2_from_p1_triangles(v, f, project_sphere=False)
    return li._finish(li.Mesh(li.SURFACE_TRI, 2, v2, f2, li.QUAD_TRI6_DEG4))


def rotation(seed: int) -> np.ndarray:
    q, r = np.linalg.qr(li.SplitMix64(seed).normal(9).reshape(3, 3))
    return q * np.sign(np.diag(r))[None, :]


def rotated(m: li.Mesh, R: np.ndarray) -> li.Mesh:
    return li._finish(li.Mesh(m.domain, m.order, m.coords @ R.T, m.conn.copy(), m.quad))


LOAD_MESHES = {
    "sphere_p1_L2": lambda: li.sphere_mesh(2, 1),
    "sphere_p2_L1": lambda: li.sphere_mesh(1, 2),
    "sphere_p2_L1_perturbed": lambda: li.perturb(li.sphere_mesh(1, 2), 5, 0.02),
    "cube_p1_n3_displaced": lambda: li.cube_mesh(3, 1, displace_seed=3),
    "cube_p2_n2_displaced": lambda: li.cube_mesh(2, 2, displace_seed=4),
}


# ------------------------------------------------------------------ load vector
@pytest.mark.parametrize("name", sorted(LOAD_MESHES))
def test_load_equals_mass_times_f(name):
    """b = M f (same rule on both sides), via the oracle's matrix path."""
    m = LOAD_MESHES[name]()
    f = li.random_field(m, 11)
    b, babs = oracle.assemble_rhs_rows(m, f[None, :], "load", with_abs=True)
    c = oracle.assemble_rows(m, ("M",))
    ref = csr_spmv(c, "M", f)
    scale = csr_abs_spmv(c, "M", f)
    assert b.shape == (1, m.n_nodes)
    assert np.all(np.abs(b[0] - ref) <= 1e-13 * scale + 1e-300)
    # the abs accumulator bounds the value and is itself a sum of |M_loc f_loc| terms
    assert np.all(np.abs(b[0]) <= babs[0] * (1 + 1e-15))
    assert np.all(babs[0] >= 0)


def test_load_constant_table12_golden():
    """f == 1 on the paper's Tables 1-2 mesh: sum b = 1 + (4/3)(sqrt2 - 1)."""
    g = json.load(open(os.path.join(GOLD, "table12.json")))
    assert g["total_mass"] == "1 + (4/3)(sqrt(2) - 1)"
    m = li.table12_mesh()
    b = oracle.assemble_rhs_rows(m, np.ones((1, m.n_nodes)), "load")
    assert abs(b.sum() - (1.0 + 4.0 / 3.0 * (math.sqrt(2.0) - 1.0))) < 1e-14


@pytest.mark.parametrize("order", [1, 2])
def test_load_constant_area_volume(order):
    """f == 1: sum_j b_j = area of the straight unit square / volume of the cube."""
    m = rotated(plane_mesh(4, order), rotation(2))
    b = oracle.assemble_rhs_rows(m, np.ones((1, m.n_nodes)), "load")
    assert abs(b.sum() - 1.0) < 1e-14
    c = li.cube_mesh(2, order, displace_seed=9)  # displacement preserves the volume (G16)
    bc = oracle.assemble_rhs_rows(c, np.ones((1, c.n_nodes)), "load")
    assert abs(bc.sum() - 1.0) < 1e-13


def test_load_linear_field_p1_closed_form():
    """P1 straight triangle, f linear: b_a = |T|/12 (2 f_a + sum_{c != a} f_c) (exact)."""
    p = np.array([[0.1, 0.2, 0.3], [1.3, -0.2, 0.5], [0.4, 0.9, -0.6]])
    m = li.single_triangle(p, 1)
    f = np.array([0.7, -1.1, 2.3])
    b = oracle.assemble_rhs_rows(m, f[None, :], "load")[0]
    area = 0.5 * np.linalg.norm(np.cross(p[1] - p[0], p[2] - p[0]))
    expect = area / 12.0 * (f + f.sum())
    assert np.allclose(b, expect, rtol=1e-14, atol=0)


# ------------------------------------------------------------------ KLL right-hand side
@pytest.mark.parametrize("mk", [lambda: li.sphere_mesh(1, 2), lambda: li.perturb(li.sphere_mesh(1, 2), 7, 0.03),
                                lambda: li.sphere_mesh(2, 1)], ids=["p2", "p2_perturbed", "p1"])
def test_kll_identity_field_alpha2_is_2(mk):
    """nu_h = x_h: grad_Gamma_h x_h = P_h, |P_h|_F^2 = 2 => f_1k = 2 M x_k, f_2 = 2 M H."""
    m = mk()
    H = li.random_field(m, 21)
    u = np.vstack([m.coords.T, H[None, :]])
    f, fabs = oracle.assemble_rhs_rows(m, u, "kll", with_abs=True)
    c = oracle.assemble_rows(m, ("M",))
    for k in range(4):
        ref = 2.0 * csr_spmv(c, "M", u[k])
        scale = 2.0 * csr_abs_spmv(c, "M", u[k])
        assert np.all(np.abs(f[k] - ref) <= 1e-12 * scale + 1e-300), k
        assert np.all(np.abs(f[k]) <= fabs[k] * (1 + 1e-15))


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("tilt", [False, True])
def test_kll_linear_field_on_plane(order, tilt):
    """nu = B x on a plane with normal n: alpha^2 = |B|_F^2 - |B n|^2, f = alpha^2 M u."""
    m = plane_mesh(3, order)
    n = np.array([0.0, 0.0, 1.0])
    if tilt:
        R = rotation(5)
        m = rotated(m, R)
        n = R @ n
    B = li.SplitMix64(8).normal(9).reshape(3, 3)
    H = li.random_field(m, 4)
    u = np.vstack([(m.coords @ B.T).T, H[None, :]])
    f = oracle.assemble_rhs_rows(m, u, "kll")
    alpha2 = np.sum(B * B) - np.dot(B @ n, B @ n)
    wrong = np.sum(B * B) - np.dot(B.T @ n, B.T @ n)  # the transposed gradient's value
    assert abs(alpha2 - wrong) > 0.1 * alpha2
    c = oracle.assemble_rows(m, ("M",))
    for k in range(4):
        ref = alpha2 * csr_spmv(c, "M", u[k])
        scale = alpha2 * csr_abs_spmv(c, "M", u[k])
        assert np.all(np.abs(f[k] - ref) <= 1e-12 * scale + 1e-300), k


def test_kll_table12_linear_field():
    """The paper's Tables 1-2 mesh (flat, curved P2 edges): same closed form."""
    m = li.table12_mesh()
    B = np.array([[1.0, 2.0, 3.0], [-1.0, 0.5, 4.0], [0.0, -2.0, 1.0]])
    u = np.vstack([(m.coords @ B.T).T, np.ones((1, m.n_nodes))])
    f = oracle.assemble_rhs_rows(m, u, "kll")
    alpha2 = np.sum(B[:, :2] ** 2)  # n = e_z
    area = 1.0 + 4.0 / 3.0 * (math.sqrt(2.0) - 1.0)
    assert abs(f[3].sum() - alpha2 * area) < 1e-12 * alpha2 * area


def test_kll_constant_nu_gives_zero():
    m = li.perturb(li.sphere_mesh(1, 2), 3, 0.02)
    u = np.vstack([np.full((3, m.n_nodes), 0.3), li.random_field(m, 2)[None, :]])
    u[1] = -0.8
    f = oracle.assemble_rhs_rows(m, u, "kll")
    assert np.max(np.abs(f)) < 1e-25


@pytest.mark.parametrize("order", [1, 2])
def test_kll_listing1_formulation_agrees(order):
    """Reading G2: g = L^{-T}[grad; 0] (Listing 1) == J G^{-1} grad (north star)."""
    rng = li.SplitMix64(40 + order)
    m = li.perturb(li.sphere_mesh(0, order), 6, 0.05)
    for e in range(m.n_elems):
        X = m.coords[m.conn[e]]
        U = 2.0 * rng.uniform(4 * m.nref).reshape(m.nref, 4) - 1.0
        f0 = oracle.element_rhs(m.domain, m.order, m.quad, X, U, "kll", 0)
        f1 = oracle.element_rhs(m.domain, m.order, m.quad, X, U, "kll", 1)
        assert np.allclose(f0, f1, rtol=1e-11, atol=1e-13 * np.abs(f0).max())


def test_kll_element_p1_closed_form():
    """P1 straight triangle: grad nu_h constant, alpha^2 = sum_k |sum_c nu_ck g_c|^2 with
    g_c = n x e_c / (2|T|) (edge e_c opposite node c) -- the textbook P1 gradient."""
    p = np.array([[0.0, 0.0, 0.1], [1.2, 0.3, -0.2], [0.2, 0.8, 0.5]])
    rng = li.SplitMix64(77)
    U = 2.0 * rng.uniform(12).reshape(3, 4) - 1.0
    F = oracle.element_rhs(li.SURFACE_TRI, 1, li.QUAD_TRI3_DEG2, p, U, "kll")
    nrm = np.cross(p[1] - p[0], p[2] - p[0])
    area2 = np.linalg.norm(nrm)
    nh = nrm / area2
    g = [np.cross(nh, p[(c + 2) % 3] - p[(c + 1) % 3]) / area2 for c in range(3)]
    alpha2 = sum(np.dot(sum(U[c, k] * g[c] for c in range(3)), sum(U[c, k] * g[c] for c in range(3)))
                 for k in range(3))
    Mloc = area2 / 2.0 / 12.0 * (np.ones((3, 3)) + np.eye(3))  # exact P1 mass (deg-2 rule is exact)
    assert np.allclose(F, alpha2 * Mloc @ U, rtol=1e-13, atol=0)


# ------------------------------------------------------------------ invariances + errors
@pytest.mark.parametrize("kind", ["load", "kll"])
def test_rhs_rows_and_threads_bit_identical(kind):
    m = li.perturb(li.sphere_mesh(2, 2), 9, 0.01)
    nc = 1 if kind == "load" else 4
    u = np.vstack([li.random_field(m, 30 + k) for k in range(nc)])
    full = oracle.assemble_rhs_rows(m, u, kind, nthreads=1)
    full8 = oracle.assemble_rhs_rows(m, u, kind, nthreads=8)
    assert np.array_equal(full, full8)
    rows = np.arange(3, m.n_nodes, 7, dtype=np.int64)
    sub = oracle.assemble_rhs_rows(m, u, kind, rows=rows, nthreads=3)
    assert np.array_equal(sub, full[:, rows])


def test_rhs_errors():
    c = li.cube_mesh(1, 1)
    with pytest.raises(oracle.OracleError) as ei:
        oracle.assemble_rhs_rows(c, np.ones((4, c.n_nodes)), "kll")
    assert ei.value.code == 2
    m = li.sphere_mesh(0, 1)
    bad = li.Mesh(m.domain, m.order, m.coords, m.conn.copy(), m.quad)
    bad.conn[5, 1] = m.n_nodes
    with pytest.raises(oracle.OracleError) as ei:
        oracle.assemble_rhs_rows(bad, np.ones((1, m.n_nodes)), "load")
    assert ei.value.code == 3 and ei.value.elem == 5
    deg = li.Mesh(m.domain, m.order, m.coords.copy(), m.conn.copy(), m.quad)
    deg.coords[deg.conn[7, 2]] = deg.coords[deg.conn[7, 0]]
    with pytest.raises(oracle.OracleError) as ei:
        oracle.assemble_rhs_rows(deg, np.ones((1, m.n_nodes)), "load")
    assert ei.value.code == 4


def test_abs_scale_is_the_value_for_nonnegative_terms():
    """The tolerance scale (absolute-value evaluation, reading G33) equals the value when every
    term is nonnegative (P1, f > 0; KLL with nu = x on a flat P1 mesh, H > 0) and bounds it otherwise."""
    m = plane_mesh(3, 1)
    f = 1.0 + 0.5 * (li.random_field(m, 3) + 1.0)
    b, babs = oracle.assemble_rhs_rows(m, f[None, :], "load", with_abs=True)
    assert np.allclose(b, babs, rtol=1e-14, atol=0)
    m2 = li.sphere_mesh(1, 2)
    f2 = li.random_field(m2, 4)
    b2, babs2 = oracle.assemble_rhs_rows(m2, f2[None, :], "load", with_abs=True)
    assert np.all(babs2 >= np.abs(b2)) and np.any(babs2 > 2 * np.abs(b2))


def _kll_test_fields(m, seed):
    """The GPU parity tests' KLL fields (tests/test_gpu_rhs.py kll_fields)."""
    x = m.coords
    r = np.sqrt(np.einsum("ij,ij->i", x, x))
    nu = (x / r[:, None]).T + 0.05 * np.vstack([li.random_field(m, seed + k) for k in range(3)])
    H = 2.0 + 0.1 * li.random_field(m, seed + 3)
    return np.vstack([nu, H[None, :]])


@pytest.mark.parametrize("level", [3, 5])
def test_kll_tolerance_scale_is_tight(level):
    """Reading G33: the KLL scale is first order in the rounding of alpha^2 = sum_k |G_k|^2
    (alpha^2 + 2 sum_k |G_k| B_k, G_k from differences), not the square of a running bound.
    On the parity tests' fields the scale stays within ~10x of the value (median) and 100x
    (90th percentile), so a 1e-12 x scale gate is a 1e-11..1e-10 relative gate.  With nu = x
    (alpha^2 = 2 exactly) the scale/value ratio no longer grows like h^-2 with refinement."""
    m = li.make_config("C5", level_override=level)
    f, fa = oracle.assemble_rhs_rows(m, _kll_test_fields(m, 5), "kll", with_abs=True)
    nz = np.abs(f) > 0
    r = fa[nz] / np.abs(f[nz])
    assert np.all(fa >= np.abs(f))
    assert np.median(r) <= 15 and np.percentile(r, 90) <= 100, (np.median(r), np.percentile(r, 90))
    u = np.vstack([m.coords.T, li.random_field(m, 1)[None, :]])
    f, fa = oracle.assemble_rhs_rows(m, u, "kll", with_abs=True)
    nz = np.abs(f) > 0
    assert np.median(fa[nz] / np.abs(f[nz])) <= 15


def test_load_with_dunavant8_on_sphere():
    """The paper's load-vector rule (Dunavant degree 8): on flat P2 elements f_h phi_j has
    degree 4, so the 6-point and 16-point rules agree to rounding; on the curved sphere they differ
    by the rule error only (small), and the sum of b over f == 1 is the area to rule accuracy."""
    m6 = li.table12_mesh()
    m16 = li.Mesh(m6.domain, m6.order, m6.coords, m6.conn, li.QUAD_TRI16_DEG8)
    f = np.array([0.3, -1.0, 2.0, 0.5, 0.1, -0.7, 1.1, 0.0, 0.9])[None, :]
    b6 = oracle.assemble_rhs_rows(m6, f, "load")
    b16 = oracle.assemble_rhs_rows(m16, f, "load")
    # table12 has curved edges (nodes 6, 9 on the circle): only the sum over f == 1 is exact-polynomial
    s16 = oracle.assemble_rhs_rows(m16, np.ones((1, 9)), "load").sum()
    assert abs(s16 - (1.0 + 4.0 / 3.0 * (math.sqrt(2.0) - 1.0))) < 1e-14
    p = plane_mesh(2, 2)
    fp = li.random_field(p, 3)[None, :]
    a6 = oracle.assemble_rhs_rows(p, fp, "load")
    a16 = oracle.assemble_rhs_rows(li.Mesh(p.domain, 2, p.coords, p.conn, li.QUAD_TRI16_DEG8), fp, "load")
    assert np.allclose(a6, a16, rtol=0, atol=1e-15)
    s = li.sphere_mesh(2, 2)
    fs = li.random_field(s, 4)[None, :]
    c6 = oracle.assemble_rhs_rows(s, fs, "load")
    c16 = oracle.assemble_rhs_rows(li.Mesh(s.domain, 2, s.coords, s.conn, li.QUAD_TRI16_DEG8), fs, "load")
    assert 0 < np.max(np.abs(c6 - c16)) < 1e-3 * np.max(np.abs(c16))
    assert b6.shape == b16.shape
