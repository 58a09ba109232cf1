"""Pins for the oracle's global assembly (CSR) against what the paper and
mathematics fix.

* Golden: PAPER.md Tables 1-2 mesh (tests/golden/table12.json): nnz = 63,
  1^T M 1 = 1 + (4/3)(sqrt2 - 1) (exact), A 1 = 0, trace identity.
* Kernel of A: A 1 = 0, A_a 1 = 0 (BASELINE.json north_star).
* 1^T M 1 = quadrature area / volume; P1: exactly sum of triangle areas;
  Kuhn cube under the G16 displacement: volume 1.
* Trace identity sum_k x_k^T A x_k = 2 |Gamma_h| (surface) / 3 |Omega_h|
  (bulk), from tr P = dim (north_star) -- pins reading G2 (the literal
  transpose gives 4.197 instead of 2 on a skewed P2 sphere).
* Weighted trace identity sum_k x_k^T A_a x_k = 2 (1^T M 1 + u^T M u)
  (surface) since int a(u_h) = int 1 + u_h^2 with the same rule.
* Special cases u == c  =>  A_a = (1 + c^2) A.
* Convergence: icosphere area -> 4 pi with EOC 2 (P1) and 4 (P2).
* Pattern: nnz closed forms: P1 sphere V + 2E, P2 sphere
  V + 7E + 12F, P2 Kuhn 230n^3 + 138n^2 + 24n + 1, P1 Kuhn 15n^3+21n^2+9n+1;
  P2 sphere row lengths in {9, 16, 19}.
* Brute force: dense N x N accumulation of the Listing 1 formulation
  (second, independent gradient formula) on tiny meshes == the std::map CSR.
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


def dense(c, n, kind):
    return oracle.to_dense(c, n, kind)


def spmv(c, kind, x):
    y = np.zeros(c.rows.size)
    for i in range(c.rows.size):
        s, e = c.row_ptr[i], c.row_ptr[i + 1]
        y[i] = np.dot(c.vals[kind][s:e], x[c.col_idx[s:e]])
    return y


def csr_spmv(c, kind, x):
    vals = c.vals[kind]
    rows = np.repeat(np.arange(c.rows.size), np.diff(c.row_ptr))
    return np.bincount(rows, weights=vals * x[c.col_idx], minlength=c.rows.size)


# ------------------------------------------------------------------ golden
def test_table12_golden():
    g = json.load(open(os.path.join(GOLD, "table12.json")))
    m = li.table12_mesh()
    assert np.array_equal(m.conn + 1, np.array(g["elements_1based"]))
    c = oracle.assemble_rows(m, ("M", "A"))
    assert c.nnz == g["nnz"] == 63
    one = np.ones(m.n_nodes)
    mass = float(one @ csr_spmv(c, "M", one))
    assert abs(mass - (1 + 4.0 / 3.0 * (math.sqrt(2) - 1))) < 1e-15
    assert np.abs(csr_spmv(c, "A", one)).max() < 1e-14
    tr = sum(float(m.coords[:, k] @ csr_spmv(c, "A", m.coords[:, k])) for k in range(3))
    assert abs(tr - 2 * mass) < 1e-13


# ------------------------------------------------------------------ invariants
def _skewed_sphere(level, order, seed=3):
    m = li.sphere_mesh(level, order)
    return li.perturb(m, seed, 0.2 * 2.0 ** -level)


SURF_CASES = [("P1 L2", lambda: _skewed_sphere(2, 1)), ("P2 L2", lambda: _skewed_sphere(2, 2)),
              ("C3 shape L3", lambda: li.make_config("C3", level_override=3)),
              ("C5 shape L2", lambda: li.make_config("C5", level_override=2))]


@pytest.mark.parametrize("name,mk", SURF_CASES, ids=[c[0] for c in SURF_CASES])
def test_surface_invariants(name, mk):
    m = mk()
    u = m.coeff if m.coeff is not None else li.random_field(m, 5)
    c = oracle.assemble_rows(m, ("M", "A", "Aa"), coeff=u)
    one = np.ones(m.n_nodes)
    mass = float(one @ csr_spmv(c, "M", one))
    for k in ("A", "Aa"):
        rowmax = np.maximum.reduceat(np.abs(c.vals[k]), c.row_ptr[:-1])
        assert np.all(np.abs(csr_spmv(c, k, one)) <= 1e-12 * rowmax), k
    tr = sum(float(m.coords[:, k] @ csr_spmv(c, "A", m.coords[:, k])) for k in range(3))
    assert abs(tr / mass - 2.0) < 1e-12
    uMu = float(u @ csr_spmv(c, "M", u))
    tra = sum(float(m.coords[:, k] @ csr_spmv(c, "Aa", m.coords[:, k])) for k in range(3))
    assert abs(tra - 2.0 * (mass + uMu)) < 1e-12 * tra
    # symmetry
    D = dense(c, m.n_nodes, "A")
    assert np.abs(D - D.T).max() < 1e-13 * np.abs(D).max()
    if m.order == 1:
        P = m.coords[m.conn]
        area = 0.5 * np.linalg.norm(np.cross(P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]), axis=1).sum()
        assert abs(mass - area) < 1e-13 * area


def test_bulk_invariants_displaced_cube():
    m = li.make_config("C4", level_override=3)
    c = oracle.assemble_rows(m, ("M", "A", "Aa"), coeff=li.random_field(m, 1))
    one = np.ones(m.n_nodes)
    vol = float(one @ csr_spmv(c, "M", one))
    assert abs(vol - 1.0) < 1e-13  # G16: the displacement keeps |Omega_h| = 1
    rowmax = np.maximum.reduceat(np.abs(c.vals["A"]), c.row_ptr[:-1])
    assert np.all(np.abs(csr_spmv(c, "A", one)) <= 1e-12 * rowmax)
    tr = sum(float(m.coords[:, k] @ csr_spmv(c, "A", m.coords[:, k])) for k in range(3))
    assert abs(tr - 3.0 * vol) < 1e-12


def test_bulk_invariants_displaced_cube_deg7_rule():
    """Reading G39: with the 35-point degree-7 rule on curved P2 tets, det J (cubic) is integrated
    exactly, so 1^T M 1 = 1 (G16) again; the trace identity holds for any rule; and the rule
    differs from the 11-point one only at quadrature-error level on the curved elements."""
    m = li.make_config("C4", level_override=3)
    m7 = li.Mesh(m.domain, m.order, m.coords, m.conn, li.QUAD_TET35_DEG7)
    u = li.random_field(m, 1)
    c7 = oracle.assemble_rows(m7, ("M", "A", "Aa"), coeff=u)
    c4 = oracle.assemble_rows(m, ("M", "A", "Aa"), coeff=u)
    one = np.ones(m.n_nodes)
    vol = float(one @ csr_spmv(c7, "M", one))
    assert abs(vol - 1.0) < 1e-13
    rowmax = np.maximum.reduceat(np.abs(c7.vals["A"]), c7.row_ptr[:-1])
    assert np.all(np.abs(csr_spmv(c7, "A", one)) <= 1e-12 * rowmax)
    assert np.all(np.abs(csr_spmv(c7, "Aa", one)) <= 1e-12 * np.maximum.reduceat(np.abs(c7.vals["Aa"]), c7.row_ptr[:-1]))
    tr = sum(float(m.coords[:, k] @ csr_spmv(c7, "A", m.coords[:, k])) for k in range(3))
    assert abs(tr - 3.0 * vol) < 1e-12
    assert np.array_equal(c7.col_idx, c4.col_idx)
    d = np.abs(c7.vals["A"] - c4.vals["A"]).max() / np.abs(c4.vals["A"]).max()
    assert 1e-12 < d < 1e-2, d  # different rules, same integrand


def test_p1_tet_cube_volume_and_trace():
    m = li.cube_mesh(3, 1, displace_seed=4)
    c = oracle.assemble_rows(m, ("M", "A"))
    one = np.ones(m.n_nodes)
    vol = float(one @ csr_spmv(c, "M", one))
    P = m.coords[m.conn]
    V = np.abs(np.linalg.det(np.stack([P[:, 1] - P[:, 0], P[:, 2] - P[:, 0], P[:, 3] - P[:, 0]], 1))).sum() / 6
    assert abs(vol - V) < 1e-14 and abs(vol - 1.0) < 1e-13
    tr = sum(float(m.coords[:, k] @ csr_spmv(c, "A", m.coords[:, k])) for k in range(3))
    assert abs(tr - 3.0 * vol) < 1e-12


def test_constant_coefficient_special_case():
    m = _skewed_sphere(2, 2)
    cst = 0.7
    c = oracle.assemble_rows(m, ("A", "Aa"), coeff=np.full(m.n_nodes, cst))
    assert np.abs(c.vals["Aa"] - (1 + cst * cst) * c.vals["A"]).max() < 1e-14 * np.abs(c.vals["A"]).max()
    c0 = oracle.assemble_rows(m, ("A", "Aa"), coeff=np.zeros(m.n_nodes))
    assert np.array_equal(c0.vals["Aa"], c0.vals["A"])


# ------------------------------------------------------------------ convergence
@pytest.mark.parametrize("order,levels,eoc", [(1, (3, 4, 5, 6), 2.0), (2, (2, 3, 4, 5), 4.0)])
def test_sphere_area_convergence(order, levels, eoc):
    errs = []
    for L in levels:
        m = li.sphere_mesh(L, order)
        c = oracle.assemble_rows(m, ("M",))
        errs.append(abs(c.vals["M"].sum() - 4 * math.pi))
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert abs(rates[-1] - eoc) < 0.05, rates


def test_icosphere_area_anchors():
    """Cross-check with SURVEY.md App. B (independent 40-digit survey scripts):
    L3 P1 12.506492733969928, L2 P2 12.565174097177067."""
    c1 = oracle.assemble_rows(li.sphere_mesh(3, 1), ("M",))
    c2 = oracle.assemble_rows(li.sphere_mesh(2, 2), ("M",))
    assert abs(c1.vals["M"].sum() - 12.506492733969928) < 1e-12
    assert abs(c2.vals["M"].sum() - 12.565174097177067) < 1e-12


# ------------------------------------------------------------------ pattern
@pytest.mark.parametrize("L", [0, 1, 2, 3])
def test_sphere_pattern_counts(L):
    V, E, F = 10 * 4 ** L + 2, 30 * 4 ** L, 20 * 4 ** L
    c1 = oracle.assemble_rows(li.sphere_mesh(L, 1), ("M",))
    assert c1.nnz == V + 2 * E
    m2 = li.sphere_mesh(L, 2)
    c2 = oracle.assemble_rows(m2, ("M",))
    assert c2.nnz == V + 7 * E + 12 * F
    lens = np.diff(c2.row_ptr)
    assert set(np.unique(lens)) <= {9, 16, 19}
    assert np.count_nonzero(lens == 9) == E  # edge nodes


@pytest.mark.parametrize("n", [1, 2, 3])
def test_cube_pattern_counts(n):
    c2 = oracle.assemble_rows(li.cube_mesh(n, 2), ("M",))
    assert c2.nnz == 230 * n ** 3 + 138 * n ** 2 + 24 * n + 1
    c1 = oracle.assemble_rows(li.cube_mesh(n, 1), ("M",))
    assert c1.nnz == 15 * n ** 3 + 21 * n ** 2 + 9 * n + 1


def test_pattern_columns_ascending_and_explicit_zeros():
    m = li.table12_mesh()
    c = oracle.assemble_rows(m, ("M",))
    for i in range(m.n_nodes):
        cols = c.col_idx[c.row_ptr[i]:c.row_ptr[i + 1]]
        assert np.all(np.diff(cols) > 0)
    # G19: the pattern is structural -- a flat P2 triangle's mass has zero
    # entries (K6[0,3] = 0) that are still stored
    t = li.single_triangle([[0, 0, 0], [1, 0, 0], [0, 1, 0]], order=2)
    ct = oracle.assemble_rows(t, ("M",))
    assert ct.nnz == 36
    assert abs(ct.vals["M"][3]) < 1e-17 and ct.col_idx[3] == 3


# ------------------------------------------------------------------ brute force
@pytest.mark.parametrize("name,mk", [("P1 L1", lambda: _skewed_sphere(1, 1)),
                                      ("P2 L1", lambda: _skewed_sphere(1, 2)),
                                      ("table12", li.table12_mesh)])
def test_brute_force_dense_listing1(name, mk):
    m = mk()
    u = li.random_field(m, 8)
    n = m.n_nodes
    D = {k: np.zeros((n, n)) for k in ("M", "A", "Aa")}
    S = np.zeros((n, n), dtype=bool)
    for e in range(m.n_elems):
        idx = m.conn[e]
        Ml, Al, Aal = oracle.element_matrices(m.domain, m.order, m.quad, m.coords[idx], u[idx], formulation=1)
        for k, L in (("M", Ml), ("A", Al), ("Aa", Aal)):
            D[k][np.ix_(idx, idx)] += L
        S[np.ix_(idx, idx)] = True
    c = oracle.assemble_rows(m, ("M", "A", "Aa"), coeff=u)
    # pattern: exactly the structural pattern
    pat = np.zeros((n, n), dtype=bool)
    for i in range(n):
        pat[i, c.col_idx[c.row_ptr[i]:c.row_ptr[i + 1]]] = True
    assert np.array_equal(pat, S)
    for k in ("M", "A", "Aa"):
        got = dense(c, n, k)
        rowmax = np.abs(D[k]).max(axis=1)
        assert np.all(np.abs(got - D[k]).max(axis=1) <= 1e-13 * rowmax), k


# ------------------------------------------------------------------ determinism
def test_row_subsets_and_threads_bitwise():
    m = li.make_config("C5", level_override=3)
    full = oracle.assemble_rows(m, ("M", "A", "Aa"), nthreads=1)
    full8 = oracle.assemble_rows(m, ("M", "A", "Aa"), nthreads=8)
    for k in ("M", "A", "Aa"):
        assert np.array_equal(full.vals[k], full8.vals[k])
    rows = np.sort(np.random.default_rng(0).choice(m.n_nodes, 300, replace=False))
    sub = oracle.assemble_rows(m, ("M", "A", "Aa"), rows=rows)
    for j, r in enumerate(rows):
        a, b = full.row_ptr[r], full.row_ptr[r + 1]
        s, e = sub.row_ptr[j], sub.row_ptr[j + 1]
        assert np.array_equal(full.col_idx[a:b], sub.col_idx[s:e])
        for k in ("M", "A", "Aa"):
            assert np.array_equal(full.vals[k][a:b], sub.vals[k][s:e])


# ------------------------------------------------------------------ errors
def test_index_error_reports_lowest_element():
    m = li.sphere_mesh(1, 1)
    conn = m.conn.copy()
    conn[7, 1] = m.n_nodes + 3
    conn[11, 0] = -1
    bad = li.Mesh(m.domain, m.order, m.coords, conn, m.quad)
    with pytest.raises(oracle.OracleError) as ei:
        oracle.assemble_rows(bad, ("M",))
    assert ei.value.code == 3 and ei.value.elem == 7


def test_degenerate_error_reports_lowest_element():
    m = li.sphere_mesh(1, 1)
    X = m.coords.copy()
    # collapse elements 9 and 4: move one node onto another
    for e in (9, 4):
        X[m.conn[e, 2]] = X[m.conn[e, 1]]
    bad = li.Mesh(m.domain, m.order, X, m.conn, m.quad)
    with pytest.raises(oracle.OracleError) as ei:
        oracle.assemble_rows(bad, ("M",))
    assert ei.value.code == 4
    P = X[m.conn]
    area = 0.5 * np.linalg.norm(np.cross(P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]), axis=1)
    assert ei.value.elem == int(np.nonzero(area == 0.0)[0].min()) == 4


def test_missing_coefficient_rejected():
    m = li.sphere_mesh(0, 1)
    with pytest.raises(oracle.OracleError) as ei:
        oracle.assemble_rows(m, ("Aa",), coeff=None)
    assert ei.value.code == 1
