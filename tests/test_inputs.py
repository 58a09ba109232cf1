"""Tests of the shared seeded input generators (lfem_inputs).

These pin the INPUT recipe, not the method: counts of the
BASELINE.json configs, the RNG stream, the spherical-harmonic basis, the
Hilbert curve, and bitwise agreement of the compiled and numpy paths.
"""
import math

import numpy as np
import pytest

import lfem_inputs as li


def test_splitmix64_reference_values():
    # splitmix64 from state 0: first outputs (public reference values of the generator)
    r = li.SplitMix64(0)
    v = r.next_u64(3)
    assert [int(x) for x in v] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    # streaming in pieces == one call
    a = li.SplitMix64(42).uniform(10)
    r2 = li.SplitMix64(42)
    b = np.concatenate([r2.uniform(3), r2.uniform(7)])
    assert np.array_equal(a, b)
    assert np.all((a >= 0) & (a < 1))


def test_normals_moments():
    z = li.SplitMix64(1).normal(200000)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01


@pytest.mark.parametrize("L", range(5))
def test_icosphere_counts(L):
    v, f = li.icosphere_p1(L)
    assert v.shape[0] == 10 * 4 ** L + 2 and f.shape[0] == 20 * 4 ** L
    assert np.abs(np.linalg.norm(v, axis=1) - 1).max() < 1e-15
    # outward orientation
    P = v[f]
    n = np.cross(P[:, 1] - P[:, 0], P[:, 2] - P[:, 0])
    assert np.all(np.einsum("ij,ij->i", n, P.mean(1)) > 0)
    nodes, conn = li.p2_from_p1_triangles(v, f, project_sphere=True)
    assert nodes.shape[0] == v.shape[0] + 30 * 4 ** L
    assert np.abs(np.linalg.norm(nodes, axis=1) - 1).max() < 1e-15


def test_config_sizes_small_and_baseline_formulas():
    # the recipes at reduced size; full sizes follow from the same formulas
    # (C1 642/1280, C2 655362/327680, C3 2621442/5242880, C4 7189057/5308416,
    #  C5 41943042/20971520 -- BASELINE.json configs)
    m1 = li.make_config("C1")
    assert (m1.n_nodes, m1.n_elems) == (642, 1280)
    r = np.linalg.norm(m1.coords, axis=1)
    assert r.min() >= 0.999 - 1e-15 and r.max() <= 1.001 + 1e-15
    assert 40 * 4 ** 7 + 2 == 655362 and 20 * 4 ** 7 == 327680          # C2: P2 nodes V+E
    assert 10 * 4 ** 9 + 2 == 2621442 and 20 * 4 ** 9 == 5242880        # C3: P1
    assert 40 * 4 ** 10 + 2 == 41943042 and 20 * 4 ** 10 == 20971520    # C5: P2
    assert 6 * 96 ** 3 == 5308416 and 193 ** 3 == 7189057
    m4 = li.make_config("C4", level_override=4)
    assert m4.n_elems == 6 * 4 ** 3 and m4.n_nodes == 9 ** 3
    m3 = li.make_config("C3", level_override=3)
    assert m3.coeff is not None and m3.extra["uB"].shape == (m3.n_nodes,)
    m5 = li.make_config("C5", level_override=2)
    assert m5.nref == 6 and m5.coeff.shape == (m5.n_nodes,)


def test_kuhn_positive_orientation_and_conformity():
    x, t = li.kuhn_cube(3, 2)
    P = x[t[:, :4]]
    det = np.linalg.det(np.stack([P[:, 1] - P[:, 0], P[:, 2] - P[:, 0], P[:, 3] - P[:, 0]], 1))
    assert np.all(det > 0)
    assert abs(det.sum() / 6 - 1.0) < 1e-14
    # edge nodes are the midpoints
    pairs = [(0, 1), (1, 2), (2, 0), (0, 3), (1, 3), (2, 3)]
    for k, (a, b) in enumerate(pairs):
        assert np.abs(x[t[:, 4 + k]] - 0.5 * (x[t[:, a]] + x[t[:, b]])).max() < 1e-15
    # every node used
    assert np.unique(t).size == x.shape[0]


def test_real_sh_orthonormal():
    # Gauss-Legendre in z x trapezoid in phi: exact for these polynomials
    zq, wz = np.polynomial.legendre.leggauss(12)
    nphi = 24
    phi = 2 * math.pi * np.arange(nphi) / nphi
    Z, PH = np.meshgrid(zq, phi, indexing="ij")
    W = (wz[:, None] * np.full(nphi, 2 * math.pi / nphi)[None, :]).ravel()
    s = np.sqrt(1 - Z ** 2)
    xyz = np.stack([s * np.cos(PH), s * np.sin(PH), Z], -1).reshape(-1, 3)
    Y = li.real_sh(xyz)
    G = (Y * W[:, None]).T @ Y
    assert np.abs(G - np.eye(25)).max() < 1e-13
    # Y_00 and Y_10 explicit
    assert np.allclose(Y[:, 0], 0.5 / math.sqrt(math.pi))
    assert np.allclose(Y[:, 2], math.sqrt(3 / (4 * math.pi)) * xyz[:, 2])
    # sh_field == Y @ c
    c = np.random.default_rng(0).standard_normal(25)
    assert np.abs(li.sh_field(xyz, c) - Y @ c).max() < 1e-13


def test_hilbert_curve_adjacency_and_fast_path():
    b = 3
    g = np.arange(2 ** b)
    P = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3).astype(float)
    lo, hi = np.zeros(3), np.full(3, 2 ** b - 1.0)
    k = li.hilbert_keys_np(P, lo, hi, bits=b)
    assert np.array_equal(np.sort(k), np.arange(8 ** b, dtype=np.uint64))
    order = np.argsort(k)
    steps = np.abs(np.diff(P[order], axis=0)).sum(1)
    assert np.all(steps == 1.0)  # consecutive cells are face neighbours
    k2 = li.hilbert_keys(P, lo, hi, bits=b)
    assert np.array_equal(k, k2)
    rng = np.random.default_rng(3)
    Q = rng.standard_normal((5000, 3))
    assert np.array_equal(li.hilbert_keys(Q, Q.min(0), Q.max(0)), li.hilbert_keys_np(Q, Q.min(0), Q.max(0)))
    c = rng.standard_normal(25)
    assert np.array_equal(li.sh_field(Q, c), li.sh_field(Q, c, use_fast=False))


def test_configs_deterministic():
    a = li.make_config("C3", level_override=3)
    b = li.make_config("C3", level_override=3)
    assert np.array_equal(a.coords, b.coords) and np.array_equal(a.conn, b.conn)
    assert np.array_equal(a.coeff, b.coeff)


def test_c4p1_recipe():
    """N2 "P1 tets at scale": C4's displaced Kuhn cube with P1 tetrahedra and the 4-point rule."""
    m = li.make_config("C4P1", level_override=3)
    assert m.domain == li.BULK_TET and m.order == 1 and m.quad == li.QUAD_TET4_DEG2
    assert m.n_elems == 6 * 27 and m.n_nodes == 64 and m.extra["kinds"] == ("M", "A")
    m2 = li.make_config("C4P1", level_override=3)
    assert np.array_equal(m.coords, m2.coords) and np.array_equal(m.conn, m2.conn)
