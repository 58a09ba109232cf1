"""GPU parity: the CUDA path (through the C-ABI liblfem.so) against the oracle.

Bar (BASELINE.json north_star): CSR pattern (row_ptr, col_idx) bit-exact;
every value within 1e-12 x the row's max |oracle entry|, fp64.  Sizes span
many tiles and ragged tails; full BASELINE.json sizes are checked on sampled
rows in test_gpu_fullsize.py.
"""
import numpy as np
import pytest
import torch

import lfem_inputs as li
import oracle
from gpu_common import TOL, check_full, compare_rows, gpu_assemble, sample_rows

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes only with -m gpu
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2605_14035_b200 import lfem  # noqa: E402

VARIANTS = [lfem.LFEM_NUMERIC_V0, lfem.LFEM_NUMERIC_TILED, lfem.LFEM_NUMERIC_AUTO, lfem.LFEM_NUMERIC_ROWS]


def _skew(m, seed, eps):
    return li.perturb(m, seed, eps)


def _q16(m):
    """The same mesh with Dunavant's 16-point degree-8 rule."""
    return li.Mesh(m.domain, m.order, m.coords, m.conn, li.QUAD_TRI16_DEG8, m.coeff)


def _q35(m):
    """The same P2 tet mesh with the 35-point degree-7 rule (the paper's degree-7 tet rule, reading G39)."""
    return li.Mesh(m.domain, m.order, m.coords, m.conn, li.QUAD_TET35_DEG7, m.coeff)


SMALL = [
    ("tri1_single", lambda: li.single_triangle([[0, 0, 0], [1, 0, 0], [0.2, 0.9, 0.3]], 1)),
    ("tri2_single", lambda: li.single_triangle([[0, 0, 0], [1, 0, 0], [0.2, 0.9, 0.3]], 2)),
    ("table12", li.table12_mesh),
    ("sphere1_L0", lambda: li.sphere_mesh(0, 1)),
    ("sphere2_L1_skew", lambda: _skew(li.sphere_mesh(1, 2), 1, 0.05)),
    ("sphere1_L4_skew", lambda: _skew(li.sphere_mesh(4, 1), 2, 0.005)),
    ("sphere2_L3_skew", lambda: _skew(li.sphere_mesh(3, 2), 3, 0.01)),
    ("sphere2_L4_natural", lambda: li.sphere_mesh(4, 2, sfc=False)),
    ("cube1_n3", lambda: li.cube_mesh(3, 1, displace_seed=1)),
    ("cube2_n1", lambda: li.cube_mesh(1, 2)),
    ("cube2_n4_disp", lambda: li.cube_mesh(4, 2, displace_seed=2)),
    ("C1", lambda: li.make_config("C1")),
    ("C3_L4", lambda: li.make_config("C3", level_override=4)),
    ("C4_n5", lambda: li.make_config("C4", level_override=5)),
    ("C4P1_n6", lambda: li.make_config("C4P1", level_override=6)),
    ("C5_L4", lambda: li.make_config("C5", level_override=4)),
    ("sphere2_L3_skew_q16", lambda: _q16(_skew(li.sphere_mesh(3, 2), 3, 0.01))),
    ("C5_L4_q16", lambda: _q16(li.make_config("C5", level_override=4))),
    ("cube2_n3_disp_q35", lambda: _q35(li.cube_mesh(3, 2, displace_seed=2))),
    ("C4_n4_q35", lambda: _q35(li.make_config("C4", level_override=4))),
]


@pytest.mark.parametrize("variant", VARIANTS, ids=["v0", "tiled", "auto", "rows"])
@pytest.mark.parametrize("name,mk", SMALL, ids=[s[0] for s in SMALL])
def test_parity_full(name, mk, variant):
    m = mk()
    u = m.coeff if m.coeff is not None else li.random_field(m, 11)
    if name.endswith("_q35") and variant == lfem.LFEM_NUMERIC_TILED:
        with pytest.raises(lfem.LfemError) as ei:  # no tile configuration for the 35-point rule
            gpu_assemble(m, ("M", "A", "Aa"), coeff=u, variant=variant)
        assert ei.value.status == 2
        return
    worst, _ = check_full(m, ("M", "A", "Aa"), coeff=u, variant=variant)
    assert worst <= TOL


@pytest.mark.parametrize("kinds", [("M",), ("A",), ("Aa",), ("M", "Aa"), ("A", "Aa"), ("M", "A")])
def test_kind_subsets(kinds):
    m = _skew(li.sphere_mesh(2, 2), 4, 0.02)
    u = li.random_field(m, 3)
    check_full(m, kinds, coeff=u)


def test_C2_full_parity():
    m = li.make_config("C2")
    worst, _ = check_full(m, ("M", "A"))
    assert worst <= TOL


def test_determinism_and_variant_bitwise():
    m = li.make_config("C5", level_override=5)
    outs = []
    for variant in (lfem.LFEM_NUMERIC_V0, lfem.LFEM_NUMERIC_TILED, lfem.LFEM_NUMERIC_AUTO, lfem.LFEM_NUMERIC_AUTO,
                    lfem.LFEM_NUMERIC_ROWS):
        _, rp, ci, vals = gpu_assemble(m, ("M", "A", "Aa"), variant=variant)
        outs.append(vals)
    for o in outs[1:]:
        for k in ("M", "A", "Aa"):
            assert np.array_equal(o[k], outs[0][k])


@pytest.mark.parametrize("nblocks", [2, 3, 8])
def test_row_block_partition_emulation(nblocks):
    """P row blocks assembled one after another reproduce the
    full assembly bitwise (the multi-GPU partition, emulated on one GPU)."""
    m = li.make_config("C5", level_override=4)
    _, rp, ci, vals = gpu_assemble(m, ("M", "A", "Aa"))
    bounds = np.linspace(0, m.n_nodes, nblocks + 1).astype(np.int64)
    for b in range(nblocks):
        r0, r1 = int(bounds[b]), int(bounds[b + 1])
        plan, brp, bci, bvals = gpu_assemble(m, ("M", "A", "Aa"), row_begin=r0, row_end=r1)
        assert plan.n_rows == r1 - r0
        s0, s1 = rp[r0], rp[r1]
        assert np.array_equal(brp, rp[r0:r1 + 1] - s0)
        assert np.array_equal(bci, ci[s0:s1])
        for k in ("M", "A", "Aa"):
            assert np.array_equal(bvals[k], vals[k][s0:s1])


def test_empty_and_degenerate_ranges():
    m = li.sphere_mesh(1, 2)
    plan, rp, ci, vals = gpu_assemble(m, ("M",), row_begin=5, row_end=5)
    assert plan.nnz == 0 and plan.n_rows == 0 and rp.tolist() == [0]
    # a mesh with no elements
    e = li.Mesh(li.SURFACE_TRI, 1, np.zeros((4, 3)), np.zeros((0, 3), np.int32), li.QUAD_TRI3_DEG2)
    plan, rp, ci, vals = gpu_assemble(e, ("M", "A"))
    assert plan.nnz == 0 and np.array_equal(rp, np.zeros(5, np.int64))


def test_moving_coords_and_host_entry_match():
    m = li.make_config("C5", level_override=3)
    plan, rp, ci, vals = gpu_assemble(m, ("M", "A", "Aa"))
    # moved geometry through lfem_assemble_numeric_coords == a fresh mesh at the moved coords
    moved = li.perturb(m, 9, 1e-3)
    X = torch.as_tensor(moved.coords, device="cuda")
    cf = torch.as_tensor(m.coeff, device="cuda")
    v = [torch.empty(plan.nnz, dtype=torch.float64, device="cuda") for _ in range(3)]
    lfem.lfem_assemble_numeric_coords(plan, 7, X, cf, v)
    lfem.lfem_plan_check(plan)
    o = oracle.assemble_rows(moved, ("M", "A", "Aa"), coeff=m.coeff)
    compare_rows(np.arange(m.n_nodes), rp, ci, {"M": v[0].cpu().numpy(), "A": v[1].cpu().numpy(),
                                                "Aa": v[2].cpu().numpy()}, o, ("M", "A", "Aa"))
    # host entry point (pinned buffers)
    hv = [torch.empty(plan.nnz, dtype=torch.float64, pin_memory=True) for _ in range(3)]
    lfem.lfem_assemble_numeric_host(plan, 7, torch.as_tensor(moved.coords).pin_memory(),
                                    torch.as_tensor(m.coeff).pin_memory(), hv)
    for k in range(3):
        assert torch.equal(hv[k], v[k].cpu())


def test_spmv_and_axpby():
    m = li.make_config("C3", level_override=4)
    plan, rp, ci, vals = gpu_assemble(m, ("M", "Aa"))
    x = torch.as_tensor(li.random_field(m, 2), device="cuda")
    y = torch.empty(plan.n_rows, dtype=torch.float64, device="cuda")
    lfem.lfem_spmv(plan, torch.as_tensor(vals["M"], device="cuda"), x, y)
    o = oracle.assemble_rows(m, ("M",))
    xr = x.cpu().numpy()
    rows = np.repeat(np.arange(m.n_nodes), np.diff(o.row_ptr))
    yo = np.bincount(rows, weights=o.vals["M"] * xr[o.col_idx], minlength=m.n_nodes)
    assert np.abs(y.cpu().numpy() - yo).max() <= 1e-13 * np.abs(yo).max()
    a = torch.as_tensor(m.extra["uA"], device="cuda")
    b = torch.as_tensor(m.extra["uB"], device="cuda")
    out = torch.empty_like(a)
    lfem.lfem_axpby(0.6, a, 0.8, b, out)
    assert torch.allclose(out, 0.6 * a + 0.8 * b, rtol=0, atol=1e-15)


# ---------------------------------------------------------------------------- errors
def test_index_error():
    m = li.sphere_mesh(1, 1)
    conn = m.conn.copy()
    conn[13, 2] = m.n_nodes
    conn[40, 0] = -7
    with pytest.raises(lfem.LfemError) as ei:
        lfem.lfem_mesh_create(0, 1, 0, torch.as_tensor(m.coords, device="cuda"), torch.as_tensor(conn, device="cuda"))
    assert ei.value.status == 3 and ei.value.element == 13


def test_degenerate_error():
    m = li.sphere_mesh(1, 1)
    X = m.coords.copy()
    for e in (30, 21):
        X[m.conn[e, 2]] = X[m.conn[e, 1]]
    P = X[m.conn]
    area = 0.5 * np.linalg.norm(np.cross(P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]), axis=1)
    bad = li.Mesh(m.domain, m.order, X, m.conn, m.quad)
    with pytest.raises(lfem.LfemError) as ei:
        gpu_assemble(bad, ("M", "A"))
    assert ei.value.status == 4 and ei.value.element == int(np.nonzero(area == 0)[0].min())
    with pytest.raises(oracle.OracleError) as eo:
        oracle.assemble_rows(bad, ("M",))
    assert eo.value.elem == ei.value.element


def test_argument_errors():
    m = li.sphere_mesh(0, 2)
    X = torch.as_tensor(m.coords, device="cuda")
    C = torch.as_tensor(m.conn, device="cuda")
    with pytest.raises(lfem.LfemError) as ei:  # tet rule on triangles
        lfem.lfem_mesh_create(0, 2, lfem.LFEM_QUAD_TET11_DEG4, X, C)
    assert ei.value.status == 2
    with pytest.raises(lfem.LfemError) as ei:
        lfem.lfem_mesh_create(0, 3, 0, X, C)
    assert ei.value.status == 2
    mh = lfem.lfem_mesh_create(0, 2, 0, X, C)
    plan = lfem.lfem_assemble_symbolic(mh)
    v = [torch.empty(plan.nnz, dtype=torch.float64, device="cuda") for _ in range(3)]
    with pytest.raises(lfem.LfemError) as ei:  # A_a without a coefficient
        lfem.lfem_assemble_numeric(plan, lfem.LFEM_STIFF_COEF, None, v)
    assert ei.value.status == 1
    with pytest.raises(lfem.LfemError) as ei:
        lfem.lfem_assemble_numeric(plan, 0, None, v)
    assert ei.value.status == 1
    with pytest.raises(lfem.LfemError) as ei:
        lfem.lfem_assemble_symbolic(mh, 5, 2)
    assert ei.value.status == 1


# ---------------------------------------------------------------------------- tile-plan edge cases
@pytest.mark.parametrize("budget", [8, 17, 64, 100])
@pytest.mark.parametrize("name,mk", [("P2tri", lambda: li.make_config("C5", level_override=3)),
                                     ("P1tri", lambda: li.make_config("C3", level_override=4)),
                                     ("P2tet", lambda: li.make_config("C4", level_override=3))],
                         ids=["P2tri", "P1tri", "P2tet"])
def test_tiled_small_budgets_bitwise(name, mk, budget, monkeypatch):
    """Tiny tile element budgets (LFEM_TILE_ELEMS): thousands of tiles with a
    handful of rows each, single-row tiles, halo-dominated tiles, ragged
    tails.  Values must be bitwise those of the default plan (summation
    order is the symbolic order, independent of tiling) and the oracle's
    within the gate."""
    m = mk()
    u = m.coeff if m.coeff is not None else li.random_field(m, 5)
    kinds = ("M", "A", "Aa")
    _, rp0, ci0, v0 = gpu_assemble(m, kinds, coeff=u, variant=lfem.LFEM_NUMERIC_V0)
    monkeypatch.setenv("LFEM_TILE_ELEMS", str(budget))
    plan, rp, ci, v = gpu_assemble(m, kinds, coeff=u, variant=lfem.LFEM_NUMERIC_TILED)
    assert np.array_equal(rp, rp0) and np.array_equal(ci, ci0)
    for k in kinds:
        assert np.array_equal(v[k], v0[k]), f"kind {k} differs from the default plan at budget {budget}"
    o = oracle.assemble_rows(m, kinds, coeff=u)
    compare_rows(np.arange(m.n_nodes), rp, ci, v, o, kinds)


def test_repeated_numeric_calls_reuse_plan_bitwise():
    """The numeric phase is re-entrant: many calls on one plan (different
    coefficients, interleaved kind subsets) give the bits of fresh plans."""
    m = li.make_config("C5", level_override=3)
    mh = lfem.lfem_mesh_create(m.domain, m.order, m.quad, torch.as_tensor(m.coords, device="cuda"),
                               torch.as_tensor(m.conn, device="cuda"))
    plan = lfem.lfem_assemble_symbolic(mh)
    for seed in range(3):
        u = li.random_field(m, 100 + seed)
        cu = torch.as_tensor(u, device="cuda")
        for kmask in (7, 1, 4, 6, 7):
            v = [torch.empty(plan.nnz, dtype=torch.float64, device="cuda") if kmask >> i & 1 else None
                 for i in range(3)]
            lfem.lfem_assemble_numeric(plan, kmask, cu if kmask & 4 else None, v)
            lfem.lfem_plan_check(plan)
            kinds = tuple(k for i, k in enumerate(("M", "A", "Aa")) if kmask >> i & 1)
            _, _, _, ref = gpu_assemble(m, kinds, coeff=u if kmask & 4 else None)
            for i, k in enumerate(("M", "A", "Aa")):
                if kmask >> i & 1:
                    assert np.array_equal(v[i].cpu().numpy(), ref[k])


def test_allocator_hook_torch_caching_allocator():
    """SURVEY §8(b) lfem_set_allocator: plans built through PyTorch's caching
    allocator give the same bits; every allocation is released with the plan."""
    import gc
    m = li.make_config("C5", level_override=3)
    _, rp0, ci0, v0 = gpu_assemble(m, ("M", "A", "Aa"))
    alloc, dealloc = lfem.torch_caching_allocator()
    n = {"a": 0, "f": 0}
    mine = set()

    def a(nb, s):
        n["a"] += 1
        ptr = alloc(nb, s)
        mine.add(ptr)
        return ptr

    def f(p, s):
        assert p in mine, "the hook must only free its own pointers"
        n["f"] += 1
        dealloc(p, s)

    lfem.lfem_set_allocator(a, f)
    try:
        plan, rp, ci, v = gpu_assemble(m, ("M", "A", "Aa"))
        assert n["a"] > 0
        assert np.array_equal(rp, rp0) and np.array_equal(ci, ci0)
        for k in ("M", "A", "Aa"):
            assert np.array_equal(v[k], v0[k])
        del plan
        gc.collect()
        torch.cuda.synchronize()
    finally:
        lfem.lfem_set_allocator(None, None)
    assert n["f"] == n["a"], n


# ---------------------------------------------------------------------------- mesh-shape edge cases
def _fan(nseg, order, rings=2):
    """Disk-like surface fan around one vertex of valence nseg (nseg up to 40: slots with up to
    40 contributions -> the tiled kernel's larger heavy entries), a second ring for more rows,
    slightly curved in z."""
    pts = [[0.0, 0.0, 0.0]]
    for r in range(1, rings + 1):
        for k in range(nseg):
            t = 2 * np.pi * (k + 0.5 * (r - 1)) / nseg
            pts.append([r * np.cos(t), r * np.sin(t), 0.05 * r * r])
    tris = []
    for k in range(nseg):
        tris.append([0, 1 + k, 1 + (k + 1) % nseg])
    for r in range(1, rings):
        a0, b0 = 1 + (r - 1) * nseg, 1 + r * nseg
        for k in range(nseg):
            a, a1 = a0 + k, a0 + (k + 1) % nseg
            b, b1 = b0 + k, b0 + (k + 1) % nseg
            tris += [[a, b, a1], [a1, b, b1]]
    v, f = np.array(pts), np.array(tris)
    if order == 2:
        v, f = li.p2_from_p1_triangles(v, f, project_sphere=False)
        return li.Mesh(li.SURFACE_TRI, 2, v, f.astype(np.int32), li.QUAD_TRI6_DEG4)
    return li.Mesh(li.SURFACE_TRI, 1, v, f.astype(np.int32), li.QUAD_TRI3_DEG2)


@pytest.mark.parametrize("variant", [lfem.LFEM_NUMERIC_V0, lfem.LFEM_NUMERIC_TILED], ids=["v0", "tiled"])
@pytest.mark.parametrize("nseg,order", [(7, 1), (13, 1), (40, 1), (9, 2), (30, 2)])
def test_high_valence_fans(nseg, order, variant):
    """Vertex valences 7..40 (icospheres have <= 6): heavy slots with up to 40
    contributions (16-, 32- and 64-word heavy entries in the tiled kernel)."""
    m = li._finish(_fan(nseg, order))
    u = li.random_field(m, 7)
    worst, _ = check_full(m, ("M", "A", "Aa"), coeff=u, variant=variant)
    assert worst <= TOL


@pytest.mark.parametrize("variant", [lfem.LFEM_NUMERIC_V0, lfem.LFEM_NUMERIC_TILED], ids=["v0", "tiled"])
def test_unreferenced_nodes_give_empty_rows(variant):
    """Nodes no element uses (interleaved with used ones) are empty CSR rows:
    row_ptr repeats, the tiles around them stay correct."""
    base = li.make_config("C5", level_override=2)
    n = base.n_nodes
    # new numbering: every 3rd new id is an unused node
    new_id = np.arange(n) + np.arange(n) // 2
    coords = np.zeros((n + (n - 1) // 2 + 1, 3))
    coords[new_id] = base.coords
    unused = np.setdiff1d(np.arange(coords.shape[0]), new_id)
    coords[unused] = np.random.default_rng(0).normal(size=(unused.size, 3))
    m = li._finish(li.Mesh(base.domain, base.order, coords, new_id[base.conn].astype(np.int32), base.quad))
    u = li.random_field(m, 3)
    worst, (plan, rp, ci, vals) = check_full(m, ("M", "A", "Aa"), coeff=u, variant=variant)
    assert worst <= TOL
    assert np.all(np.diff(rp)[unused] == 0)



@pytest.mark.parametrize("mk", [lambda: li.make_config("C4P1", level_override=12),
                                lambda: li.perturb(li.sphere_mesh(4, 1), 3, 0.01),
                                lambda: li.make_config("C4", level_override=4)], ids=["tet1", "tri1", "tet2"])
def test_rows_variant_bitwise(mk):
    """ROWS (warp per row, elements recomputed per row) == V0 bit for bit (same element code, same
    ascending-element order per slot); P2 tets with rows > 64 columns fall back to V0."""
    m = mk()
    u = li.random_field(m, 2)
    _, _, _, a = gpu_assemble(m, ("M", "A", "Aa"), coeff=u, variant=lfem.LFEM_NUMERIC_V0)
    plan, _, _, b = gpu_assemble(m, ("M", "A", "Aa"), coeff=u, variant=lfem.LFEM_NUMERIC_ROWS)
    for k in ("M", "A", "Aa"):
        assert np.array_equal(a[k], b[k]), k
    if m.order == 1:
        assert lfem.lfem_numeric_launches(plan, 7) == 1
