"""GPU tests of the C-ABI's robustness (include/lfem.h conventions): the error
latch across reuse of a plan, alignment rules of the TILED kernel's bulk
copies, and the symbolic phase's long-row path (rows with more than 512
candidate (element, column) entries), each checked against the oracle."""
import numpy as np
import pytest
import torch

import lfem_inputs as li
import oracle
from gpu_common import TOL, check_full, compare_rows, gpu_assemble

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2605_14035_b200 import lfem  # noqa: E402


def _plan(m):
    X = torch.as_tensor(m.coords, device="cuda").contiguous()
    C = torch.as_tensor(m.conn, device="cuda").contiguous()
    mh = lfem.lfem_mesh_create(m.domain, m.order, m.quad, X, C)
    plan = lfem.lfem_assemble_symbolic(mh)
    plan._keep = (X, C)
    return plan


def _vals(plan):
    return [torch.empty(plan.nnz, dtype=torch.float64, device="cuda") for _ in range(3)]


@pytest.mark.parametrize("variant", [lfem.LFEM_NUMERIC_AUTO, lfem.LFEM_NUMERIC_V0])
def test_degenerate_then_valid_coords_on_one_plan(variant):
    """A degenerate call is reported once by lfem_plan_check; the same plan then
    assembles valid moving coordinates with an OK status and the fresh-plan bits."""
    m = li.make_config("C3", level_override=2)  # P1: a collapsed edge makes mu = 0 exactly
    plan = _plan(m)
    lfem.lfem_plan_set_variant(plan, variant)
    u = torch.as_tensor(li.random_field(m, 3), device="cuda")
    bad = m.coords.copy()
    bad[m.conn[11, 2]] = bad[m.conn[11, 1]]  # element 11 (and the other element on that edge) collapse
    v = _vals(plan)
    lfem.lfem_assemble_numeric_coords(plan, 7, torch.as_tensor(bad, device="cuda"), u, v)
    with pytest.raises(lfem.LfemError) as ei:
        lfem.lfem_plan_check(plan)
    assert ei.value.status == 4
    with pytest.raises(oracle.OracleError) as eo:
        oracle.assemble_rows(li.Mesh(m.domain, m.order, bad, m.conn, m.quad), ("M",))
    assert ei.value.element == eo.value.elem
    good = m.coords * 1.01
    lfem.lfem_assemble_numeric_coords(plan, 7, torch.as_tensor(good, device="cuda"), u, v)
    lfem.lfem_plan_check(plan)  # no stale error
    _, _, _, ref = gpu_assemble(li.Mesh(m.domain, m.order, good, m.conn, m.quad), ("M", "A", "Aa"),
                                coeff=u.cpu().numpy())
    for i, k in enumerate(("M", "A", "Aa")):
        assert np.array_equal(v[i].cpu().numpy(), ref[k])
    # the host entry point checks at its end: degenerate, then valid
    vh = [np.empty(plan.nnz) for _ in range(3)]
    with pytest.raises(lfem.LfemError):
        lfem.lfem_assemble_numeric_host(plan, 7, bad, u.cpu().numpy(), vh)
    lfem.lfem_assemble_numeric_host(plan, 7, good, u.cpu().numpy(), vh)
    assert np.array_equal(vh[0], ref["M"])


def _offset_view(a, shift):
    """a copy of `a` (float64) stored at a byte offset `shift` from a 256-B aligned allocation"""
    n = a.size
    raw = torch.zeros(n * 8 + 64, dtype=torch.uint8, device="cuda")
    v = raw[shift:shift + n * 8].view(torch.float64)
    v.copy_(torch.as_tensor(a.ravel(), device="cuda"))
    return v.view(a.shape), raw


def test_tiled_needs_16_byte_alignment():
    """coords / coeff at an 8-byte (not 16-byte) boundary: AUTO runs V0 (same bits, no
    misaligned-address fault), an explicit TILED request is INVALID_ARG; a 4-byte offset
    is INVALID_ARG for every variant."""
    m = li.make_config("C5", level_override=3)
    u = li.random_field(m, 4)
    _, rp, ci, ref = gpu_assemble(m, ("M", "A", "Aa"), coeff=u)
    X8, keep1 = _offset_view(m.coords, 8)
    U8, keep2 = _offset_view(u, 8)
    assert X8.data_ptr() % 16 == 8
    C = torch.as_tensor(m.conn, device="cuda")
    mh = lfem.lfem_mesh_create(m.domain, m.order, m.quad, X8, C)
    plan = lfem.lfem_assemble_symbolic(mh)
    v = _vals(plan)
    lfem.lfem_assemble_numeric(plan, 7, U8, v)
    lfem.lfem_plan_check(plan)
    for i, k in enumerate(("M", "A", "Aa")):
        assert np.array_equal(v[i].cpu().numpy(), ref[k]), k
    assert lfem.lfem_numeric_launches(plan, 7) == 2  # V0: element kernel + slot reduce
    lfem.lfem_plan_set_variant(plan, lfem.LFEM_NUMERIC_TILED)
    with pytest.raises(lfem.LfemError) as ei:
        lfem.lfem_assemble_numeric(plan, 7, U8, v)
    assert ei.value.status == 1
    # 4-byte offsets (no torch float64 tensor can live there): through the C ABI directly
    import ctypes
    raw = torch.zeros(m.n_nodes * 24 + 64, dtype=torch.uint8, device="cuda")
    p4 = ctypes.c_void_p(raw.data_ptr() + 4)
    h = ctypes.c_void_p()
    st = lfem._lib().lfem_mesh_create(m.domain, m.order, m.quad, m.n_nodes, p4, m.n_elems,
                                      ctypes.c_void_p(C.data_ptr()), ctypes.c_void_p(0), ctypes.byref(h))
    assert st == 1
    lfem.lfem_plan_set_variant(plan, lfem.LFEM_NUMERIC_V0)
    st = lfem._lib().lfem_assemble_numeric(plan.handle, 7, p4, lfem._vals_array(v), ctypes.c_void_p(0))
    assert st == 1


def _tet_star(level):
    """P2 tetrahedra around one interior vertex: every face of an icosphere of the
    given level is coned to the origin (level 1: 80 tets, level 2: 320 tets share vertex 0,
    i.e. 800 / 3200 candidate entries in row 0)."""
    s = li.icosphere_p1(level)
    v, f = s[0], s[1]
    pts = np.vstack([np.zeros((1, 3)), v * (1.0 + 0.1 * np.sin(3 * v[:, :1]))])
    tets = np.hstack([np.zeros((f.shape[0], 1), dtype=np.int64), f + 1])
    # orientation: det > 0 (|det| is used anyway, reading G17)
    P = pts[tets]
    d = np.einsum("ij,ij->i", np.cross(P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]), P[:, 3] - P[:, 0])
    tets[d < 0] = tets[d < 0][:, [0, 2, 1, 3]]
    # P2 edge nodes (1,2),(2,3),(3,1),(1,4),(2,4),(3,4) at chord midpoints (reading G26)
    edges = {}
    node_list = [p for p in pts]
    conn2 = []
    for t in tets:
        row = list(t)
        for a, b in ((0, 1), (1, 2), (2, 0), (0, 3), (1, 3), (2, 3)):
            key = (min(t[a], t[b]), max(t[a], t[b]))
            if key not in edges:
                edges[key] = len(node_list)
                node_list.append(0.5 * (pts[t[a]] + pts[t[b]]))
            row.append(edges[key])
        conn2.append(row)
    return li._finish(li.Mesh(li.BULK_TET, 2, np.array(node_list), np.array(conn2, dtype=np.int32),
                              li.QUAD_TET11_DEG4))


@pytest.mark.parametrize("level", [1, 2])
@pytest.mark.parametrize("variant", [lfem.LFEM_NUMERIC_AUTO, lfem.LFEM_NUMERIC_V0, lfem.LFEM_NUMERIC_ROWS])
def test_high_valence_tet_star_long_rows(level, variant):
    """A vertex shared by 80 / 320 P2 tets (more than 512 candidate entries in its row):
    the symbolic phase's long-row path gives the oracle's pattern, the values are in the gate."""
    m = _tet_star(level)
    assert np.sum(m.conn == 0) in (80, 320)
    u = li.random_field(m, 9)
    worst, _ = check_full(m, ("M", "A", "Aa"), coeff=u, variant=variant)
    assert worst <= TOL


def test_high_valence_tet_star_explicit_tiled():
    """An explicit TILED request on a row wider than the tile holds is UNSUPPORTED (no
    silent wrong values); AUTO on the same plan still assembles (V0)."""
    m = _tet_star(2)
    u = torch.as_tensor(li.random_field(m, 9), device="cuda")
    plan = _plan(m)
    v = _vals(plan)
    lfem.lfem_plan_set_variant(plan, lfem.LFEM_NUMERIC_TILED)
    with pytest.raises(lfem.LfemError) as ei:
        lfem.lfem_assemble_numeric(plan, 7, u, v)
    assert ei.value.status == 2
    lfem.lfem_plan_set_variant(plan, lfem.LFEM_NUMERIC_AUTO)
    lfem.lfem_assemble_numeric(plan, 7, u, v)
    lfem.lfem_plan_check(plan)
    o = oracle.assemble_rows(m, ("M", "A", "Aa"), coeff=u.cpu().numpy())
    rp, ci = lfem.lfem_csr_get(plan)
    compare_rows(np.arange(m.n_nodes), rp.cpu().numpy(), ci.cpu().numpy(),
                 {k: v[i].cpu().numpy() for i, k in enumerate(("M", "A", "Aa"))}, o, ("M", "A", "Aa"))


@pytest.mark.parametrize("variant", [lfem.LFEM_NUMERIC_AUTO, lfem.LFEM_NUMERIC_V0])
def test_p2_triangle_fan_long_row(variant):
    """A P2 surface vertex of valence 100 (600 candidate entries in its row)."""
    from test_gpu_parity import _fan
    m = li._finish(_fan(100, 2))
    u = li.random_field(m, 7)
    worst, _ = check_full(m, ("M", "A", "Aa"), coeff=u, variant=variant)
    assert worst <= TOL
