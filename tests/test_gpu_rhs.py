"""GPU parity of the right-hand sides: the CUDA path
(lfem_assemble_rhs through the C-ABI liblfem.so) against the oracle.

Bar: every entry within 1e-12 x the oracle's rounding-error scale of that
entry (reading G33: every quadrature term with |w| mu, |u_h| and |phi| in
absolute value; for KLL alpha^2 replaced by its first-order error scale
alpha^2 + 2 sum_k |G_k| B_k, G_k formed from differences on both sides), and
exactly 0 where a row has no incident element.  On these fields the scale is
within ~10x of the value (median; test_oracle_rhs.py pins it), so the gate is
~1e-11 relative.
"""
import numpy as np
import pytest
import torch

import lfem_inputs as li
import oracle
from gpu_common import sample_rows

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2605_14035_b200 import lfem  # noqa: E402

TOL = 1e-12


def kll_fields(m, seed):
    """u = (nu; H): a perturbed unit-normal-like field and a curvature-like scalar (reading: synthetic)."""
    x = m.coords
    r = np.sqrt(np.einsum("ij,ij->i", x, x))
    r[r == 0] = 1.0
    nu = (x / r[:, None]).T + 0.05 * np.vstack([li.random_field(m, seed + k) for k in range(3)])
    H = 2.0 + 0.1 * li.random_field(m, seed + 3)
    return np.ascontiguousarray(np.vstack([nu, H[None, :]]))


def fields(m, kind, seed=5):
    return kll_fields(m, seed) if kind == "kll" else li.random_field(m, seed)[None, :]


def check(g, o, oabs):
    g = np.asarray(g)
    assert g.shape == o.shape
    err = np.abs(g - o)
    bad = err > TOL * oabs
    assert not bad.any(), f"{bad.sum()} entries out of tolerance; worst {np.max(err / np.maximum(oabs, 1e-300)):.3e}"
    assert np.all(g[oabs == 0] == 0.0)


SURF = [
    ("tri1_single", lambda: li.single_triangle([[0, 0, 0], [1, 0, 0], [0.2, 0.9, 0.3]], 1)),
    ("tri2_single", lambda: li.single_triangle([[0, 0, 0], [1, 0, 0], [0.2, 0.9, 0.3]], 2)),
    ("table12", li.table12_mesh),
    ("sphere1_L4_skew", lambda: li.perturb(li.sphere_mesh(4, 1), 2, 0.005)),
    ("sphere2_L3_skew", lambda: li.perturb(li.sphere_mesh(3, 2), 3, 0.01)),
    ("sphere2_L4_natural", lambda: li.sphere_mesh(4, 2, sfc=False)),
    ("C5_L5", lambda: li.make_config("C5", level_override=5)),
    ("sphere2_L3_q16", lambda: li.Mesh(li.SURFACE_TRI, 2, li.sphere_mesh(3, 2).coords, li.sphere_mesh(3, 2).conn,
                                       li.QUAD_TRI16_DEG8)),
]
BULK = [
    ("cube1_n3", lambda: li.cube_mesh(3, 1, displace_seed=1)),
    ("cube2_n1", lambda: li.cube_mesh(1, 2)),
    ("cube2_n4_disp", lambda: li.cube_mesh(4, 2, displace_seed=2)),
    ("C4_n5", lambda: li.make_config("C4", level_override=5)),
]


VARIANTS = [lfem.LFEM_NUMERIC_V0, lfem.LFEM_NUMERIC_TILED]


@pytest.mark.parametrize("variant", VARIANTS, ids=["v0", "fused"])
@pytest.mark.parametrize("name,mk", SURF + BULK, ids=[s[0] for s in SURF + BULK])
def test_load_parity(name, mk, variant):
    m = mk()
    u = fields(m, "load")
    plan, out = lfem.assemble_rhs(m, u, "load", variant=variant)
    o, oabs = oracle.assemble_rhs_rows(m, u, "load", with_abs=True)
    check(out.cpu().numpy(), o, oabs)
    assert lfem.lfem_rhs_launches(plan, lfem.LFEM_RHS_LOAD) == (2 if variant == lfem.LFEM_NUMERIC_V0 else 1)
    if variant == lfem.LFEM_NUMERIC_V0:
        _, out2 = lfem.assemble_rhs(m, u, "load", plan=plan, variant=lfem.LFEM_NUMERIC_TILED)
        assert torch.equal(out, out2)


@pytest.mark.parametrize("variant", VARIANTS, ids=["v0", "fused"])
@pytest.mark.parametrize("name,mk", SURF, ids=[s[0] for s in SURF])
def test_kll_parity(name, mk, variant):
    m = mk()
    u = fields(m, "kll")
    _, out = lfem.assemble_rhs(m, u, "kll", variant=variant)
    o, oabs = oracle.assemble_rhs_rows(m, u, "kll", with_abs=True)
    check(out.cpu().numpy(), o, oabs)


@pytest.mark.parametrize("kind", ["load", "kll"])
def test_rhs_variants_bitwise(kind):
    """The fused and the two-kernel variants sum the same element values in the same order."""
    m = li.make_config("C5", level_override=6)
    u = fields(m, kind)
    _, a = lfem.assemble_rhs(m, u, kind, variant=lfem.LFEM_NUMERIC_V0)
    plan, b = lfem.assemble_rhs(m, u, kind, variant=lfem.LFEM_NUMERIC_TILED)
    assert lfem.lfem_rhs_launches(plan, lfem.RHS_KINDS[kind]) == 1
    assert torch.equal(a, b)
    # the matrices on the same plan after the rhs built its tile plan, and the rhs again after them
    vals = [torch.empty(plan.nnz, dtype=torch.float64, device="cuda"), None, None]
    lfem.lfem_assemble_numeric(plan, lfem.LFEM_MASS, None, vals)
    _, c = lfem.assemble_rhs(m, u, kind, plan=plan)
    assert torch.equal(a, c)
    _, d = lfem.assemble_rhs(m, u, kind, plan=plan, variant=lfem.LFEM_NUMERIC_AUTO)  # AUTO = the two kernels
    assert torch.equal(a, d) and lfem.lfem_rhs_launches(plan, lfem.RHS_KINDS[kind]) == 2


def test_kll_identity_field_gives_2Mx():
    """nu = x (P2 sphere): f_1k = 2 M x_k on the GPU too (through the GPU's own M)."""
    m = li.perturb(li.sphere_mesh(3, 2), 8, 0.01)
    H = li.random_field(m, 1)
    u = np.vstack([m.coords.T, H[None, :]])
    plan, out = lfem.assemble_rhs(m, u, "kll")
    _, rp, ci, vals = lfem.assemble(m, ("M",))
    torch.cuda.synchronize()
    M = vals["M"].cpu().numpy()
    rows = np.repeat(np.arange(m.n_nodes), np.diff(rp.cpu().numpy()))
    ci = ci.cpu().numpy()
    f = out.cpu().numpy()
    for k in range(4):
        ref = 2.0 * np.bincount(rows, weights=M * u[k][ci], minlength=m.n_nodes)
        scale = 2.0 * np.bincount(rows, weights=np.abs(M * u[k][ci]), minlength=m.n_nodes)
        assert np.all(np.abs(f[k] - ref) <= 1e-12 * scale)


@pytest.mark.parametrize("kind", ["load", "kll"])
def test_rhs_row_blocks_bitwise(kind):
    """Multi-GPU row blocks (one GPU, sequential): each block's rows == the full result, bit for bit."""
    m = li.perturb(li.sphere_mesh(4, 2), 4, 0.01)
    u = fields(m, kind)
    _, full = lfem.assemble_rhs(m, u, kind)
    full = full.cpu().numpy()
    cuts = [0, 1, m.n_nodes // 3, m.n_nodes // 3 + 7, m.n_nodes - 5, m.n_nodes]
    for a, b in zip(cuts[:-1], cuts[1:]):
        for variant in VARIANTS:
            _, part = lfem.assemble_rhs(m, u, kind, row_begin=a, row_end=b, variant=variant)
            assert np.array_equal(part.cpu().numpy(), full[:, a:b]), (a, b, variant)


@pytest.mark.parametrize("kind", ["load", "kll"])
def test_rhs_repeat_and_moving_coords(kind):
    m = li.perturb(li.sphere_mesh(3, 2), 6, 0.01)
    u = fields(m, kind)
    plan, out1 = lfem.assemble_rhs(m, u, kind)
    _, out2 = lfem.assemble_rhs(m, u, kind, plan=plan)
    assert torch.equal(out1, out2)
    # moving geometry: same plan, new coordinates
    m2 = li.perturb(m, 12, 0.01)
    k = lfem.RHS_KINDS[kind]
    c2 = torch.as_tensor(m2.coords, device="cuda").contiguous()
    uu = torch.as_tensor(u, device="cuda").contiguous()
    out3 = torch.empty_like(out1)
    lfem.lfem_assemble_rhs(plan, k, c2, uu, out3)
    lfem.lfem_plan_check(plan)
    o, oabs = oracle.assemble_rhs_rows(m2, u, kind, with_abs=True)
    check(out3.cpu().numpy(), o, oabs)


def test_rhs_unreferenced_nodes_and_errors():
    m = li.sphere_mesh(2, 1)
    # append two nodes no element references
    m2 = li.Mesh(m.domain, m.order, np.vstack([m.coords, [[3.0, 0, 0], [0, 3.0, 0]]]), m.conn.copy(), m.quad)
    u = fields(m2, "load")
    _, out = lfem.assemble_rhs(m2, u, "load")
    o, oabs = oracle.assemble_rhs_rows(m2, u, "load", with_abs=True)
    check(out.cpu().numpy(), o, oabs)
    assert np.all(out.cpu().numpy()[:, -2:] == 0.0)
    c = li.cube_mesh(1, 1)
    with pytest.raises(lfem.LfemError) as ei:
        lfem.assemble_rhs(c, np.ones((4, c.n_nodes)), "kll")
    assert ei.value.status == 2
    plan, _ = lfem.assemble_rhs(m, fields(m, "load"), "load")
    uu = torch.ones(1, m.n_nodes, dtype=torch.float64, device="cuda")
    out = torch.empty(1, plan.n_rows, dtype=torch.float64, device="cuda")
    with pytest.raises(lfem.LfemError) as ei:
        lfem.lfem_assemble_rhs(plan, 7, None, uu, out)
    assert ei.value.status == 1
    with pytest.raises(lfem.LfemError) as ei:
        lfem.lfem_assemble_rhs(plan, lfem.LFEM_RHS_LOAD, None, None, out)
    assert ei.value.status == 1


def test_rhs_degenerate_element_latched():
    m = li.sphere_mesh(2, 2)
    bad = li.Mesh(m.domain, m.order, m.coords.copy(), m.conn.copy(), m.quad)
    e = 37
    for a in range(6):
        bad.coords[bad.conn[e, a]] = bad.coords[bad.conn[e, 0]]
    with pytest.raises(lfem.LfemError) as ei:
        lfem.assemble_rhs(bad, fields(bad, "kll"), "kll")
    assert ei.value.status == 4
    with pytest.raises(oracle.OracleError) as eo:
        oracle.assemble_rhs_rows(bad, fields(bad, "kll"), "kll")
    assert ei.value.element == eo.value.elem


@pytest.mark.slow
@pytest.mark.parametrize("cfg,kind", [("C5", "kll"), ("C5", "load"), ("C4", "load")])
def test_rhs_fullsize_sampled(cfg, kind):
    """BASELINE.json full sizes, sampled rows against the oracle (bench's launch configuration)."""
    m = li.make_config(cfg)
    u = fields(m, kind, seed=9)
    _, out = lfem.assemble_rhs(m, u, kind)
    rows = sample_rows(m.n_nodes, 3000, seed=3)
    o, oabs = oracle.assemble_rhs_rows(m, u, kind, rows=rows, with_abs=True)
    check(out[:, torch.as_tensor(rows, device="cuda")].cpu().numpy(), o, oabs)


@pytest.mark.slow
@pytest.mark.parametrize("cfg,kind", [("C5", "kll"), ("C4", "load")])
def test_rhs_fullsize_every_row(cfg, kind):
    """BASELINE.json full sizes, EVERY row against the oracle (the oracle over all rows at once)."""
    m = li.make_config(cfg)
    u = fields(m, kind, seed=9)
    _, out = lfem.assemble_rhs(m, u, kind)
    o, oabs = oracle.assemble_rhs_rows(m, u, kind, with_abs=True)
    check(out.cpu().numpy(), o, oabs)


@pytest.mark.parametrize("variant", VARIANTS, ids=["v0", "fused"])
def test_rhs_empty_row_block_and_tiny_mesh(variant):
    """Degenerate sizes: an empty owned-row block, a one-row block, and a single element."""
    m = li.sphere_mesh(2, 2)
    u = fields(m, "kll")
    _, out = lfem.assemble_rhs(m, u, "kll", row_begin=7, row_end=7, variant=variant)
    assert tuple(out.shape) == (4, 0)
    _, one = lfem.assemble_rhs(m, u, "kll", row_begin=7, row_end=8, variant=variant)
    o, oabs = oracle.assemble_rhs_rows(m, u, "kll", rows=np.array([7], dtype=np.int64), with_abs=True)
    check(one.cpu().numpy(), o, oabs)
    t = li.single_triangle([[0, 0, 0], [1, 0, 0], [0.2, 0.9, 0.3]], 2)
    ut = fields(t, "load")
    _, ot = lfem.assemble_rhs(t, ut, "load", variant=variant)
    o2, oabs2 = oracle.assemble_rhs_rows(t, ut, "load", with_abs=True)
    check(ot.cpu().numpy(), o2, oabs2)
