"""GPU parity of the curve family (Table 4 "surface 1D"): P1/P2
line elements in R^3 through the C-ABI (domain LFEM_SURFACE_LINE) against the oracle.
Bar as for the matrices: CSR pattern bit-exact, values within 1e-12 of the row max."""
import numpy as np
import pytest
import torch

import lfem_inputs as li
import oracle
from gpu_common import TOL, check_full

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2605_14035_b200 import lfem  # noqa: E402


def space_curve(n, order, seed):
    """A closed curve in R^3: the circle with a seeded radial and vertical perturbation."""
    m = li.circle_mesh(n, order)
    rng = li.SplitMix64(seed)
    x = m.coords.copy()
    x *= (1.0 + 0.1 * (rng.uniform(m.n_nodes) - 0.5))[:, None]
    x[:, 2] += 0.2 * (rng.uniform(m.n_nodes) - 0.5)
    return li.Mesh(m.domain, m.order, x, m.conn, m.quad)


def _gauss6(m):
    """The same P2 curve with the 6-point Gauss rule (the paper's order-10 rule, reading G38)."""
    return li.Mesh(m.domain, m.order, m.coords, m.conn, li.QUAD_LINE6_DEG11)


CURVES = [
    ("circle1_n5", lambda: li.circle_mesh(5, 1)),
    ("circle2_n7", lambda: li.circle_mesh(7, 2)),
    ("curve1_n4000", lambda: space_curve(4000, 1, 1)),
    ("curve2_n3000", lambda: space_curve(3000, 2, 2)),
    ("circle2_n7_gauss6", lambda: _gauss6(li.circle_mesh(7, 2))),
    ("curve2_n3000_gauss6", lambda: _gauss6(space_curve(3000, 2, 2))),
]


@pytest.mark.parametrize("variant", [lfem.LFEM_NUMERIC_V0, lfem.LFEM_NUMERIC_AUTO, lfem.LFEM_NUMERIC_ROWS],
                         ids=["v0", "auto", "rows_fallback"])
@pytest.mark.parametrize("name,mk", CURVES, ids=[c[0] for c in CURVES])
def test_curve_parity(name, mk, variant):
    m = mk()
    u = li.random_field(m, 4)
    worst, _ = check_full(m, ("M", "A", "Aa"), coeff=u, variant=variant)
    assert worst <= TOL


def test_curve_length_and_load():
    m = li.circle_mesh(4096, 2)
    plan, rp, ci, vals = lfem.assemble(m, ("M", "A"))
    one = torch.ones(m.n_nodes, dtype=torch.float64, device="cuda")
    y = torch.empty(plan.n_rows, dtype=torch.float64, device="cuda")
    lfem.lfem_spmv(plan, vals["M"], one, y)
    assert abs(float(y.sum()) - 2 * np.pi) < 1e-12
    f = li.random_field(m, 9)
    _, b = lfem.assemble_rhs(m, f[None, :], "load", plan=plan)
    o, oabs = oracle.assemble_rhs_rows(m, f[None, :], "load", with_abs=True)
    assert np.all(np.abs(b.cpu().numpy() - o) <= 1e-12 * oabs)


def test_curve_tiled_and_kll_unsupported():
    m = li.circle_mesh(16, 1)
    with pytest.raises(lfem.LfemError) as ei:
        lfem.assemble(m, ("M",), variant=lfem.LFEM_NUMERIC_TILED)
    assert ei.value.status == 2
    with pytest.raises(lfem.LfemError) as ei:
        lfem.assemble_rhs(m, np.ones((4, m.n_nodes)), "kll")
    assert ei.value.status == 2


def test_gauss6_load_vector_and_length():
    m = _gauss6(space_curve(2000, 2, 5))
    f = li.random_field(m, 9)
    plan, b = lfem.assemble_rhs(m, f[None, :], "load")
    o, oabs = oracle.assemble_rhs_rows(m, f[None, :], "load", with_abs=True)
    assert np.all(np.abs(b.cpu().numpy() - o) <= 1e-12 * oabs)
