"""GPU parity of Dziuk's MCF step and the CG solver against the
oracle (oracle/mcf.py: the oracle's own M, A and a direct sparse solve).

Tolerance (reading G34): CG stops at ||r_k|| <= 1e-13 ||b_k||; K = M + tau A is SPD
with a modest condition number (<= ~1e3 for these meshes and steps), so each step's solution
is within ~1e-10 of the direct solve; over a few steps we assert 1e-9 * max|x|.
"""
import numpy as np
import pytest
import torch

import lfem_inputs as li
from oracle import mcf as omcf
import oracle

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2605_14035_b200 import lfem  # noqa: E402

TOL = 1e-13


def gpu_plan(m):
    coords = torch.as_tensor(m.coords, device="cuda").contiguous()
    conn = torch.as_tensor(m.conn, device="cuda").contiguous()
    mesh = lfem.lfem_mesh_create(m.domain, m.order, m.quad, coords, conn)
    plan = lfem.lfem_assemble_symbolic(mesh, 0, m.n_nodes)
    plan._keep = (coords, conn)
    return plan, coords


@pytest.mark.parametrize("mk", [lambda: li.perturb(li.sphere_mesh(3, 2), 2, 0.01), lambda: li.dziuk_surface(3, 2),
                                lambda: li.sphere_mesh(4, 1)], ids=["p2_sphere", "dziuk_p2", "p1_sphere"])
def test_mcf_steps_match_oracle(mk):
    m = mk()
    tau, steps = 0.005, 3
    xs = omcf.mcf(m, tau, steps)
    plan, coords = gpu_plan(m)
    x = coords.clone()
    y = torch.empty_like(x)
    for n in range(steps):
        it = lfem.lfem_mcf_step(plan, tau, x, y, tol=TOL)
        assert 0 < it < 2000
        x, y = y, x
        err = np.max(np.abs(x.cpu().numpy() - xs[n + 1]))
        assert err <= 1e-9 * np.max(np.abs(xs[n + 1])), (n, err)
    lfem.lfem_plan_check(plan)


def test_mcf_sphere_radius_law_on_gpu():
    """r(T)^2 = 1 - 4T within the scheme's first-order error (oracle pin, here through the GPU)."""
    m = li.sphere_mesh(3, 2)
    plan, coords = gpu_plan(m)
    x = coords.clone()
    tau, T = 0.002, 0.04
    for _ in range(int(round(T / tau))):
        lfem.lfem_mcf_step(plan, tau, x, x, tol=TOL)
    r = float(torch.sqrt(torch.mean(torch.sum(x * x, dim=1))))
    assert abs(r - np.sqrt(1 - 4 * T)) < 1e-3


def test_cg_matches_direct_solve():
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    m = li.perturb(li.sphere_mesh(4, 2), 5, 0.01)
    c = oracle.assemble_rows(m, ("M", "A"))
    K = c.vals["M"] + 0.01 * c.vals["A"]
    plan, _ = gpu_plan(m)
    rng = np.random.default_rng(0)
    b = rng.standard_normal((m.n_nodes, 3))
    x = torch.zeros((m.n_nodes, 3), dtype=torch.float64, device="cuda")
    it = lfem.lfem_cg_solve(plan, torch.as_tensor(K, device="cuda"), torch.as_tensor(b, device="cuda"), x, tol=TOL)
    Ks = sp.csr_matrix((K, c.col_idx, c.row_ptr), shape=(m.n_nodes, m.n_nodes)).tocsc()
    ref = spla.splu(Ks).solve(b)
    assert np.max(np.abs(x.cpu().numpy() - ref)) <= 1e-9 * np.max(np.abs(ref)), it
    # deterministic: same iterations, same bits
    x2 = torch.zeros_like(x)
    it2 = lfem.lfem_cg_solve(plan, torch.as_tensor(K, device="cuda"), torch.as_tensor(b, device="cuda"), x2, tol=TOL)
    assert it2 == it and torch.equal(x, x2)


def test_mcf_errors():
    m = li.sphere_mesh(2, 2)
    coords = torch.as_tensor(m.coords, device="cuda").contiguous()
    conn = torch.as_tensor(m.conn, device="cuda").contiguous()
    mesh = lfem.lfem_mesh_create(m.domain, m.order, m.quad, coords, conn)
    block = lfem.lfem_assemble_symbolic(mesh, 0, m.n_nodes // 2)
    x = coords.clone()
    with pytest.raises(lfem.LfemError) as ei:
        lfem.lfem_mcf_step(block, 0.01, x, x)
    assert ei.value.status == 2
    plan = lfem.lfem_assemble_symbolic(mesh, 0, m.n_nodes)
    with pytest.raises(lfem.LfemError) as ei:
        lfem.lfem_mcf_step(plan, 0.01, x, x, tol=1e-14, max_it=1)
    assert ei.value.status == 7
    with pytest.raises(lfem.LfemError) as ei:
        lfem.lfem_mcf_step(plan, -1.0, x, x)
    assert ei.value.status == 1
    c = li.cube_mesh(1, 1)
    cc = torch.as_tensor(c.coords, device="cuda").contiguous()
    cn = torch.as_tensor(c.conn, device="cuda").contiguous()
    cp = lfem.lfem_assemble_symbolic(lfem.lfem_mesh_create(c.domain, c.order, c.quad, cc, cn), 0, c.n_nodes)
    with pytest.raises(lfem.LfemError) as ei:
        lfem.lfem_mcf_step(cp, 0.01, cc.clone(), cc.clone())
    assert ei.value.status == 2
