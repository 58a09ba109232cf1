"""GPU parity of the mean-free surface Poisson solve (PAPER.md
P:152-166) against the oracle (oracle/poisson.py, direct solve of the Lagrange
form of [A; e^T] u = [b; 0]), the whole pipeline on the device: A by lfem_assemble_numeric,
b = M f_I by lfem_assemble_rhs (load), then lfem_solve_meanfree.

Tolerance (reading G35): PCG to ||r|| <= 1e-12 ||b~||; cond(A on e-perp) <= ~1e3 at
these levels, so |u_gpu - u_orc| <= 1e-9 max|u|.
"""
import math

import numpy as np
import pytest
import torch

import lfem_inputs as li
import oracle
from oracle import poisson

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2605_14035_b200 import lfem  # noqa: E402


def gpu_poisson(level, order):
    m = li.sphere_mesh(level, order)
    x = m.coords
    u = np.stack([x[:, 0] * x[:, 1], x[:, 1] * x[:, 2], x[:, 2] * x[:, 0]], axis=1)
    plan, rp, ci, vals = lfem.assemble(m, ("M", "A"))
    f = torch.as_tensor(np.ascontiguousarray((6.0 * u).T), device="cuda")  # (3, n) component-major
    cols = []
    for k in range(3):
        _, bk = lfem.assemble_rhs(m, f[k:k + 1], "load", plan=plan)
        cols.append(bk[0])
    b = torch.stack(cols, dim=1).contiguous()  # (n, 3) AoS
    uh = torch.empty_like(b)
    it = lfem.lfem_solve_meanfree(plan, vals["A"], b, uh, tol=1e-12)
    torch.cuda.synchronize()
    return m, u, uh.cpu().numpy(), b.cpu().numpy(), vals["M"].cpu().numpy(), rp.cpu().numpy(), ci.cpu().numpy(), it


@pytest.mark.parametrize("level,order", [(3, 2), (4, 1), (2, 2)])
def test_poisson_matches_oracle(level, order):
    m, u, uh, b, _, _, _, it = gpu_poisson(level, order)
    assert it > 0
    ref = poisson.solve_meanfree(m, b)
    assert np.max(np.abs(uh - ref)) <= 1e-9 * np.max(np.abs(ref))
    assert np.all(np.abs(uh.sum(axis=0)) <= 1e-12 * m.n_nodes * np.max(np.abs(ref)))


def test_poisson_eoc_on_gpu():
    errs = []
    for L in (2, 3, 4):
        m, u, uh, _, M, rp, ci, _ = gpu_poisson(L, 2)
        rows = np.repeat(np.arange(m.n_nodes), np.diff(rp))
        e = uh - (u - u.mean(axis=0))
        errs.append([math.sqrt(float(np.dot(e[:, k], np.bincount(rows, weights=M * e[ci, k], minlength=m.n_nodes))))
                     for k in range(3)])
    errs = np.array(errs)
    eoc = np.log2(errs[-2] / errs[-1])
    assert np.all(eoc > 2.7), eoc
