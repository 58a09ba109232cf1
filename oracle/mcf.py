"""Oracle of Dziuk's algorithm for mean curvature flow.

TEST INFRASTRUCTURE ONLY (see lfem_oracle.cpp's header): only tests/ and
bench.py's CPU legs use it.

PAPER.md §"Dziuk's algorithm": the linearly implicit Euler /
ESFEM discretisation of  d/dt X = Laplace_{Gamma[X]} Id  is

    (M(x^{n-1}) + tau A(x^{n-1})) x^n = M(x^{n-1}) x^{n-1},

one linear system per coordinate (x^n is the n_nodes x 3 node array).  Each
step: the oracle's own M and A (oracle_assemble_rows, C++) at x^{n-1}, then a
direct sparse solve (scipy's SuperLU: a library routine as one step).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import oracle as _o


def csr_matrix(c, kind, n_cols):
    return sp.csr_matrix((c.vals[kind], c.col_idx, c.row_ptr), shape=(c.rows.size, n_cols))


def mcf_step(mesh, x_prev: np.ndarray, tau: float, nthreads=None) -> np.ndarray:
    """x^n from x^{n-1} (n_nodes x 3) on the mesh's topology."""
    import lfem_inputs as li
    m = li.Mesh(mesh.domain, mesh.order, np.ascontiguousarray(x_prev, dtype=np.float64), mesh.conn, mesh.quad)
    c = _o.assemble_rows(m, ("M", "A"), nthreads=nthreads)
    M = csr_matrix(c, "M", m.n_nodes)
    A = csr_matrix(c, "A", m.n_nodes)
    K = (M + tau * A).tocsc()
    rhs = M @ x_prev
    lu = spla.splu(K)
    return np.ascontiguousarray(lu.solve(rhs))


def mcf(mesh, tau: float, steps: int, nthreads=None):
    """Run `steps` steps from the mesh's coordinates; returns the list of node arrays."""
    xs = [np.ascontiguousarray(mesh.coords, dtype=np.float64)]
    for _ in range(steps):
        xs.append(mcf_step(mesh, xs[-1], tau, nthreads))
    return xs
