"""Oracle of the mean-free surface Poisson problem.

TEST INFRASTRUCTURE ONLY (see lfem_oracle.cpp's header).

PAPER.md P:152-166: A_0 u = b_0 with A_0 = [A; e^T] ((N+1) x N, e = ones) and
b_0 = [b; 0].  Its least-squares solution (MATLAB's backslash on the
rectangular system) solves the Lagrange system  [[A, e], [e^T, 0]] [u; l] =
[b; 0]  (A u + l e = b, e^T u = 0; since A e = 0 and A is symmetric, l =
mean(b) and A u = b - mean(b) e) -- solved here directly (SuperLU), one
column at a time.  b = M f_I (b = M f for f_h = sum f_j phi_j).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import oracle as _o


def solve_meanfree(mesh, b: np.ndarray, nthreads=None) -> np.ndarray:
    """u (n x k) with [A; e^T] u = [b; 0] in the least-squares sense, b: n x k."""
    c = _o.assemble_rows(mesh, ("A",), nthreads=nthreads)
    n = mesh.n_nodes
    A = sp.csr_matrix((c.vals["A"], c.col_idx, c.row_ptr), shape=(n, n))
    e = sp.csr_matrix(np.ones((n, 1)))
    S = sp.bmat([[A, e], [e.T, None]]).tocsc()
    lu = spla.splu(S)
    b = np.asarray(b, dtype=np.float64).reshape(n, -1)
    rhs = np.vstack([b, np.zeros((1, b.shape[1]))])
    return np.ascontiguousarray(lu.solve(rhs)[:n])
