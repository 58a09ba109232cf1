"""Host-side multi-GPU decomposition.

The numeric phase partitions into independent row blocks: rank g owns the
contiguous global rows [bounds[g], bounds[g+1]) of the SFC-ordered mesh, runs
lfem_assemble_symbolic(mesh, bounds[g], bounds[g+1]) (elements touching its
rows, halo duplicated) and keeps only its rows -- no collective in the
numeric phase.  Blocks are balanced by incidences (element-local rows), a
proxy for nnz and element work.
"""
from __future__ import annotations

import numpy as np


def partition_rows(conn: np.ndarray, n_nodes: int, world: int) -> list:
    """Contiguous row blocks [b[g], b[g+1]) with about equal numbers of
    (element, local row) incidences.  Returns world + 1 bounds."""
    if world <= 1:
        return [0, int(n_nodes)]
    w = np.bincount(np.asarray(conn).ravel(), minlength=n_nodes).astype(np.int64)
    c = np.cumsum(w)
    tot = int(c[-1]) if c.size else 0
    bounds = [0]
    for r in range(1, world):
        bounds.append(max(bounds[-1], int(np.searchsorted(c, tot * r / world))))
    bounds.append(int(n_nodes))
    return bounds
