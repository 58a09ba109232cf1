"""Shared helpers of the GPU parity tests: run the CUDA path through the C-ABI
binding and compare with the oracle (tests only)."""
from __future__ import annotations

import numpy as np
import torch

import oracle
from paper_2605_14035_b200 import lfem

TOL = 1e-12  # BASELINE.json north_star: |gpu - oracle| <= 1e-12 * max_j |oracle(i, j)| per row


def gpu_assemble(mesh, kinds, coeff=None, row_begin=0, row_end=None, variant=lfem.LFEM_NUMERIC_AUTO):
    plan, row_ptr, col_idx, vals = lfem.assemble(mesh, kinds, coeff=coeff, row_begin=row_begin, row_end=row_end,
                                                 variant=variant)
    torch.cuda.synchronize()
    return plan, row_ptr.cpu().numpy(), col_idx.cpu().numpy(), {k: v.cpu().numpy() for k, v in vals.items()}


def compare_rows(rows, g_row_ptr, g_col, g_vals, o, kinds, row_offset=0):
    """rows: global row ids present in oracle result `o` (same order);
    g_*: the GPU plan's CSR (plan-relative rows, row_offset = plan row_begin)."""
    worst = 0.0
    for j, r in enumerate(rows):
        gr = r - row_offset
        a, b = g_row_ptr[gr], g_row_ptr[gr + 1]
        s, e = o.row_ptr[j], o.row_ptr[j + 1]
        gc = g_col[a:b]
        oc = o.col_idx[s:e]
        assert np.array_equal(gc, oc), f"pattern mismatch in row {r}: {gc} vs {oc}"
        for k in kinds:
            ov = o.vals[k][s:e]
            gv = g_vals[k][a:b]
            scale = np.abs(ov).max() if ov.size else 0.0
            err = np.abs(gv - ov).max() if ov.size else 0.0
            assert err <= TOL * scale, f"kind {k} row {r}: err {err:.3e} > {TOL:.0e} * {scale:.3e}"
            if scale > 0:
                worst = max(worst, err / scale)
    return worst


def check_full(mesh, kinds, coeff=None, variant=lfem.LFEM_NUMERIC_AUTO, nthreads=None):
    plan, rp, ci, vals = gpu_assemble(mesh, kinds, coeff=coeff, variant=variant)
    o = oracle.assemble_rows(mesh, kinds, coeff=coeff, nthreads=nthreads)
    assert plan.nnz == o.nnz
    assert np.array_equal(rp, o.row_ptr), "row_ptr mismatch"
    assert np.array_equal(ci, o.col_idx), "col_idx mismatch"
    return compare_rows(np.arange(mesh.n_nodes), rp, ci, vals, o, kinds), (plan, rp, ci, vals)


def sample_rows(n_nodes, count, seed=0):
    rng = np.random.default_rng(seed)
    r = set(rng.choice(n_nodes, size=min(count, n_nodes), replace=False).tolist())
    r.update([0, n_nodes - 1, n_nodes // 2])
    return np.array(sorted(r), dtype=np.int64)
