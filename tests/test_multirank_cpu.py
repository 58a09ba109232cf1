"""Multi-rank path on CPU (gloo, world size 2): the row-block decomposition of
DESIGN.md §7 / SURVEY.md §8(e), exercised with the oracle as the per-rank
assembler (the GPU kernels run the same plan per rank; their 1-GPU emulation
is tests/test_gpu_parity.py::test_row_block_partition_emulation).

Checks: (1) the blocks cover every row once and are balanced; (2) the blocks'
CSR, gathered, is bitwise the whole-mesh assembly (halo elements duplicated,
only owned rows kept); (3) the verification step of bench.py -- NCCL/gloo
all-gather of a sharded x, local SpMV on the owned rows, all-reduce of the
checksums -- reproduces the whole-matrix SpMV; (4) max-over-ranks timing;
(5) the same for the KLL right-hand side.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import lfem_inputs as li
import oracle
from paper_2605_14035_b200.partition import partition_rows

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spmv(rp, ci, v, x):
    y = np.zeros(len(rp) - 1)
    for r in range(len(rp) - 1):
        y[r] = np.dot(v[rp[r]:rp[r + 1]], x[ci[rp[r]:rp[r + 1]]])
    return y


def _kll_u(m):
    return np.vstack([m.coords.T, m.coeff[None, :]])


def _worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        # rank 0 generates (seeded), broadcast to the others (bench.py's plumbing)
        if rank == 0:
            m = li.make_config("C5", level_override=2)
            meta = torch.tensor([m.n_nodes, m.n_elems], dtype=torch.int64)
        else:
            meta = torch.empty(2, dtype=torch.int64)
        dist.broadcast(meta, 0)
        n_nodes, n_elems = (int(x) for x in meta)
        if rank == 0:
            coords = torch.from_numpy(m.coords.copy())
            conn = torch.from_numpy(m.conn.copy())
            coeff = torch.from_numpy(m.coeff.copy())
        else:
            coords = torch.empty((n_nodes, 3), dtype=torch.float64)
            conn = torch.empty((n_elems, 6), dtype=torch.int32)
            coeff = torch.empty(n_nodes, dtype=torch.float64)
        for t in (coords, conn, coeff):
            dist.broadcast(t, 0)
        mesh = li.Mesh(li.SURFACE_TRI, 2, coords.numpy(), conn.numpy(), li.QUAD_TRI6_DEG4, coeff=coeff.numpy())
        bounds = partition_rows(mesh.conn, n_nodes, WORLD)
        r0, r1 = bounds[rank], bounds[rank + 1]
        blk = oracle.assemble_rows(mesh, ("M", "A", "Aa"), rows=np.arange(r0, r1, dtype=np.int64), nthreads=1)
        # N1: the KLL right-hand side of the owned rows (same decomposition, no collective)
        f_blk = oracle.assemble_rhs_rows(mesh, _kll_u(mesh), "kll", rows=np.arange(r0, r1, dtype=np.int64), nthreads=1)
        # (2) gather the blocks on rank 0
        objs = [None] * WORLD
        dist.all_gather_object(objs, (r0, r1, blk.row_ptr, blk.col_idx, {k: v for k, v in blk.vals.items()}, f_blk))
        # (3) verification SpMV: x sharded, all-gathered, local rows, checksum all-reduced
        x = mesh.coords[:, 0].copy()
        shard = (n_nodes + WORLD - 1) // WORLD
        loc = torch.zeros(shard, dtype=torch.float64)
        mine = x[rank * shard:min(n_nodes, (rank + 1) * shard)]
        loc[:mine.size] = torch.from_numpy(mine)
        xs = [torch.zeros(shard, dtype=torch.float64) for _ in range(WORLD)]
        dist.all_gather(xs, loc)
        xg = torch.cat(xs)[:n_nodes].numpy()
        y = _spmv(blk.row_ptr, blk.col_idx, blk.vals["A"], xg)
        chk = torch.tensor([float(np.dot(xg[r0:r1], y)), float(blk.vals["M"].sum())], dtype=torch.float64)
        dist.all_reduce(chk)
        # (4) max over ranks
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            out.put((bounds, objs, chk.numpy().tolist(), float(t)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_row_blocks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    bounds, objs, chk, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = li.make_config("C5", level_override=2)
    full = oracle.assemble_rows(m, ("M", "A", "Aa"), nthreads=1)
    # (1) coverage and balance
    assert bounds[0] == 0 and bounds[-1] == m.n_nodes and all(a < b for a, b in zip(bounds, bounds[1:]))
    inc = np.bincount(m.conn.ravel(), minlength=m.n_nodes)
    parts = [inc[a:b].sum() for a, b in zip(bounds, bounds[1:])]
    assert max(parts) <= 1.05 * sum(parts) / WORLD + inc.max()
    # (2) bitwise equal to the whole assembly
    rp = [np.asarray(o[2]) for o in objs]
    ci = np.concatenate([o[3] for o in objs])
    assert np.array_equal(ci, full.col_idx)
    offs = np.cumsum([0] + [r[-1] for r in rp])
    glued = np.concatenate([rp[0]] + [r[1:] + offs[i] for i, r in enumerate(rp) if i > 0])
    assert np.array_equal(glued, full.row_ptr)
    for k in ("M", "A", "Aa"):
        assert np.array_equal(np.concatenate([o[4][k] for o in objs]), full.vals[k])
    # N1 right-hand side: the gathered row blocks == the whole-mesh vector, bit for bit
    f_full = oracle.assemble_rhs_rows(m, _kll_u(m), "kll", nthreads=1)
    assert np.array_equal(np.concatenate([o[5] for o in objs], axis=1), f_full)
    # (3) distributed SpMV checksum == whole-matrix values
    x = m.coords[:, 0]
    yf = _spmv(full.row_ptr, full.col_idx, full.vals["A"], x)
    assert abs(chk[0] - float(np.dot(x, yf))) <= 1e-12 * max(1.0, abs(float(np.dot(x, yf))))
    assert abs(chk[1] - float(full.vals["M"].sum())) <= 1e-12 * float(full.vals["M"].sum())
    # (4) max over ranks
    assert tmax == float(WORLD)
