#!/usr/bin/env python
"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every numeric variant on small meshes, the tiled kernel with tiny tile budgets (8, 17
elements: thousands of tiles, ragged tails, single-row tiles), the right-hand sides and
one MCF step.  Each case is checked against the oracle so a silent corruption would also
fail here.  Usage: compute-sanitizer --tool <tool> python scripts/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import lfem_inputs as li  # noqa: E402
from gpu_common import TOL, check_full  # noqa: E402
from paper_2605_14035_b200 import lfem  # noqa: E402

V = {"v0": lfem.LFEM_NUMERIC_V0, "tiled": lfem.LFEM_NUMERIC_TILED, "rows": lfem.LFEM_NUMERIC_ROWS}


def case(name, m, variant, budget=None):
    if budget is not None:
        os.environ["LFEM_TILE_ELEMS"] = str(budget)
    else:
        os.environ.pop("LFEM_TILE_ELEMS", None)
    u = m.coeff if m.coeff is not None else li.random_field(m, 3)
    worst, _ = check_full(m, ("M", "A", "Aa"), coeff=u, variant=V[variant])
    assert worst <= TOL, (name, variant, worst)
    print(f"ok {name} {variant} budget={budget} worst={worst:.2e}", flush=True)


def main():
    torch.cuda.set_device(0)
    c1 = li.make_config("C1")
    c5 = li.make_config("C5", level_override=3)
    c3 = li.make_config("C3", level_override=3)
    c4 = li.make_config("C4", level_override=2)
    for v in ("tiled", "v0", "rows"):
        case("C1", c1, v)
    for b in (None, 8, 17):
        case("C5_L3", c5, "tiled", b)
        case("C3_L3", c3, "tiled", b)
    case("C4_n2", c4, "v0")
    case("C4_n2", c4, "tiled", 17)
    os.environ.pop("LFEM_TILE_ELEMS", None)
    # right-hand sides (two-kernel and fused variants) on the C5 mesh
    uk = np.vstack([c5.coords.T, li.random_field(c5, 1)[None, :]])
    for var in (lfem.LFEM_NUMERIC_V0, lfem.LFEM_NUMERIC_TILED):
        lfem.assemble_rhs(c5, uk, "kll", variant=var)
        lfem.assemble_rhs(c5, li.random_field(c5, 2)[None, :], "load", variant=var)
    # one MCF step (assembly on moving nodes + PCG)
    m = li.dziuk_surface(2, 2)
    X = torch.as_tensor(m.coords, device="cuda").contiguous()
    C = torch.as_tensor(m.conn, device="cuda").contiguous()
    plan = lfem.lfem_assemble_symbolic(lfem.lfem_mesh_create(m.domain, m.order, m.quad, X, C))
    xn = torch.empty_like(X)
    lfem.lfem_mcf_step(plan, 0.005, X, xn, tol=1e-10, max_it=2000)
    torch.cuda.synchronize()
    print("sanitize workload done", flush=True)


if __name__ == "__main__":
    main()
