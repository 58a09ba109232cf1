import sys, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import lfem_inputs as li, oracle
from gpu_common import gpu_assemble
from paper_2605_14035_b200 import lfem
m = li.perturb(li.sphere_mesh(4, 1), 2, 0.005)
u = li.random_field(m, 11)
o = oracle.assemble_rows(m, ("M","A","Aa"), coeff=u)
for rep in range(6):
    for v in (lfem.LFEM_NUMERIC_TILED, lfem.LFEM_NUMERIC_AUTO):
        plan, rp, ci, vals = gpu_assemble(m, ("M","A","Aa"), coeff=u, variant=v)
        bad = {}
        for k in ("M","A","Aa"):
            d = np.abs(vals[k]-o.vals[k]); rows = np.repeat(np.arange(m.n_nodes), np.diff(rp))
            rowmax = np.maximum.reduceat(np.abs(o.vals[k]), rp[:-1])[rows]
            w = np.nonzero(d > 1e-12*rowmax)[0]
            if len(w): bad[k] = (len(w), w[:8].tolist(), rows[w[:8]].tolist())
        print(rep, v, plan.nnz, bad if bad else "ok", flush=True)
print("tiles", m.n_nodes, m.n_elems)
