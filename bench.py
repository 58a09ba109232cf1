#!/usr/bin/env python
"""Benchmark of the ℓFEM numeric assembly hot path on B200 (BASELINE.json metric:
elements/s and CSR nnz/s of fp64 mass+stiffness numeric assembly, % HBM
roofline, 1/2/4/8 GPU).

One "step" = one lfem_assemble_numeric call producing every kind the config
names (C5: M, A, A_a) over the whole mesh (all ranks together), inputs
resident in HBM.  The one-time symbolic phase is timed and reported
separately (`symbolic_ms`).  Multi-GPU: one process per GPU (torchrun),
contiguous row blocks of the SFC-ordered mesh, halo elements duplicated,
no collective in the numeric phase; time = max over ranks (CUDA events).

  python bench.py [--gpus N --steps K --warmup W --config C5]
  python bench.py --impl reference ...   (the CPU oracle arm, rank 0 only)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

L2_BYTES = 126 * 2 ** 20
KIND_BITS = {"M": 1, "A": 2, "Aa": 4}
KIND_INDEX = {"M": 0, "A": 1, "Aa": 2}
CONFIG_DESC = {
    "C1": "P1 icosphere L3 (1,280 tri), radial noise 1e-3, M+A, TRI3_DEG2",
    "C2": "P2 icosphere L7 (327,680 curved tri), M+A, TRI6_DEG4",
    "C3": "P1 perturbed icosphere L9 (5,242,880 tri), M+A_a, u updated per step, TRI3_DEG2",
    "C4": "P2 Kuhn cube 96^3x6 (5,308,416 tets), displaced, M+A, TET11_DEG4",
    "C5": "P2 icosphere L10 (20,971,520 curved tri, 41,943,042 nodes), SFC order, M+A+A_a, TRI6_DEG4",
    "C4P1": "P1 Kuhn cube 96^3x6 (5,308,416 tets, 912,673 nodes), displaced, M+A, TET4_DEG2 (SURVEY N2)",
    "CURVE2": "P2 unit circle, 8,388,608 line elements (16,777,216 nodes), M+A, 3-point Gauss (SURVEY N2)",
}
FLOP_PER_ELEM = {"C1": 120, "C2": 1780, "C3": 120, "C4": 9600, "C5": 2640,  # SURVEY §8(d).3 model
                 "C4P1": 700, "CURVE2": 150}  # P1 tet: J, cofactors, det per point (4 points) + 2 x 10 entries


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def algorithmic_bytes(name, n_elems, nref, n_nodes, nnz, kinds, has_coeff):
    """BASELINE.json: connectivity + coordinates (each node once) + CSR values
    written once; + the coefficient u (one read per node) for C3/C5."""
    b = n_elems * nref * 4 + n_nodes * 24 + len(kinds) * nnz * 8
    if has_coeff:
        b += n_nodes * 8
    return b


# one metric string per workload, shared by the GPU arm and the reference arm (the driver pairs them)
METRIC_MATRICES = "elements/s (fp64 numeric assembly of all kinds of the config into CSR)"


def metric_rhs(kind):
    return f"elements/s (fp64 {kind} right-hand side assembly)"


# configs whose step moves < 4 x L2 (504 MB): L2 flushed (256 MiB write) between timed steps
FLUSH_L2 = {"C1", "C2", "C3", "C4P1"}


def l2_note(name):
    return "flushed (256 MiB write) between steps" if name in FLUSH_L2 else "inputs+outputs > L2 (126 MB); no flush"


def config_matrices(name, m, kinds, world, variant):
    """The bench line's `config` (identical in the GPU arm and the reference arm)."""
    return {"workload": f"{name}: {CONFIG_DESC[name]}" + (" [Dunavant-8 rule, 16 points]" if QUAD8 else "")
                        + (" [natural generator order, no SFC renumbering]" if NATURAL else ""),
            "kinds": list(kinds), "n_elems": int(m.n_elems), "n_nodes": int(m.n_nodes),
            "parallelism": f"row-blocks x{world}", "l2": l2_note(name), "variant": variant}


def config_rhs(name, m, kind, nc, world, variant):
    return {"workload": f"{name} mesh ({m.n_elems} elements, {m.n_nodes} nodes), {kind} right-hand "
                        f"side ({nc} components)" + (", Dunavant-8 rule" if QUAD8 else ""),
            "rhs": kind, "parallelism": f"row-blocks x{world}", "variant": variant, "l2": l2_note(name)}


QUAD8 = False  # --quad8: P2 triangle configs with Dunavant's 16-point degree-8 rule
NATURAL = False  # --natural: C2 in the generator's own numbering (SURVEY §8(d).2 sensitivity point)
CPU_THREADS = None  # --cpu-threads: threads of the oracle's cpu_baseline sample (default: all host cores)


def build_mesh(name):
    import lfem_inputs as li
    t0 = time.time()
    if NATURAL and name != "C2":
        raise SystemExit("--natural applies to C2")
    m = li.make_config(name, natural=NATURAL)
    if QUAD8:
        if not (m.domain == li.SURFACE_TRI and m.order == 2):
            raise SystemExit("--quad8 applies to P2 triangle configs (C2, C5)")
        m.quad = li.QUAD_TRI16_DEG8
        m.extra["quad8"] = True
    return m, time.time() - t0


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle (CPU) legs
def _oracle_rows_for(m, kinds, coeff, target_s, nt, call=None):
    """Rows of a contiguous block that take about target_s seconds in the oracle.
    The oracle has a per-call setup (node -> element incidence over the whole
    mesh) and a per-row cost: a tiny sample measures the first, a 5 % sample the
    second; the per-row cost grows with the sample (map sizes, caches), hence a
    safety factor of 1.7 (measured on C5 at level 8: 0.8 us/row at 2 %, 1.35 at 100 %)."""
    import oracle
    if call is None:
        def call(rows):
            oracle.assemble_rows(m, kinds, rows=rows, coeff=coeff, nthreads=nt)
    r0 = min(m.n_nodes, 100)
    r1 = min(m.n_nodes, max(50000, m.n_nodes // 20))
    t0 = time.perf_counter()
    call(np.arange(r0, dtype=np.int64))
    setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    call(np.arange(r1, dtype=np.int64))
    t1 = time.perf_counter() - t0
    per_row = max((t1 - setup) / max(1, r1 - r0), t1 / r1 * 1e-3, 1e-9)
    rows = int(r0 + max(0.0, target_s - setup) / (1.7 * per_row))
    return int(min(m.n_nodes, max(r0, rows)))


def oracle_sample(m, kinds, coeff, target_s):
    """Time the oracle as it stands on a contiguous block of rows sized for
    about target_s seconds; returns (elements/s equivalent, rows, seconds, threads)."""
    import oracle
    nt = CPU_THREADS or os.cpu_count() or 1
    rows = _oracle_rows_for(m, kinds, coeff, target_s, nt)
    t0 = time.perf_counter()
    c = oracle.assemble_rows(m, kinds, rows=np.arange(rows, dtype=np.int64), coeff=coeff, nthreads=nt)
    dt = time.perf_counter() - t0
    equiv_elems = m.n_elems * rows / m.n_nodes
    return equiv_elems / dt, rows, dt, nt, c.nnz


def rhs_fields(m, kind):
    """Synthetic nodal data of the right-hand side workloads: load f = a seeded
    smooth-ish field; KLL u = (nu; H), nu = x/|x| + 0.05 noise (a perturbed unit normal on the
    sphere), H = 2 + 0.1 noise (the unit sphere's mean curvature, perturbed)."""
    import lfem_inputs as li
    if kind == "load":
        return np.ascontiguousarray(li.random_field(m, 5)[None, :])
    x = m.coords
    r = np.sqrt(np.einsum("ij,ij->i", x, x))
    r[r == 0] = 1.0
    nu = (x / r[:, None]).T + 0.05 * np.vstack([li.random_field(m, 5 + k) for k in range(3)])
    H = 2.0 + 0.1 * li.random_field(m, 8)
    return np.ascontiguousarray(np.vstack([nu, H[None, :]]))


def rhs_alg_bytes(n_elems, nref, n_nodes_in, n_rows, nc):
    """conn + coords (each node once) + nodal input u (ncomp per node) + output (ncomp per owned row)."""
    return n_elems * nref * 4 + n_nodes_in * 24 + n_nodes_in * nc * 8 + n_rows * nc * 8


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if args.rhs:
        return run_reference_rhs(args)
    name = args.config
    m, gen_s = build_mesh(name)
    kinds = m.extra["kinds"]
    coeff = m.coeff
    import oracle
    nt = os.cpu_count() or 1
    # calibrate, then size each step for ~budget/(K+W) seconds
    budget = float(os.environ.get("LFEM_REF_BUDGET_S", "90"))
    per_step = budget / max(1, args.steps + args.warmup)
    rows = max(2000, _oracle_rows_for(m, kinds, coeff, per_step, nt))
    times = []
    for it in range(args.warmup + args.steps):
        r0 = (it * rows) % max(1, m.n_nodes - rows + 1)
        rr = np.arange(r0, r0 + rows, dtype=np.int64)
        t0 = time.perf_counter()
        oracle.assemble_rows(m, kinds, rows=rr, coeff=coeff, nthreads=nt)
        if it >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = sum(times)
    equiv = m.n_elems * rows / m.n_nodes * len(times)
    value = equiv / t
    line = {"impl": "reference", "metric": METRIC_MATRICES,
            "value": value, "unit": "elements/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t / len(times), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, lfem_inputs)",
            "config": config_matrices(name, m, kinds, args.gpus, args.variant),
            "cpu_baseline": {"value": value, "unit": "elements/s", "cores": nt, "kind": "oracle",
                             "sample": f"{rows} contiguous rows per step of {m.n_nodes} "
                                       f"(elements/s = n_elems * rows/n_rows / t); per-step sample"},
            "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_reference_rhs(args):
    import oracle
    name, kind = args.config, args.rhs
    m, _ = build_mesh(name)
    u = rhs_fields(m, kind)
    nt = os.cpu_count() or 1
    budget = float(os.environ.get("LFEM_REF_BUDGET_S", "90"))
    per_step = budget / max(1, args.steps + args.warmup)

    def call(rows):
        oracle.assemble_rhs_rows(m, u, kind, rows=rows, nthreads=nt)
    rows = max(2000, _oracle_rows_for(m, None, None, per_step, nt, call=call))
    times = []
    for it in range(args.warmup + args.steps):
        r0 = (it * rows) % max(1, m.n_nodes - rows + 1)
        t0 = time.perf_counter()
        call(np.arange(r0, r0 + rows, dtype=np.int64))
        if it >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = sum(times)
    value = m.n_elems * rows / m.n_nodes * len(times) / t
    line = {"impl": "reference", "metric": metric_rhs(kind),
            "value": value, "unit": "elements/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t / len(times), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, lfem_inputs)",
            "config": config_rhs(name, m, kind, u.shape[0], args.gpus, args.variant),
            "cpu_baseline": {"value": value, "unit": "elements/s", "cores": nt, "kind": "oracle",
                             "sample": f"{rows} contiguous rows per step of {m.n_nodes}"},
            "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU leg: right-hand sides
def run_rhs(args):
    """One step = one lfem_assemble_rhs call over the config's mesh; 1 GPU
    or row blocks over ranks like the matrices (no collective)."""
    import torch
    import torch.distributed as dist

    from paper_2605_14035_b200 import lfem
    from paper_2605_14035_b200.partition import partition_rows

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("LFEM_BENCH_DEVICE") is not None:
        local = int(os.environ["LFEM_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("LFEM_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    name, kind = args.config, args.rhs
    k = lfem.RHS_KINDS[kind]
    nc = lfem.lfem_rhs_ncomp(k)
    m, gen_s = build_mesh(name)  # every rank generates the same seeded mesh (no broadcast needed)
    u_np = rhs_fields(m, kind)
    coords = torch.as_tensor(m.coords).to(dev)
    conn = torch.as_tensor(m.conn).to(dev)
    u = torch.as_tensor(u_np).to(dev)
    bounds = partition_rows(m.conn, m.n_nodes, world) if world > 1 else [0, m.n_nodes]
    r0, r1 = bounds[rank], bounds[rank + 1]
    stream = torch.cuda.current_stream()
    mesh = lfem.lfem_mesh_create(m.domain, m.order, m.quad, coords, conn)
    plan = lfem.lfem_assemble_symbolic(mesh, r0, r1)
    lfem.lfem_plan_set_variant(plan, {"auto": lfem.LFEM_NUMERIC_AUTO, "v0": lfem.LFEM_NUMERIC_V0,
                                      "tiled": lfem.LFEM_NUMERIC_TILED, "rows": lfem.LFEM_NUMERIC_V0}[args.variant])
    out = torch.empty((nc, plan.n_rows), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lfem.lfem_assemble_rhs(plan, k, None, u, out)  # first call builds the row incidence lists
    torch.cuda.synchronize()
    first_ms = 1e3 * (time.perf_counter() - t0)
    for _ in range(1, args.warmup):
        lfem.lfem_assemble_rhs(plan, k, None, u, out)
    lfem.lfem_plan_check(plan)
    # per-kernel events inside the timed region (event pool filled by as many profiled warm-up calls)
    lfem.lfem_profile_enable(plan, True)
    for _ in range(min(args.steps, 500)):
        lfem.lfem_assemble_rhs(plan, k, None, u, out)
    torch.cuda.synchronize()
    lfem.lfem_profile_read(plan)
    alg = rhs_alg_bytes(plan.n_elems_local, m.nref, m.n_nodes, plan.n_rows, nc)
    flush = name in FLUSH_L2
    flush_buf = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device=dev) if flush else None
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for t in range(args.steps):
        if flush:
            flush_buf.zero_()
        ev[t][0].record(stream)
        lfem.lfem_assemble_rhs(plan, k, None, u, out)
        ev[t][1].record(stream)
    torch.cuda.synchronize()
    elapsed_ms = sum(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        dist.barrier()
    lfem.lfem_plan_check(plan)
    prof = lfem.lfem_profile_read(plan)  # the timed calls' own kernel times
    lfem.lfem_profile_enable(plan, False)
    nprof = args.steps
    clk = clocks.stop()
    tmax = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    elapsed_ms = float(tmax)
    ms_per_step = elapsed_ms / args.steps
    value = m.n_elems * args.steps / (elapsed_ms * 1e-3)

    # e2e through the public API: pinned host coords + u -> device, lfem_assemble_rhs, device -> pinned host
    e2e = None
    if not args.no_e2e:
        coords_h = torch.as_tensor(m.coords).pin_memory()
        u_h = torch.as_tensor(u_np).pin_memory()
        out_h = torch.empty((nc, plan.n_rows), dtype=torch.float64, pin_memory=True)
        c_d, u_d = torch.empty_like(coords), torch.empty_like(u)
        ke = max(1, min(args.steps, args.e2e_steps))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ke):
            c_d.copy_(coords_h, non_blocking=True)
            u_d.copy_(u_h, non_blocking=True)
            lfem.lfem_assemble_rhs(plan, k, c_d, u_d, out)
            out_h.copy_(out, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        assert torch.equal(out_h, out.cpu()), "e2e result differs from the device path"
        e2e = {"value": m.n_elems * ke / (float(te) * 1e-3), "unit": "elements/s",
               "h2d_bytes_per_step": int((coords_h.numel() + u_h.numel()) * 8 * world),
               "d2h_bytes_per_step": int(m.n_nodes * nc * 8), "api": "lfem_assemble_rhs (+ pinned H2D/D2H copies)",
               "steps": ke}

    # verification (untimed): per-component sums of the owned rows, all-reduced over the ranks
    vsum = out.sum(dim=1).double()
    if world > 1:
        dist.all_reduce(vsum)
    verify = {"component_sums": [float(x) for x in vsum.cpu()]}
    hbm, peak_src = peaks()
    step_kernel_ms = sum(v[0] for v in prof.values()) / max(1, nprof)
    achieved = alg / (step_kernel_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp))
        tr = [tj.get(f"{name}-{kind}:{kn}") for kn in prof]
        traffic = sum(tr) if tr and all(x is not None for x in tr) else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "kernel": "+".join(prof), "algorithmic_bytes_per_launch": int(alg),
                "kernel_ms": step_kernel_ms, "peak_source": peak_src,
                "per_kernel_ms": {kn: v[0] / max(1, v[1]) for kn, v in prof.items()},
                "note": "algorithmic bytes of the whole step (two kernels); traffic = their ncu DRAM sum"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        nt = os.cpu_count() or 1

        def call(rows):
            oracle.assemble_rhs_rows(m, u_np, kind, rows=rows, nthreads=nt)
        rows = _oracle_rows_for(m, None, None, args.cpu_seconds, nt, call=call)
        t0 = time.perf_counter()
        call(np.arange(rows, dtype=np.int64))
        dt = time.perf_counter() - t0
        cpu = {"value": m.n_elems * rows / m.n_nodes / dt, "unit": "elements/s", "cores": nt, "kind": "oracle",
               "sample": f"rows [0, {rows}) of {m.n_nodes} ({dt:.1f} s); elements/s = n_elems * rows/n_rows / t"}
    if rank == 0:
        line = {"metric": metric_rhs(kind), "value": value,
                "unit": "elements/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (seeded generators, lfem_inputs)",
                "config": config_rhs(name, m, kind, nc, world, args.variant),
                "first_call_ms": first_ms, "generate_s": gen_s,
                "gpu_launches": lfem.lfem_rhs_launches(plan, k) * args.steps,
                "roofline": roofline, "clocks": clk, "e2e": e2e, "cpu_baseline": cpu, "verify": verify}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- GPU leg: Dziuk MCF (N3)
MCF_LEVEL = {"C2": 7, "C5": 10}


def run_mcf(args):
    """One step = lfem_mcf_step (assembly of M, A at x^{n-1} + K = M + tau A + PCG for the three
    coordinates) on the paper's Dziuk surface at the config's icosphere level, P2, tau = 0.005
    (P:842).  The CG needs the whole mesh: with N ranks every rank runs an independent replica."""
    import torch
    import torch.distributed as dist

    import lfem_inputs as li
    from paper_2605_14035_b200 import lfem

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("LFEM_BENCH_DEVICE") is not None:
        local = int(os.environ["LFEM_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("LFEM_BENCH_BACKEND", "nccl")
        dist.init_process_group(backend, device_id=dev) if backend == "nccl" else dist.init_process_group(backend)
    level = MCF_LEVEL.get(args.config, 7)
    tau, tol = 0.005, 1e-10
    t0 = time.time()
    m = li.dziuk_surface(level, 2)
    gen_s = time.time() - t0
    coords = torch.as_tensor(m.coords).to(dev)
    conn = torch.as_tensor(m.conn).to(dev)
    mesh = lfem.lfem_mesh_create(m.domain, m.order, m.quad, coords, conn)
    plan = lfem.lfem_assemble_symbolic(mesh, 0, m.n_nodes)
    x = coords.clone()
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()
    iters = []
    for _ in range(args.warmup):
        iters.append(lfem.lfem_mcf_step(plan, tau, x, y, tol=tol))
        x, y = y, x
    lfem.lfem_plan_check(plan)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    it_timed = []
    for _ in range(args.steps):
        it_timed.append(lfem.lfem_mcf_step(plan, tau, x, y, tol=tol))
        x, y = y, x
    e1.record(stream)
    torch.cuda.synchronize()
    elapsed_ms = e0.elapsed_time(e1)
    lfem.lfem_plan_check(plan)
    # per-kernel profile over a few more steps (assembly kernel(s) and the CG SpMM)
    lfem.lfem_profile_enable(plan, True)
    nprof = 3
    it_prof = []
    t0p = torch.cuda.Event(enable_timing=True)
    t1p = torch.cuda.Event(enable_timing=True)
    t0p.record(stream)
    for _ in range(nprof):
        it_prof.append(lfem.lfem_mcf_step(plan, tau, x, y, tol=tol))
        x, y = y, x
    t1p.record(stream)
    prof = lfem.lfem_profile_read(plan)
    lfem.lfem_profile_enable(plan, False)
    torch.cuda.synchronize()
    prof_step_ms = t0p.elapsed_time(t1p) / nprof
    clk = clocks.stop()
    tmax = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    elapsed_ms = float(tmax)
    ms_per_step = elapsed_ms / args.steps
    value = world * m.n_elems * args.steps / (elapsed_ms * 1e-3)
    hbm, peak_src = peaks()
    asm = {k: v for k, v in prof.items() if k != "k_spmm3"}
    asm_ms = sum(v[0] for v in asm.values()) / nprof
    spmm_ms, spmm_n = prof.get("k_spmm3", (0.0, 0))
    n, nnz = m.n_nodes, plan.nnz
    spmm_bytes = (n + 1) * 8 + nnz * 12 + 2 * n * 24
    asm_bytes = algorithmic_bytes("C2", m.n_elems, m.nref, n, nnz, ("M", "A"), False)
    if spmm_ms / nprof > asm_ms:
        dom, dom_bytes, dom_ms = "k_spmm3", spmm_bytes, spmm_ms / max(1, spmm_n)
    else:
        dom, dom_bytes, dom_ms = "+".join(asm), asm_bytes, asm_ms
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": None, "kernel": dom, "algorithmic_bytes_per_launch": int(dom_bytes), "kernel_ms": dom_ms,
                "peak_source": peak_src,
                "note": "k_spmm3 bytes: row_ptr + col + vals + x and y (each node once); K (nnz*12 B) may sit in L2"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import mcf as omcf
        ms_ = li.dziuk_surface(5, 2)
        t0 = time.perf_counter()
        omcf.mcf_step(ms_, ms_.coords, tau)
        dt = time.perf_counter() - t0
        cpu = {"value": ms_.n_elems / dt, "unit": "elements/s", "cores": os.cpu_count() or 1, "kind": "oracle",
               "sample": f"one oracle MCF step (std::map assembly + SuperLU direct solve) on the level-5 Dziuk "
                         f"surface ({ms_.n_elems} elements, {dt:.2f} s); elements/s = n_elems / t"}
    if rank == 0:
        line = {"metric": "elements/s (Dziuk MCF steps: fp64 assembly of M, A + PCG solve of 3 coordinates)",
                "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak" if world > 1 else "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (the paper's Dziuk surface, P:842)",
                "config": {"workload": f"Dziuk MCF on the P:842 surface, icosphere level {level} P2 ({m.n_elems} "
                                       f"elements, {n} nodes), tau {tau}, CG tol {tol}",
                           "parallelism": "replicas" if world > 1 else "1 GPU"},
                "cg_iterations_mean": float(np.mean(it_timed)),
                "assembly_ms_per_step": asm_ms, "spmm_ms_per_step": spmm_ms / nprof, "profiled_step_ms": prof_step_ms,
                "assembly_share": asm_ms / prof_step_ms, "generate_s": gen_s,
                "gpu_launches": None, "roofline": roofline, "clocks": clk, "e2e": None, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- GPU leg: surface Poisson (N4)
def run_poisson(args):
    """One step = the P:725-728 pipeline on the unit sphere (P2, icosphere level of the config):
    numeric assembly of M and A, the load vectors b = M f_I of f = 6 u for u = x1x2, x2x3, x3x1
    (lfem_assemble_rhs), and the mean-free solve of the three systems (lfem_solve_meanfree)."""
    import torch

    import lfem_inputs as li
    from paper_2605_14035_b200 import lfem

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dev = torch.device("cuda", torch.cuda.current_device())
    level = MCF_LEVEL.get(args.config, 7)
    m = li.sphere_mesh(level, 2)
    x = m.coords
    u = np.stack([x[:, 0] * x[:, 1], x[:, 1] * x[:, 2], x[:, 2] * x[:, 0]], axis=1)
    coords = torch.as_tensor(m.coords).to(dev)
    conn = torch.as_tensor(m.conn).to(dev)
    mesh = lfem.lfem_mesh_create(m.domain, m.order, m.quad, coords, conn)
    plan = lfem.lfem_assemble_symbolic(mesh, 0, m.n_nodes)
    vals = [torch.empty(plan.nnz, dtype=torch.float64, device=dev) for _ in range(2)] + [None]
    f = torch.as_tensor(np.ascontiguousarray((6.0 * u).T)).to(dev)
    bc = torch.empty((3, m.n_nodes), dtype=torch.float64, device=dev)
    b = torch.empty((m.n_nodes, 3), dtype=torch.float64, device=dev)
    uh = torch.empty_like(b)
    stream = torch.cuda.current_stream()
    its = []

    def step():
        lfem.lfem_assemble_numeric(plan, lfem.LFEM_MASS | lfem.LFEM_STIFF, None, vals)
        for k in range(3):
            lfem.lfem_assemble_rhs(plan, lfem.LFEM_RHS_LOAD, None, f[k:k + 1], bc[k:k + 1])
        b.copy_(bc.t())  # component-major -> AoS (the solver's layout)
        its.append(lfem.lfem_solve_meanfree(plan, vals[1], b, uh, tol=1e-10))
    for _ in range(args.warmup):
        step()
    lfem.lfem_plan_check(plan)
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its.clear()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    lfem.lfem_profile_enable(plan, True)
    t0p, t1p = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0p.record(stream)
    step()
    t1p.record(stream)
    prof = lfem.lfem_profile_read(plan)
    lfem.lfem_profile_enable(plan, False)
    torch.cuda.synchronize()
    clk = clocks.stop()
    prof_ms = t0p.elapsed_time(t1p)
    asm_ms = sum(v[0] for k, v in prof.items() if k != "k_spmm3")
    spmm_ms, spmm_n = prof.get("k_spmm3", (0.0, 1))
    n, nnz = m.n_nodes, plan.nnz
    spmm_bytes = (n + 1) * 8 + nnz * 12 + 2 * n * 24
    hbm, peak_src = peaks()
    achieved = spmm_bytes / (spmm_ms / max(1, spmm_n) * 1e-3) / 1e9
    # accuracy of the run: ||u_h - u_I||_M per column
    e = uh - (torch.as_tensor(u).to(dev) - torch.as_tensor(u.mean(axis=0)).to(dev))
    Me = torch.empty_like(e)
    err = []
    for k in range(3):
        ek = e[:, k].contiguous()
        y = torch.empty(n, dtype=torch.float64, device=dev)
        lfem.lfem_spmv(plan, vals[0], ek, y)
        err.append(float(torch.dot(ek, y)) ** 0.5)
    del Me
    line = {"metric": "elements/s (surface Poisson pipeline: fp64 M, A, 3 load vectors, mean-free PCG solve)",
            "value": m.n_elems / (ms * 1e-3), "unit": "elements/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (unit sphere, u = x1x2 etc., f = 6u; P:727)",
            "config": {"workload": f"P2 unit icosphere level {level} ({m.n_elems} elements, {n} nodes), 3 right-hand "
                                   f"sides, PCG tol 1e-10", "parallelism": "1 GPU"},
            "pcg_iterations_mean": float(np.mean(its)), "assembly_ms": asm_ms, "spmm_ms": spmm_ms,
            "profiled_step_ms": prof_ms, "error_M_norm": err,
            "gpu_launches": None,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": None, "kernel": "k_spmm3", "algorithmic_bytes_per_launch": int(spmm_bytes),
                         "kernel_ms": spmm_ms / max(1, spmm_n), "peak_source": peak_src},
            "clocks": clk, "e2e": None, "cpu_baseline": None}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU leg
def run_lfem(args):
    import torch
    import torch.distributed as dist

    from paper_2605_14035_b200 import lfem
    from paper_2605_14035_b200.partition import partition_rows

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}")
    # test-only overrides (exercise the multi-rank path on one GPU): LFEM_BENCH_DEVICE pins every rank to
    # one device, LFEM_BENCH_BACKEND=gloo replaces NCCL (NCCL refuses two ranks on one GPU)
    if os.environ.get("LFEM_BENCH_DEVICE") is not None:
        local = int(os.environ["LFEM_BENCH_DEVICE"])
    backend = os.environ.get("LFEM_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init (ranks, NVLink / NVLS paths) in the log
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        log(f"rank {rank}/{world}: {backend} process group on cuda:{local}"
            + (f", NCCL {torch.cuda.nccl.version()}" if backend == "nccl" else ""))
    name = args.config

    # ---- inputs: rank 0 generates (seeded), broadcast over NCCL (plumbing, untimed)
    gen_s = 0.0
    if rank == 0:
        m, gen_s = build_mesh(name)
        meta = torch.tensor([m.n_nodes, m.n_elems, m.nref, m.domain, m.order, m.quad,
                             1 if m.coeff is not None else 0], dtype=torch.int64, device=dev)
    else:
        m = None
        meta = torch.empty(7, dtype=torch.int64, device=dev)
    if world > 1:
        dist.broadcast(meta, 0)
    n_nodes, n_elems, nref, domain, order, quad, has_coeff = [int(x) for x in meta.tolist()]
    if rank == 0:
        coords = torch.as_tensor(m.coords).to(dev)
        conn = torch.as_tensor(m.conn).to(dev)
        coeff = torch.as_tensor(m.coeff).to(dev) if has_coeff else None
        kinds = tuple(m.extra["kinds"])
        extra_uB = torch.as_tensor(m.extra["uB"]).to(dev) if "uB" in m.extra else None
    else:
        coords = torch.empty((n_nodes, 3), dtype=torch.float64, device=dev)
        conn = torch.empty((n_elems, nref), dtype=torch.int32, device=dev)
        coeff = torch.empty(n_nodes, dtype=torch.float64, device=dev) if has_coeff else None
        kinds = None
        extra_uB = torch.empty(n_nodes, dtype=torch.float64, device=dev) if name == "C3" else None
    if world > 1:
        dist.broadcast(coords, 0)
        dist.broadcast(conn, 0)
        if coeff is not None:
            dist.broadcast(coeff, 0)
        if extra_uB is not None:
            dist.broadcast(extra_uB, 0)
        obj = [kinds]
        dist.broadcast_object_list(obj, 0)
        kinds = obj[0]
    kmask = sum(KIND_BITS[k] for k in kinds)

    # ---- partition + symbolic (one-time, timed separately)
    conn_np = conn.cpu().numpy() if world > 1 else None
    bounds = partition_rows(conn_np, n_nodes, world) if world > 1 else [0, n_nodes]
    r0, r1 = bounds[rank], bounds[rank + 1]
    stream = torch.cuda.current_stream()
    mesh = lfem.lfem_mesh_create(domain, order, quad, coords, conn)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = lfem.lfem_assemble_symbolic(mesh, r0, r1)
    torch.cuda.synchronize()
    symbolic_ms = 1e3 * (time.perf_counter() - t0)
    variant = {"auto": lfem.LFEM_NUMERIC_AUTO, "v0": lfem.LFEM_NUMERIC_V0, "tiled": lfem.LFEM_NUMERIC_TILED,
               "rows": lfem.LFEM_NUMERIC_ROWS}[args.variant]
    lfem.lfem_plan_set_variant(plan, variant)
    vals = [None, None, None]
    for k in kinds:
        vals[KIND_INDEX[k]] = torch.empty(plan.nnz, dtype=torch.float64, device=dev)

    # C3: u(t) = cos(2 pi t/100) uA + sin(2 pi t/100) uB (reading G12) by lfem_axpby each step
    u_work = torch.empty_like(coeff) if (name == "C3" and coeff is not None) else None

    def step(t):
        cf = coeff
        if u_work is not None:
            th = 2 * math.pi * (t % 100) / 100
            lfem.lfem_axpby(math.cos(th), coeff, math.sin(th), extra_uB, u_work)
            cf = u_work
        lfem.lfem_assemble_numeric(plan, kmask, cf, vals)

    # global sizes
    tot = torch.tensor([plan.nnz, plan.n_elems_local], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(tot)
    nnz_total, elems_local_total = int(tot[0]), int(tot[1])
    alg_bytes_rank = algorithmic_bytes(name, plan.n_elems_local, nref, plan.n_rows, plan.nnz, kinds, has_coeff)
    alg_bytes_total = algorithmic_bytes(name, n_elems, nref, n_nodes, nnz_total, kinds, has_coeff)
    flush = name in FLUSH_L2
    flush_buf = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device=dev) if flush else None

    # first call builds the TILED variant's tile plan (one-time, like the symbolic phase): timed apart
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step(0)
    torch.cuda.synchronize()
    first_call_ms = 1e3 * (time.perf_counter() - t0)
    for t in range(1, args.warmup):
        step(t)
    lfem.lfem_plan_check(plan)
    # per-kernel CUDA events are recorded INSIDE the timed region (the roofline's kernel time is the
    # timed launches' own, not a separate pass): fill the event pool with as many profiled steps first
    # A step of ONE kernel launch (C1, C2, C5: k_tiled) needs no extra events: the timed region's own
    # events bracket exactly its launches, so its per-step time is the kernel's launch duration.
    single = lfem.lfem_numeric_launches(plan, kmask) == 1 and u_work is None
    lfem.lfem_profile_enable(plan, True)
    for t in range(min(args.steps, 500) if not single else 1):
        step(t)
    torch.cuda.synchronize()
    warm_prof = lfem.lfem_profile_read(plan)
    if single:
        lfem.lfem_profile_enable(plan, False)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    # ---- timed region (device time, max over ranks)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if flush:
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for t in range(args.steps):
            flush_buf.zero_()
            ev[t][0].record(stream)
            step(t)
            ev[t][1].record(stream)
        torch.cuda.synchronize()
        elapsed_ms = sum(a.elapsed_time(b) for a, b in ev)
    else:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for t in range(args.steps):
            step(t)
        e1.record(stream)
        torch.cuda.synchronize()
        elapsed_ms = e0.elapsed_time(e1)
    if world > 1:
        dist.barrier()
    lfem.lfem_plan_check(plan)
    # per-kernel times of the timed launches (events recorded around each kernel on its stream)
    prof = lfem.lfem_profile_read(plan)
    lfem.lfem_profile_enable(plan, False)
    if single and warm_prof:
        prof = {next(iter(warm_prof)): (elapsed_ms, args.steps)}
    nprof = args.steps
    # --graph: the same numeric step captured once into a CUDA graph and replayed (SURVEY §8(d).6:
    # launch overhead of the small configs); the graph's output is checked against the eager step
    graph = None
    if args.graph and u_work is None:
        ref = [v.clone() if v is not None else None for v in vals]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            lfem.lfem_assemble_numeric(plan, kmask, coeff, vals)
        torch.cuda.synchronize()
        for v in vals:
            if v is not None:
                v.zero_()
        g.replay()
        torch.cuda.synchronize()
        same = all(torch.equal(a, b) for a, b in zip(vals, ref) if a is not None)
        gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        gs = torch.cuda.current_stream()
        for t in range(args.steps):
            if flush:
                flush_buf.zero_()
            gev[t][0].record(gs)
            g.replay()
            gev[t][1].record(gs)
        torch.cuda.synchronize()
        gms = sum(a.elapsed_time(b) for a, b in gev) / args.steps
        graph = {"ms_per_step": gms, "value": n_elems / (gms * 1e-3), "eager_ms_per_step": None,
                 "bitwise_equal_to_eager": bool(same), "note": "one CUDA-graph replay per step, events around each"}
        del g
    clk = clocks.stop()
    evals, n_tiles = lfem.lfem_numeric_stats(plan)

    # per-rank shape of the partition (N > 1): rows, nnz, elements assembled (halo included), device ms
    mine_info = torch.tensor([plan.n_rows, plan.nnz, plan.n_elems_local, elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        parts = [torch.empty_like(mine_info) for _ in range(world)]
        dist.all_gather(parts, mine_info)
        info = torch.stack(parts).cpu().numpy()
    else:
        info = mine_info.cpu().numpy()[None, :]
    ranks = {"rows": [int(v) for v in info[:, 0]], "nnz": [int(v) for v in info[:, 1]],
             "n_elems_local": [int(v) for v in info[:, 2]],
             "ms_per_step": [float(v) / args.steps for v in info[:, 3]],
             "nnz_spread_max_over_min": float(info[:, 1].max() / max(1.0, info[:, 1].min())),
             "halo_factor_per_rank": [float(v) * world / n_elems for v in info[:, 2]]}
    tmax = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    elapsed_ms = float(tmax)
    ms_per_step = elapsed_ms / args.steps
    value = n_elems * args.steps / (elapsed_ms * 1e-3)

    # ---- e2e through the public API with HOST buffers (pinned), H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        coords_h = coords.cpu().pin_memory()
        vals_h = [torch.empty(plan.nnz, dtype=torch.float64, pin_memory=True) if vals[i] is not None else None
                  for i in range(3)]
        ke = max(1, min(args.steps, args.e2e_steps))
        # per-step coefficient on the host (C3: u(t), reading G12; else the config's u), pinned, copied in the timed region
        if coeff is None:
            coeffs_h = [None] * ke
        elif u_work is not None:
            uA, uB = coeff.cpu(), extra_uB.cpu()
            coeffs_h = [(math.cos(2 * math.pi * (t % 100) / 100) * uA + math.sin(2 * math.pi * (t % 100) / 100) * uB)
                        .pin_memory() for t in range(ke)]
        else:
            coeffs_h = [coeff.cpu().pin_memory()] * ke
        lfem.lfem_assemble_numeric_host(plan, kmask, coords_h, coeffs_h[0], vals_h)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for t in range(ke):
            lfem.lfem_assemble_numeric_host(plan, kmask, coords_h, coeffs_h[t], vals_h)
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        h2d = (n_nodes * 24 + (n_nodes * 8 if coeff is not None else 0)) * world
        e2e = {"value": n_elems * ke / (float(te) * 1e-3), "unit": "elements/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(nnz_total * 8 * len(kinds)),
               "api": "lfem_assemble_numeric_host", "steps": ke}
        # e2e must produce the same bits as the device path with the same inputs
        cf_last = coeffs_h[-1].to(dev) if coeffs_h[-1] is not None else None
        lfem.lfem_assemble_numeric(plan, kmask, cf_last, vals)
        torch.cuda.synchronize()
        for i in range(3):
            if vals[i] is not None:
                assert torch.equal(vals_h[i], vals[i].cpu()), "e2e values differ from the device path"
        del vals_h, coords_h, coeffs_h

    # ---- multi-GPU verification: NCCL all_gather of x + local SpMV; checksums all-reduced
    verify = None
    if args.verify or world > 1:
        x = coords[:, 0].contiguous()
        shard = (n_nodes + world - 1) // world
        xs = torch.zeros(shard * world, dtype=torch.float64, device=dev)
        mine = x[rank * shard:min(n_nodes, (rank + 1) * shard)]
        loc = torch.zeros(shard, dtype=torch.float64, device=dev)
        loc[:mine.numel()] = mine
        if world > 1:
            parts = [torch.empty_like(loc) for _ in range(world)]
            dist.all_gather(parts, loc)
            xs = torch.cat(parts)
        else:
            xs = loc
        xg = xs[:n_nodes]
        y = torch.empty(plan.n_rows, dtype=torch.float64, device=dev)
        one = torch.ones(n_nodes, dtype=torch.float64, device=dev)
        sums = torch.zeros(3, dtype=torch.float64, device=dev)
        lfem.lfem_spmv(plan, vals[0], one, y)
        sums[0] = y.sum()
        k2 = vals[1] if vals[1] is not None else vals[2]
        tr = 0.0
        for c in range(3):
            xc = coords[:, c].contiguous()
            lfem.lfem_spmv(plan, k2, xc, y)
            tr = tr + torch.dot(xc[r0:r1], y)
        sums[1] = tr
        lfem.lfem_spmv(plan, k2, xg, y)
        sums[2] = torch.dot(xg[r0:r1], y)
        if world > 1:
            dist.all_reduce(sums)
        verify = {"one_M_one": float(sums[0]), "trace_xAx": float(sums[1]), "xAx_gathered": float(sums[2]),
                  "allgather_bytes": int(shard * world * 8)}

    # ---- roofline of the numeric step
    hbm, peak_src = peaks()
    kern = sorted(prof.items(), key=lambda kv: -kv[1][0])
    dom_name, (dom_ms, dom_n) = kern[0] if kern else ("numeric", (ms_per_step * nprof, nprof))
    step_kernel_ms = sum(v[0] for v in prof.values()) / max(1, nprof)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp))
        traffic = tj.get(f"{name}:{dom_name}")
    achieved = alg_bytes_rank / (step_kernel_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic,
                "kernel": "+".join(k for k, _ in kern) if len(kern) > 1 else dom_name,
                "algorithmic_bytes_per_launch": int(alg_bytes_rank), "kernel_ms": step_kernel_ms,
                "peak_source": peak_src,
                "per_kernel_ms": {k: v[0] / max(1, v[1]) for k, v in prof.items()},
                "frac_of_8TBs_spec": alg_bytes_rank / (step_kernel_ms * 1e-3) / 8e12}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        mh = m
        rate, rows, dt, nt, _ = oracle_sample(mh, kinds, mh.coeff if has_coeff else None, args.cpu_seconds)
        cpu = {"value": rate, "unit": "elements/s", "cores": nt, "kind": "oracle",
               "sample": f"rows [0, {rows}) of {n_nodes} ({dt:.1f} s); elements/s = n_elems * rows/n_rows / t"}

    if rank == 0:
        line = {
            "metric": METRIC_MATRICES,
            "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded generators, lfem_inputs)",
            "config": config_matrices(name, m, kinds, world, args.variant), "nnz": nnz_total,
            "nnz_per_s": nnz_total * args.steps / (elapsed_ms * 1e-3),
            "value_slots_per_s": len(kinds) * nnz_total * args.steps / (elapsed_ms * 1e-3),
            "symbolic_ms": symbolic_ms, "first_numeric_call_ms": first_call_ms, "generate_s": gen_s,
            "halo_factor": elems_local_total / n_elems, "ranks": ranks if world > 1 else None,
            "gpu_launches": (lfem.lfem_numeric_launches(plan, kmask) + (1 if u_work is not None else 0)) * args.steps,
            "roofline": roofline,
            "fp64": {"flop_model_per_elem": FLOP_PER_ELEM[name],
                     "achieved_tflops": FLOP_PER_ELEM[name] * plan.n_elems_local / (step_kernel_ms * 1e-3) / 1e12,
                     # element evaluations the kernel actually performs (tile halo recompute included)
                     "elem_evals_per_step": evals, "processed_factor": evals / max(1, plan.n_elems_local),
                     "executed_tflops": FLOP_PER_ELEM[name] * evals / (step_kernel_ms * 1e-3) / 1e12},
            "clocks": clk, "e2e": e2e, "cpu_baseline": cpu, "verify": verify,
        }
        if graph is not None:
            graph["eager_ms_per_step"] = ms_per_step
            line["graph"] = graph
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C4", "C5", "C4P1", "CURVE2"])
    ap.add_argument("--impl", default="lfem", choices=["lfem", "reference"])
    ap.add_argument("--variant", default="auto", choices=["auto", "v0", "tiled", "rows"])
    ap.add_argument("--natural", action="store_true", help="C2 without the SFC renumbering (sensitivity point)")
    ap.add_argument("--cpu-threads", type=int, default=None, help="threads of the oracle cpu_baseline sample")
    ap.add_argument("--graph", action="store_true",
                    help="also time the numeric step replayed from a captured CUDA graph (launch overhead)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--verify", action="store_true")
    ap.add_argument("--poisson", action="store_true",
                    help="time the surface Poisson pipeline (SURVEY §8(f) N4) at the config's icosphere level")
    ap.add_argument("--mcf", action="store_true",
                    help="time Dziuk MCF steps (SURVEY §8(f) N3) on the paper's surface at the config's level")
    ap.add_argument("--quad8", action="store_true",
                    help="P2 triangle configs with Dunavant's 16-point degree-8 rule (the paper's load-vector rule)")
    ap.add_argument("--rhs", default=None, choices=["load", "kll"],
                    help="time the right-hand side (SURVEY §8(f) N1) instead of the matrices")
    args = ap.parse_args()
    global QUAD8, NATURAL, CPU_THREADS
    QUAD8 = args.quad8
    NATURAL = args.natural
    CPU_THREADS = args.cpu_threads
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.rhs:
        return run_rhs(args)
    if args.mcf:
        return run_mcf(args)
    if args.poisson:
        return run_poisson(args)
    return run_lfem(args)


if __name__ == "__main__":
    sys.exit(main())
