"""The multi-rank bench path (torchrun, row blocks, verification all-gather +
SpMV + all-reduce) run end to end on one GPU: two ranks pinned to cuda:0 with
the gloo backend (test-only overrides; NCCL refuses two ranks per GPU).  The
distributed checksums must reproduce the single-rank run's and the trace
identity."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(cmd, env):
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_two_ranks_match_one(cfg):
    env = dict(os.environ)
    base = [sys.executable, "bench.py", "--config", cfg, "--steps", "3", "--warmup", "3", "--verify",
            "--no-cpu-baseline", "--no-e2e"]
    one = _run(base + ["--gpus", "1"], env)
    env2 = dict(env, LFEM_BENCH_DEVICE="0", LFEM_BENCH_BACKEND="gloo")
    two = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                "--master-addr", "127.0.0.1", "--master-port", str(_port())] + base[1:] + ["--gpus", "2"], env2)
    assert two["n_gpus"] == 2 and two["nnz"] == one["nnz"]
    # per-rank partition report (N > 1): rows and nnz add up, halo elements counted per rank
    r = two["ranks"]
    assert sum(r["nnz"]) == one["nnz"] and sum(r["rows"]) == one["config"]["n_nodes"]
    assert sum(r["n_elems_local"]) >= one["config"]["n_elems"] and r["nnz_spread_max_over_min"] >= 1.0
    assert one["ranks"] is None
    assert two["gpu_launches"] > 0 and two["value"] > 0
    for k in ("one_M_one", "trace_xAx", "xAx_gathered"):
        a, b = one["verify"][k], two["verify"][k]
        assert abs(a - b) <= 1e-12 * max(1.0, abs(a)), (k, a, b)
    if "A" in two["config"]["kinds"]:  # trace identity sum_k x_k^T A x_k = 2 * area (surface, tr P = 2)
        assert abs(two["verify"]["trace_xAx"] - 2 * two["verify"]["one_M_one"]) <= 1e-9 * two["verify"]["one_M_one"]


def test_two_ranks_rhs_match_one():
    """bench.py --rhs kll over two row-block ranks: the all-reduced component sums equal one rank's."""
    env = dict(os.environ)
    base = [sys.executable, "bench.py", "--config", "C2", "--rhs", "kll", "--steps", "3", "--warmup", "3",
            "--no-cpu-baseline", "--no-e2e"]
    one = _run(base + ["--gpus", "1"], env)
    env2 = dict(env, LFEM_BENCH_DEVICE="0", LFEM_BENCH_BACKEND="gloo")
    two = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                "--master-addr", "127.0.0.1", "--master-port", str(_port())] + base[1:] + ["--gpus", "2"], env2)
    assert two["n_gpus"] == 2 and two["gpu_launches"] > 0 and two["value"] > 0
    for a, b in zip(one["verify"]["component_sums"], two["verify"]["component_sums"]):
        assert abs(a - b) <= 1e-12 * max(1.0, abs(a)), (a, b)
