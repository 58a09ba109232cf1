#!/bin/bash
# The GPU parity suite against the bounds + poison build (scripts/variants/bounds: -DLFEM_BOUNDS=1
# -DLFEM_TILED_POISON=1), the stand-in for compute-sanitizer, then the default build's C5 bench.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
LFEM_SO=scripts/variants/bounds/liblfem.so timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_bounds.log 2>&1; echo "bounds pytest exit $?" >> gpurun_out/pytest_bounds.log
tail -4 gpurun_out/pytest_bounds.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b_C5_default.json 2> gpurun_out/b_C5_default.log
python -c "import json; d=json.load(open('gpurun_out/b_C5_default.json')); print('C5', d['ms_per_step'], d['roofline']['frac'])"
