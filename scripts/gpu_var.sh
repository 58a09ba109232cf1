#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "C5 or C3 or tri2 or sphere2 or determinism or partition" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
run() { # so debug tag
  LFEM_SO=$1 LFEM_DEBUG_TILED=$2 timeout 600 python bench.py --config C5 --variant tiled --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$3.json 2> gpurun_out/b_$3.log
  python -c "import json,sys; d=json.load(open('gpurun_out/b_$3.json')); r=d['roofline']; print('$3', 'ms/step %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'])" 2>&1 | tail -1
}
for v in ${VARS:-t192m2r256 t128m3r160 t256m1r384 t384m1r512}; do
  so=scripts/variants/$v/liblfem.so
  run $so 0 ${v}_full
  run $so 1 ${v}_skipA
  run $so 2 ${v}_skipB
done
