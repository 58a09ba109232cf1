#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
run() { # cfg variant rows debug tag
  LFEM_TILE_ROWS=$3 LFEM_DEBUG_TILED=$4 timeout 600 python bench.py --config $1 --variant $2 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$5.json 2> gpurun_out/b_$5.log
  python -c "import json,sys; d=json.load(open('gpurun_out/b_$5.json')); r=d['roofline']; print('$5', 'ms/step %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'])" 2>&1 | tail -1
}
run C5 tiled 256 0 full
run C5 tiled 256 1 skipA
run C5 tiled 256 2 skipB
run C5 tiled 256 3 skipAB
run C5 tiled 192 0 full192
run C2 tiled 256 0 C2full
run C3 tiled 512 0 C3full
