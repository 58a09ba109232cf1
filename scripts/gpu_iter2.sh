#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
run() { # cfg variant rows tag
  LFEM_TILE_ROWS=$3 timeout 600 python bench.py --config $1 --variant $2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b_$4.json 2> gpurun_out/b_$4.log
  python -c "import json,sys; d=json.load(open('gpurun_out/b_$4.json')); r=d['roofline']; print('$4', 'ms/step %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'], r['per_kernel_ms'], 'fp64 TF %.2f'%d['fp64']['achieved_tflops'])" 2>&1 | tail -1
}
for R in ${ROWS:-256 128 512}; do run C5 tiled $R C5_R$R; done
run C2 tiled 256 C2_R256
run C3 tiled 512 C3_R512
run C4 v0 0 C4_v0
