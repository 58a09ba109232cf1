#!/bin/bash
# iteration: parity tests (not slow) + benches of C5 and C2, variants
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for cfg in ${CONFIGS:-C5 C2}; do
  for v in ${VARIANTS:-tiled v0}; do
    timeout 600 python bench.py --config $cfg --variant $v --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${cfg}_${v}.json 2> gpurun_out/bench_${cfg}_${v}.log
    echo "$cfg $v exit $?"
    python -c "import json,sys; d=json.load(open('gpurun_out/bench_${cfg}_${v}.json')); r=d['roofline']; print('$cfg $v', 'ms/step %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'], r['per_kernel_ms'], 'fp64 TF %.2f'%d['fp64']['achieved_tflops'])" 2>&1 | tail -1
  done
done
