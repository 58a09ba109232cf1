#!/bin/bash
# snapshot: parity tests (not slow), smoke, bench each config (variants auto/tiled/v0)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
for cfg in C5 C2 C3 C4 C1; do for v in ${VARIANTS:-auto tiled v0}; do
  timeout 600 python bench.py --config $cfg --variant $v --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${cfg}_${v}.json 2> gpurun_out/bench_${cfg}_${v}.log
  echo "$cfg $v exit $?"
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_${cfg}_${v}.json')); r=d['roofline']; print('$cfg $v', 'ms/step %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'], r['per_kernel_ms'], 'fp64 TF %.2f'%d['fp64']['achieved_tflops'], d['clocks'])" 2>&1 | tail -1
done; done
