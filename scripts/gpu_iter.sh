#!/bin/bash
# iteration: parity tests (not slow) + benches (CONFIGS x VARIANTS); optional ncu of one config (NCU_CFG)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_iter.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_iter.log
tail -15 gpurun_out/pytest_iter.log
for cfg in ${CONFIGS:-C5 C2 C3}; do
  for v in ${VARIANTS:-auto}; do
    timeout 600 python bench.py --config $cfg --variant $v --steps ${STEPS:-30} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${cfg}_${v}.json 2> gpurun_out/bench_${cfg}_${v}.log
    echo "$cfg $v exit $?"
    python -c "import json,sys; d=json.load(open('gpurun_out/bench_${cfg}_${v}.json')); r=d['roofline']; print('$cfg $v', 'ms/step %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'], r['per_kernel_ms'], 'fp64 TF %.2f'%d['fp64']['achieved_tflops'], d['clocks'])" 2>&1 | tail -1
  done
done
if [ -n "$NCU_CFG" ]; then
  CMD="python bench.py --config $NCU_CFG --variant ${NCU_VAR:-auto} --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
  $CMD > gpurun_out/plain_ncu.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:${NCU_K:-k_tiled} -s ${NCU_S:-3} -c 1 -o gpurun_out/${NCU_TAG:-prof} $CMD > gpurun_out/ncu.log 2>&1
  echo "ncu exit $?"; tail -2 gpurun_out/ncu.log
fi
