#!/bin/bash
# compare library variants (scripts/variants/<name>/liblfem.so) on configs: VARS="base ru2 ..." CFGS="C5 C2"
# EXTRA="--rhs kll --variant v0" adds bench flags
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in $VARS; do
  so=paper_2605_14035_b200/liblfem.so; [ "$v" != base ] && so=scripts/variants/$v/liblfem.so
  for c in $CFGS; do
    LFEM_SO=$so timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $EXTRA > gpurun_out/v_${v}_$c.json 2> gpurun_out/v_${v}_$c.log
    python -c "import json; d=json.load(open('gpurun_out/v_${v}_$c.json')); print('$v $c $EXTRA', 'ms %.4f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], d['roofline'].get('per_kernel_ms'))" 2>&1 | tail -1
  done
done
