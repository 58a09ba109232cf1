#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --config C2 --variant tiled --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
for d in ${DBGS:-2 1}; do
  LFEM_DEBUG_TILED=$d $CMD > gpurun_out/plain_dbg$d.log 2>&1 && \
  LFEM_DEBUG_TILED=$d ncu --set full --clock-control none --import-source on -k regex:k_tiled -s 3 -c 1 -o gpurun_out/c2_dbg${d}${TAG} $CMD > gpurun_out/ncu_dbg$d.log 2>&1
  echo "dbg $d exit $?"
done
