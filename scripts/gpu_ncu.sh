#!/bin/bash
# ncu capture of one kernel: CFG, VAR, KREGEX, TAG, SO (library variant, default in-tree) env
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CFG=${CFG:-C2}; VAR=${VAR:-auto}; KREGEX=${KREGEX:-k_tiled}; TAG=${TAG:-prof}
[ -n "$SO" ] && export LFEM_SO=$SO
CMD="python bench.py --config $CFG --variant $VAR --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s ${SKIP:-3} -c 1 -o gpurun_out/$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu $TAG exit $?"
tail -2 gpurun_out/ncu_$TAG.log
