#!/bin/bash
# ncu capture of one kernel: CFG, VAR, KREGEX env
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CFG=${CFG:-C2}; VAR=${VAR:-tiled}; KREGEX=${KREGEX:-k_tiled}; TAG=${TAG:-prof}
CMD="python bench.py --config $CFG --variant $VAR --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 3 -c 1 -o gpurun_out/$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu exit $?"
tail -5 gpurun_out/ncu_$TAG.log
