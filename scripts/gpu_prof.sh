#!/bin/bash
# ncu full capture of one kernel + fp64 peak microbenchmark.  env: CFG VAR KREGEX TAG
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CFG=${CFG:-C5}; VAR=${VAR:-auto}; KREGEX=${KREGEX:-k_tiled}; TAG=${TAG:-prof}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak scripts/microbench/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
cat gpurun_out/fp64_peak.txt
CMD="python bench.py --config $CFG --variant $VAR --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 3 -c 1 -o gpurun_out/$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu exit $?"
tail -3 gpurun_out/ncu_$TAG.log
