#!/bin/bash
# round evidence: default bench line, ncu launch list (same command), ncu --set full of the top kernel, fp64 peak
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.log; echo "bench exit $?"
cat gpurun_out/${TAG}_bench.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo "ncu launches exit $?"
CMD2="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD2 > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tiled -s 3 -c 1 -o gpurun_out/${TAG}_c5_full $CMD2 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full exit $?"
