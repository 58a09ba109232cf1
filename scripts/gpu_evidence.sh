#!/bin/bash
# round evidence: default bench line, every config's bench line, ncu launch list (same command as the
# default bench, shortened), ncu --set full of the dominant kernels (C5 k_tiled; C4 k_elem_v0 + k_slot_reduce)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench_C5.json 2> gpurun_out/${TAG}_bench_C5.log; echo "bench C5 exit $?"
for cfg in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $cfg --steps 30 --warmup 5 > gpurun_out/${TAG}_bench_$cfg.json 2> gpurun_out/${TAG}_bench_$cfg.log; echo "bench $cfg exit $?"
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo "ncu launches exit $?"
CMD2="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD2 > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tiled -s 3 -c 1 -o gpurun_out/${TAG}_C5_full $CMD2 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full C5 exit $?"
CMD3="python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD3 > gpurun_out/${TAG}_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_elem_v0|k_slot_reduce" -s 6 -c 2 -o gpurun_out/${TAG}_C4_full $CMD3 > gpurun_out/${TAG}_ncu_full4.log 2>&1
echo "ncu full C4 exit $?"
