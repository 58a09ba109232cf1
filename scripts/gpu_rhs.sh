#!/bin/bash
# N1 right-hand side evidence: bench lines (KLL on C5, load on C5 and C4), ncu launch list and
# ncu --set full of the two RHS kernels on C5 KLL
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 900 python bench.py --rhs kll --steps 20 --warmup 5 > gpurun_out/${TAG}_rhs_kll_C5.json 2> gpurun_out/${TAG}_rhs_kll_C5.log; echo "kll C5 exit $?"
tail -c 600 gpurun_out/${TAG}_rhs_kll_C5.json
for spec in load:C5 load:C4; do k=${spec%%:*}; c=${spec##*:}
  timeout 900 python bench.py --rhs $k --config $c --steps 20 --warmup 5 > gpurun_out/${TAG}_rhs_${k}_$c.json 2> gpurun_out/${TAG}_rhs_${k}_$c.log; echo "$k $c exit $?"
done
if [ "${NCU:-1}" = "1" ]; then
CMD="python bench.py --rhs kll --steps 2 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_rhs_launches.csv $CMD > gpurun_out/${TAG}_rhs_ncu_launches.log 2>&1
echo "ncu launches exit $?"
CMD2="python bench.py --rhs kll --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --set full --clock-control none --import-source on -k regex:"k_rhs_elem|k_rhs_reduce" -s 4 -c 2 -o gpurun_out/${TAG}_rhs_kll_full $CMD2 > gpurun_out/${TAG}_rhs_ncu_full.log 2>&1
echo "ncu full exit $?"
fi
