#!/bin/bash
# Round-2 evidence: FP64 peak microbenchmark, bench lines of every config and workload, the ncu
# launch list of the default bench command, and ncu --set full captures of the dominant kernels
# (C5 / C2 / C3 k_tiled; C4 k_elem_v0 + k_slot_reduce).  All ncu runs of one gpurun call count as
# one tool use; every ncu command runs only after the same command exited 0 without ncu.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
if [ -z "$SKIP_PEAK" ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak scripts/microbench/fp64_peak.cu && \
    /tmp/fp64_peak > gpurun_out/${TAG}_fp64_peak.txt 2>&1; echo "fp64 peak exit $?"
fi
B="timeout 900 python bench.py"
if [ -z "$SKIP_BENCH" ]; then
  $B > gpurun_out/${TAG}_bench_C5.json 2> gpurun_out/${TAG}_bench_C5.log; echo "bench C5 exit $?"
  for cfg in C1 C2 C3 C4 C4P1 CURVE2; do
    $B --config $cfg --steps 30 --warmup 5 > gpurun_out/${TAG}_bench_$cfg.json 2> gpurun_out/${TAG}_bench_$cfg.log
    echo "bench $cfg exit $?"
  done
  $B --config C5 --quad8 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_C5_quad8.json 2> gpurun_out/${TAG}_bench_C5_quad8.log; echo "quad8 exit $?"
  $B --config C5 --rhs kll --steps 20 --warmup 3 > gpurun_out/${TAG}_bench_rhs_kll_C5.json 2> gpurun_out/${TAG}_bench_rhs_kll_C5.log; echo "rhs kll exit $?"
  $B --config C5 --rhs load --steps 20 --warmup 3 > gpurun_out/${TAG}_bench_rhs_load_C5.json 2> gpurun_out/${TAG}_bench_rhs_load_C5.log; echo "rhs load exit $?"
  $B --config C4 --rhs load --steps 20 --warmup 3 > gpurun_out/${TAG}_bench_rhs_load_C4.json 2> gpurun_out/${TAG}_bench_rhs_load_C4.log; echo "rhs load C4 exit $?"
  $B --config C2 --mcf --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_mcf_C2.json 2> gpurun_out/${TAG}_bench_mcf_C2.log; echo "mcf exit $?"
  $B --config C2 --poisson --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_poisson_C2.json 2> gpurun_out/${TAG}_bench_poisson_C2.log; echo "poisson exit $?"
  LFEM_REF_BUDGET_S=60 $B --impl reference --steps 10 --warmup 3 > gpurun_out/${TAG}_reference_C5.json 2> gpurun_out/${TAG}_reference_C5.log; echo "reference exit $?"
fi
if [ -z "$SKIP_NCU" ]; then
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
  $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
  echo "ncu launches exit $?"
  for cfg in C5 C2 C3; do
    CMDF="python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
    $CMDF > gpurun_out/${TAG}_plain_$cfg.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:k_tiled -s 3 -c 1 -o gpurun_out/${TAG}_${cfg}_full $CMDF > gpurun_out/${TAG}_ncu_full_$cfg.log 2>&1
    echo "ncu full $cfg exit $?"
    # summarise here (the reports exceed what gpurun brings back), keep the text only
    LCSV=-; [ $cfg = C5 ] && LCSV=gpurun_out/${TAG}_launches.csv
    python scripts/ncu_summary.py gpurun_out/${TAG}_${cfg}_full.ncu-rep $LCSV gpurun_out/profiles_${TAG} $cfg > /dev/null 2>&1
    ncu -i gpurun_out/${TAG}_${cfg}_full.ncu-rep --page raw --csv > gpurun_out/profiles_${TAG}/ncu_${cfg}_raw.csv 2>/dev/null
    rm -f gpurun_out/${TAG}_${cfg}_full.ncu-rep
  done
  CMD4="python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
  $CMD4 > gpurun_out/${TAG}_plain_C4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"${C4_KERNELS:-k_elem_v0|k_slot_reduce}" -s ${C4_SKIP:-6} -c ${C4_COUNT:-2} -o gpurun_out/${TAG}_C4_full $CMD4 > gpurun_out/${TAG}_ncu_full_C4.log 2>&1
  echo "ncu full C4 exit $?"
  for row in 0 1; do
    NCU_KERNEL_ROW=$row python scripts/ncu_summary.py gpurun_out/${TAG}_C4_full.ncu-rep - gpurun_out/profiles_${TAG} C4 > /dev/null 2>&1
  done
  ncu -i gpurun_out/${TAG}_C4_full.ncu-rep --page raw --csv > gpurun_out/profiles_${TAG}/ncu_C4_raw.csv 2>/dev/null
  rm -f gpurun_out/${TAG}_C4_full.ncu-rep
  du -sh gpurun_out
fi
