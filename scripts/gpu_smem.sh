#!/bin/bash
# shared-memory wavefront accounting of the tile kernel (one C5 / C3 launch each), ncu after a clean run
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
M=l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,sm__cycles_elapsed.avg,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,gpu__time_duration.sum
for cfg in ${CFGS:-C5 C3}; do
  CMD="python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
  $CMD > gpurun_out/smem_plain_$cfg.log 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:k_tiled -s 3 -c 1 --csv $CMD > gpurun_out/smem_$cfg.csv 2> gpurun_out/smem_$cfg.err
  echo "ncu $cfg exit $?"
done
