#!/bin/bash
# Round-2 evidence, part 2: compute-sanitizer (memcheck / racecheck / synccheck / initcheck) on the
# small sanitizer workload, CUDA-graph replay lines for C1 / C2, the natural-order C2 point, and
# single-thread oracle baselines for C1-C3.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/evid2
CS=${CS:-/usr/local/cuda/bin/compute-sanitizer}
$CS --version > gpurun_out/evid2/sanitizer_version.txt 2>&1
if [ -z "$SKIP_SAN" ]; then
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  timeout ${SAN_TIMEOUT:-900} $CS --tool $tool --print-limit 50 python scripts/sanitize_run.py > gpurun_out/evid2/sanitizer_$tool.txt 2>&1
  echo "sanitizer $tool exit $?" | tee -a gpurun_out/evid2/sanitizer_$tool.txt
  tail -3 gpurun_out/evid2/sanitizer_$tool.txt
done
fi
B="timeout 600 python bench.py"
for cfg in C1 C2; do
  $B --config $cfg --graph --steps 200 --warmup 10 --cpu-threads 1 --cpu-seconds 10 > gpurun_out/evid2/bench_${cfg}_graph.json 2> gpurun_out/evid2/bench_${cfg}_graph.log; echo "graph $cfg exit $?"
done
$B --config C2 --natural --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/evid2/bench_C2_natural.json 2> gpurun_out/evid2/bench_C2_natural.log; echo "natural exit $?"
$B --config C3 --steps 20 --warmup 3 --cpu-threads 1 --cpu-seconds 10 --no-e2e > gpurun_out/evid2/bench_C3_cpu1.json 2> gpurun_out/evid2/bench_C3_cpu1.log; echo "C3 cpu1 exit $?"
