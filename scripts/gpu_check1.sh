#!/bin/bash
# first GPU call: parity tests (not slow), smoke, short benches
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --config C2 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.log; echo "exit $?" >> gpurun_out/bench_C2.log
timeout 900 python bench.py --config C5 --steps 50 --warmup 5 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.log; echo "exit $?" >> gpurun_out/bench_C5.log
tail -5 gpurun_out/pytest_gpu.log
cat gpurun_out/bench_C2.json gpurun_out/bench_C5.json
