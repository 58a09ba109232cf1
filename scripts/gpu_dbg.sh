#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
run() { # cfg variant rows debug tag
  LFEM_TILE_ROWS=$3 LFEM_DEBUG_TILED=$4 timeout 600 python bench.py --config $1 --variant $2 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$5.json 2> gpurun_out/b_$5.log
  python -c "import json,sys; d=json.load(open('gpurun_out/b_$5.json')); r=d['roofline']; print('$5', 'ms/step %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'])" 2>&1 | tail -1
}
run C5 tiled 256 0 full
run C5 tiled 256 1 skipA
run C5 tiled 256 2 skipB
run C5 tiled 256 3 skipAB
run C5 tiled 512 0 full512
run C5 tiled 512 1 skipA512
run C5 tiled 512 2 skipB512
