#!/bin/bash
# timing experiments: role isolation of the tiled kernel (LFEM_DEBUG_TILED) and tile sizes
# SPECS="cfg:rows:debug:tag cfg:rows:debug:tag ..."
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for spec in $SPECS; do
  IFS=: read cfg rows dbg tag <<< "$spec"
  LFEM_TILE_ELEMS=$rows LFEM_DEBUG_TILED=$dbg timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r_$tag.json 2> gpurun_out/r_$tag.log
  python -c "import json,sys; d=json.load(open('gpurun_out/r_$tag.json')); r=d['roofline']; print('$tag', 'ms/step %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'])" 2>&1 | tail -1
done
