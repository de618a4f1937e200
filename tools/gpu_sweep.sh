#!/bin/bash
# Tile/lane sweep of the synth 3e9 bench.  Usage: bash tools/gpu_sweep.sh TAG "tw:gs:c ..."
TAG=$1; shift
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
for spec in $@; do
  IFS=: read tw gs c <<< "$spec"
  SPICE_GROUP_LANES=$gs timeout 200 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline --profile-steps 20 --e2e-steps 10 --tile-width $tw --ctas-per-tile $c > gpurun_out/sweep_${TAG}_${tw}_${gs}_${c}.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/sweep_${TAG}_${tw}_${gs}_${c}.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('tw $tw gs $gs c $c ms/step %.4f frac %.3f'%(d['ms_per_step'],d['roofline']['frac']), {x:round(y*1e3,1) for x,y in k.items()})" 2>&1 | tail -1
done
