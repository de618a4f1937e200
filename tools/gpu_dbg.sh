#!/bin/bash
# Diagnostic decomposition: SPICE_DEBUG_MODE bit0 no smem reductions, bit1 no synapse loads
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
for m in ${MODES:-0 1 3}; do
  SPICE_DEBUG_MODE=$m timeout 200 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline --profile-steps 20 --e2e-steps 10 $EXTRA > gpurun_out/dbg_$m.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/dbg_$m.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('mode $m ms/step %.4f'%d['ms_per_step'], {x:round(y*1e3,1) for x,y in k.items()})" 2>&1 | tail -1
done
