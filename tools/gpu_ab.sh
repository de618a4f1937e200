#!/bin/bash
# A/B of env settings on the synth bench: bash tools/gpu_ab.sh "ENV1=.. ENV2=.." "ENV=.." ...
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
i=0
for spec in "$@"; do
  i=$((i+1))
  env $spec timeout 200 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline --profile-steps 20 --e2e-steps 10 $EXTRA > gpurun_out/ab_$i.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_$i.log').read().strip().splitlines()[-1]); k=d['roofline']['kernel_ms']; print('[$spec] ms/step %.4f frac %.3f'%(d['ms_per_step'],d['roofline']['frac']), {x:round(y*1e3,1) for x,y in k.items()})" 2>&1 | tail -1
done
