#!/bin/bash
# Same-box A/B of the in-tree library against another build: bash tools/ab_lib.sh OTHER.so [reps]
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
for rep in $(seq ${2:-2}); do
  for lib in "" "$1"; do
    SPICE_LIB=$lib timeout 300 python bench.py --steps 3000 --warmup 50 --no-cpu-baseline --profile-steps 50 --e2e-steps 20 $EXTRA > gpurun_out/ab.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print('${lib:-current}', d['ms_per_step'], d['roofline']['kernel_ms']['fused_in_graph'])"
  done
done
