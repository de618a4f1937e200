#!/bin/bash
# Staged-ring A/B: parity, then synth bench at SPICE_RSTAGES = 0 / 4 / 8 and C = 1 / 2.
TAG=${1:-rs}
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 > gpurun_out/parity_$TAG.log 2>&1
tail -3 gpurun_out/parity_$TAG.log
for cfg in ${CFGS:-"0 1" "4 1" "8 1" "8 2"}; do
  set -- $cfg
  SPICE_RSTAGES=$1 timeout 300 python bench.py --steps 3000 --warmup 50 --no-cpu-baseline --profile-steps 50 --e2e-steps 20 --ctas-per-tile $2 $EXTRA > gpurun_out/bench_${TAG}_r$1_c$2.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_${TAG}_r$1_c$2.log').read().strip().splitlines()[-1]); print('rstages=$1 C=$2 ms/step %.4f'%d['ms_per_step'],'frac %.3f'%d['roofline']['frac'], {k:round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()})" 2>&1 | tail -1
done
