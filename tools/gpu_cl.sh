#!/bin/bash
# Cluster-tile A/B: parity tests, then synth bench at C = 1, 2, 4.  Usage: bash tools/gpu_cl.sh TAG
TAG=${1:-cl}
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 > gpurun_out/parity_$TAG.log 2>&1
tail -4 gpurun_out/parity_$TAG.log
for c in ${CS:-1 2 4}; do
  timeout 300 python bench.py --steps 3000 --warmup 50 --no-cpu-baseline --profile-steps 50 --e2e-steps 20 --ctas-per-tile $c $EXTRA > gpurun_out/bench_${TAG}_c$c.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_${TAG}_c$c.log').read().strip().splitlines()[-1]); print('C=$c ms/step %.4f'%d['ms_per_step'],'frac %.3f'%d['roofline']['frac'], d['config']['delivery'], {k:round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()})" 2>&1 | tail -1
done
