#!/bin/bash
# One GPU session: tests, bench, tile sweep.  Usage: bash tools/gpu_round.sh TAG [sweep]
TAG=${1:-x}
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests_$TAG.log 2>&1
tail -5 gpurun_out/gpu_tests_$TAG.log
timeout 300 python bench.py --steps 5000 --warmup 100 --cpu-seconds 3 --profile-steps 50 > gpurun_out/bench_$TAG.log 2>&1
tail -c 600 gpurun_out/bench_$TAG.log
if [ "$2" == "sweep" ]; then
  for tw in 4704 9376 18752 37504; do
    for gs in 1 2 4 8; do
      SPICE_GROUP_LANES=$gs timeout 200 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline --profile-steps 20 --e2e-steps 10 --tile-width $tw > gpurun_out/sweep_${TAG}_tw${tw}_gs${gs}.log 2>&1
      python -c "import json,sys; d=json.loads(open('gpurun_out/sweep_${TAG}_tw${tw}_gs${gs}.log').read().strip().splitlines()[-1]); print('tw',$tw,'gs',$gs,'ms/step %.4f'%d['ms_per_step'],'frac %.3f'%d['roofline']['frac'], d['roofline']['kernel_ms'])" 2>&1 | tail -1
    done
  done
fi
