#!/bin/bash
# Tests + short bench of every workload + optional full ncu capture.  Usage: bash tools/gpu_quick.sh TAG [ncu]
TAG=${1:-x}
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/gpu_tests_$TAG.log 2>&1
tail -15 gpurun_out/gpu_tests_$TAG.log | grep -E "passed|failed|Error|error|assert" | head -12
for w in synth brunel100k vogels4000; do
  timeout 300 python bench.py --workload $w --steps 4000 --warmup 100 --no-cpu-baseline --profile-steps 50 --e2e-steps 200 > gpurun_out/bench_${TAG}_$w.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_${TAG}_$w.log').read().strip().splitlines()[-1]); print('$w ms/step %.4f'%d['ms_per_step'],'value %.3e'%d['value'],'frac %.3f'%d['roofline']['frac'], {k:round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()})" 2>&1 | tail -1
done
if [ "$2" == "ncu" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -s 40 -c 1 -o gpurun_out/prof_${TAG}_fused python bench.py --steps 64 --warmup 5 --profile-steps 2 --e2e-steps 2 --no-cpu-baseline > /dev/null 2>&1
  ls gpurun_out/prof_${TAG}_fused.ncu-rep
fi
