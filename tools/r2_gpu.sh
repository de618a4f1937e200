#!/bin/bash
# Round-2 GPU session: build, GPU tests, short benches of every workload, optional ncu.
# Usage (under gpurun): bash tools/r2_gpu.sh TAG [tests|notests] [ncu]
TAG=${1:-x}
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
python -m paper_2102_04681_b200.build > gpurun_out/build_$TAG.log 2>&1 || { tail -20 gpurun_out/build_$TAG.log; exit 1; }
if [ "$2" != "notests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 900 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests_$TAG.log 2>&1
  grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests_$TAG.log | tail -15
fi
for w in ${WORKLOADS:-synth brunel100k brunelplus50k vogels4000}; do
  timeout 400 python bench.py --workload $w --steps ${STEPS:-2000} --warmup 50 --no-cpu-baseline --profile-steps 64 --e2e-steps 256 > gpurun_out/bench_${TAG}_$w.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_${TAG}_$w.log').read().strip().splitlines()[-1]); print('$w ms/step %.4f'%d['ms_per_step'],'value %.3e'%d['value'],'frac %.3f'%d['roofline']['frac'],'e2e %.3e'%d['e2e']['value'],'launches',d['gpu_launches'],'parity',(d['parity'] or {}).get('ok'), {k:round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()})" 2>&1 | tail -1
done
if [ "$3" == "ncu" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -s 40 -c 1 -o gpurun_out/prof_${TAG}_fused python bench.py --steps 64 --warmup 5 --profile-steps 2 --e2e-steps 32 --no-cpu-baseline --no-parity > /dev/null 2>&1
  ls gpurun_out/prof_${TAG}_fused.ncu-rep
fi
