#!/bin/bash
# Persistent fused kernel A/B: bench of each workload with and without SPICE_NO_PERSIST, then GPU tests.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
python -m paper_2102_04681_b200.build > gpurun_out/build_p.log 2>&1 || { tail -20 gpurun_out/build_p.log; exit 1; }
for w in ${WORKLOADS:-synth brunel100k brunelplus50k}; do
  for e in "" "SPICE_NO_PERSIST=1"; do
    env $e timeout 300 python bench.py --workload $w --steps ${STEPS:-2000} --warmup 50 --no-cpu-baseline --profile-steps 64 --e2e-steps 256 > gpurun_out/bench_p_$w.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/bench_p_$w.log').read().strip().splitlines()[-1]); print('$w [$e] us/step %.2f'%(d['ms_per_step']*1e3),'frac %.3f'%d['roofline']['frac'],'e2e %.3e'%d['e2e']['value'],'launches',d['gpu_launches'],'parity',(d.get('parity') or {}).get('ok'), {k:round(v*1e3,2) for k,v in d['roofline']['kernel_ms'].items()})" 2>&1 | tail -1
  done
done
if [ "$1" == "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests_p.log 2>&1
  grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests_p.log | tail -15
fi
