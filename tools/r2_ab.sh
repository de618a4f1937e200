#!/bin/bash
# A/B of the default build against env switches on the synth bench (same box, alternating).
# Usage: bash tools/r2_ab.sh "ENV=1" [steps]
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
python -m paper_2102_04681_b200.build > /dev/null 2>&1
S=${2:-3000}
for rep in 1 2; do
  for v in "" "$1"; do
    env $v python bench.py --steps $S --warmup 100 --no-cpu-baseline --profile-steps 32 --e2e-steps 64 --no-parity ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[${v:-default}]', 'ms/step %.5f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'fused_in_graph %.5f'%d['roofline']['kernel_ms']['fused_in_graph'])"
  done
done
