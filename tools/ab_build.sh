#!/bin/bash
# Same-box A/B of compile-time variants: bash tools/ab_build.sh "DEF=1" ["DEF2=1" ...]
# builds /tmp/libspice_<i>.so per define set and benches each against the in-tree library.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
i=0
for defs in "$@"; do
  python -c "
import sys; sys.path.insert(0, '.')
import importlib.util
spec = importlib.util.spec_from_file_location('b', 'paper_2102_04681_b200/build.py'); b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)
b.build(out='/tmp/libspice_$i.so', defines='$defs'.split())" > /dev/null 2>&1
  i=$((i+1))
done
for rep in 1 2; do
  timeout 300 python bench.py --steps 3000 --warmup 50 --no-cpu-baseline --profile-steps 50 --e2e-steps 20 $EXTRA > gpurun_out/ab_base.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_base.log').read().strip().splitlines()[-1]); print('base', d['ms_per_step'], d['roofline']['kernel_ms']['fused_in_graph'])"
  i=0
  for defs in "$@"; do
    SPICE_LIB=/tmp/libspice_$i.so timeout 300 python bench.py --steps 3000 --warmup 50 --no-cpu-baseline --profile-steps 50 --e2e-steps 20 $EXTRA > gpurun_out/ab_$i.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/ab_$i.log').read().strip().splitlines()[-1]); print('$defs', d['ms_per_step'], d['roofline']['kernel_ms']['fused_in_graph'])"
    i=$((i+1))
  done
done
