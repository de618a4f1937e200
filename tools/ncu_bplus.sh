#!/bin/bash
# ncu --set full of one Brunel+ fused launch (dense warp sampling), source page exported.
TAG=${1:-x}; W=${2:-brunelplus50k}
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
python -m paper_2102_04681_b200.build > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:"k_fused" -s 200 -c 1 \
  -o gpurun_out/prof_${TAG}_$W python bench.py --workload $W --steps 256 --warmup 5 --profile-steps 2 --e2e-steps 32 --no-cpu-baseline --no-parity > gpurun_out/ncu_${TAG}.log 2>&1
ncu -i gpurun_out/prof_${TAG}_$W.ncu-rep --page source --print-source cuda,sass --csv > gpurun_out/src_${TAG}_$W.csv 2>/dev/null
ls -la gpurun_out/prof_${TAG}_$W.ncu-rep gpurun_out/src_${TAG}_$W.csv
