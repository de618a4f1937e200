#!/bin/bash
# ncu --set full of the weak-scaling proxy's fused kernel and bitmap->list (one launch each).
TAG=${1:-x}; A=${2:-8}
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
python -m paper_2102_04681_b200.build > /dev/null 2>&1
for k in k_fused k_b2l; do
PROXY_R=1 timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:"$k" -s 20 -c 1 \
  -o gpurun_out/prof_${TAG}_${k}_g$A python tools/g_proxy.py $A > /dev/null 2>&1
ncu -i gpurun_out/prof_${TAG}_${k}_g$A.ncu-rep --page source --print-source cuda,sass --csv > gpurun_out/src_${TAG}_${k}_g$A.csv 2>/dev/null
done
ls -la gpurun_out/*${TAG}*
