#!/bin/bash
# Diagnostics session: shared-atomic micro, per-CTA phase clocks of synth and Brunel+.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 120 ./tools/micro/atoms_micro.bin > gpurun_out/atoms_micro.txt 2>&1; cat gpurun_out/atoms_micro.txt
for w in ${WORKLOADS:-synth brunelplus50k}; do
  PHASES_DUMP=gpurun_out/phases_$w.npz timeout 600 python tools/phases.py $w 2048 > gpurun_out/phases_$w.txt 2>&1; cat gpurun_out/phases_$w.txt
done
