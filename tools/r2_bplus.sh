#!/bin/bash
# Brunel+ diagnostics: event statistics, phase timeline, PL_U variants.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
python -m paper_2102_04681_b200.build > /dev/null 2>&1
timeout 300 python tools/bp_stats.py 2>&1 | tail -2
timeout 300 python tools/phases.py brunelplus50k 2048 2>&1 | tail -16
for d in ${VARIANTS}; do
  echo "== $d"; SPICE_DEFINES=$d timeout 300 python tools/phases.py brunelplus50k 2048 2>&1 | tail -16
done
