#!/bin/bash
# Round-2 evidence session: full GPU tests, smoke, every workload's bench line, the ncu launch
# list of the default bench and one full ncu capture per workload's step kernel.
# Usage (under gpurun): bash tools/r2_evidence.sh TAG
TAG=${1:-x}
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
python -m paper_2102_04681_b200.build > gpurun_out/build_$TAG.log 2>&1 || { tail -20 gpurun_out/build_$TAG.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests_$TAG.log 2>&1
tail -3 gpurun_out/gpu_tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -3 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}_default.json 2> gpurun_out/bench_${TAG}_default.err; tail -c 300 gpurun_out/bench_${TAG}_default.json
for w in brunel100k brunelplus50k vogels4000 synth250m; do
  timeout 400 python bench.py --workload $w --steps 5000 --warmup 100 > gpurun_out/bench_${TAG}_$w.json 2> gpurun_out/bench_${TAG}_$w.err
done
timeout 400 python bench.py --setup > gpurun_out/setup_$TAG.json 2> gpurun_out/setup_$TAG.err
SPICE_NO_COOP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 64 --warmup 5 --profile-steps 4 --e2e-steps 64 --no-cpu-baseline --no-parity > /dev/null 2>&1
# synth: the persistent kernel (ncu cannot replay cooperative cluster launches: SPICE_NO_COOP=1);
# launch 2 is the timed region's spice_step(32): 31 steps in one launch
SPICE_NO_COOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_synth_run" -s 1 -c 1 -o gpurun_out/prof_${TAG}_synth python bench.py --workload synth --steps 32 --warmup 5 --profile-steps 2 --e2e-steps 32 --no-cpu-baseline --no-parity > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -s 40 -c 1 -o gpurun_out/prof_${TAG}_brunel100k python bench.py --workload brunel100k --steps 64 --warmup 5 --profile-steps 2 --e2e-steps 32 --no-cpu-baseline --no-parity > /dev/null 2>&1
# Brunel+: the persistent kernel (launch 2: the timed spice_step(32), 31 steps)
SPICE_NO_COOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_plastic_run" -s 1 -c 1 -o gpurun_out/prof_${TAG}_brunelplus50k python bench.py --workload brunelplus50k --steps 32 --warmup 5 --profile-steps 2 --e2e-steps 32 --no-cpu-baseline --no-parity > /dev/null 2>&1
WORKLOADS="synth brunel100k brunelplus50k" bash tools/r2_diag.sh > gpurun_out/diag_$TAG.txt 2>&1
for g in 2 4 8; do timeout 300 python tools/g_proxy.py $g 2>&1 | tail -1; done > gpurun_out/gproxy_$TAG.txt
timeout 1100 python tools/checked_run.py > gpurun_out/checked_$TAG.txt 2>&1
ls gpurun_out | grep $TAG
