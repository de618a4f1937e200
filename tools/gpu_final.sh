#!/bin/bash
# Round evidence: default bench (synth), other BASELINE workloads, A/B global atomics,
# launch list + one full ncu capture of the dominant kernel.  Usage: bash tools/gpu_final.sh TAG
TAG=${1:-r01}
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/bench_${TAG}_synth.json 2> gpurun_out/bench_${TAG}_synth.err
tail -c 400 gpurun_out/bench_${TAG}_synth.json
for w in brunel100k brunelplus50k vogels4000; do
  timeout 400 python bench.py --workload $w --steps 10000 --cpu-seconds 8 > gpurun_out/bench_${TAG}_$w.json 2> gpurun_out/bench_${TAG}_$w.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_${TAG}_$w.json').read().strip().splitlines()[-1]); print('$w', 'value %.3e'%d['value'], 'ms/step %.4f'%d['ms_per_step'], 'cpu %.3e'%d['cpu_baseline']['value'], 'frac %.3f'%d['roofline']['frac'])" 2>&1 | tail -1
done
timeout 300 python bench.py --global-atomics --steps 2000 --warmup 50 --no-cpu-baseline > gpurun_out/bench_${TAG}_globalatomics.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_${TAG}_globalatomics.json').read().strip().splitlines()[-1]); print('global-atomics A/B: ms/step %.4f'%d['ms_per_step'], d['roofline']['kernel_ms'])" 2>&1 | tail -1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 120 --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 400 --warmup 20 --profile-steps 5 --e2e-steps 5 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"k_fused" -s 40 -c 1 -o gpurun_out/prof_${TAG}_fused python bench.py --steps 64 --warmup 5 --profile-steps 2 --e2e-steps 2 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | tail -5
