#!/bin/bash
# ncu launch list (per-kernel durations) of the weak-scaling proxy: bash tools/gl_kernels.sh 2 8 ...
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
for a in "$@"; do
PROXY_R=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gl_$a.csv python tools/g_proxy.py $a > /dev/null 2>&1
python - "$a" <<'PY'
import csv, collections, sys
a = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/gl_{a}.csv")))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
H = rows[h]; ik = H.index("Kernel Name"); iv = H.index("Metric Value")
ks = [(r[ik].split("(")[0], float(r[iv])) for r in rows[h + 1:] if len(r) > iv][-96:]
agg = collections.defaultdict(list)
for k, v in ks:
    agg[k].append(v)
print(a, {k: (len(v), round(sum(v) / len(v) / 1e3, 2)) for k, v in agg.items()})
PY
done
