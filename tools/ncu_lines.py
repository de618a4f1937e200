#!/usr/bin/env python
"""Per-CUDA-line instruction and stall shares from `ncu --page source --print-source cuda,sass --csv`."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
    h = rows[hi]
    iex = h.index("Instructions Executed")
    ist = h.index("Warp Stall Sampling (All Samples)")

    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0
    agg = collections.defaultdict(lambda: [0, 0])
    for r in rows[hi + 1:]:
        if len(r) > iex and r[2] == "-":
            k = (r[0], r[1][:100])
            agg[k][0] += num(r[iex])
            agg[k][1] += num(r[ist])
    tot = sum(v[0] for v in agg.values())
    tots = sum(v[1] for v in agg.values())
    print(f"total warp-instructions {tot}, stall samples {tots}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{v[0]:9d} {100 * v[0] / tot:5.1f}%  stall {100 * v[1] / max(tots, 1):5.1f}% | L{k[0]:>4} {k[1]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
