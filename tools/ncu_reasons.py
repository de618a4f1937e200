#!/usr/bin/env python
"""Stall-reason breakdown per CUDA line from `ncu --page source --print-source cuda,sass --csv`.
Usage: python tools/ncu_reasons.py src.csv [min_share]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
ist = h.index("Warp Stall Sampling (All Samples)")
rc = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = 0
lines = []
for r in rows[hi + 1:]:
    if len(r) > ist and r[2] == "-":
        v = int(r[ist] or 0)
        tot += v
        lines.append((r[0], r[1][:80], v, {h[i][6:]: int(r[i] or 0) for i in rc if (r[i] or "0") != "0"}))
for ln, s, v, d in sorted(lines, key=lambda x: -x[2]):
    if v < thr * tot:
        break
    top = sorted(d.items(), key=lambda kv: -kv[1])[:4]
    print(f"L{ln:>5} {100 * v / tot:5.1f}%  " + " ".join(f"{k}:{100 * c / max(v, 1):.0f}%" for k, c in top) + f" | {s}")
