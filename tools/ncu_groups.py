#!/usr/bin/env python
"""Instruction / stall-sample shares of k_fused phases by source-line range of sim.cu.
Usage: ncu_groups.py SRC.csv  (from `ncu -i R --page source --print-source cuda,sass --csv`)"""
import collections, csv, re, sys

def ranges(path="paper_2102_04681_b200/csrc/sim.cu"):
    src = open(path).read().splitlines()
    marks = []
    for i, l in enumerate(src, 1):
        m = re.match(r"^(?:template <[^>]*>\s*)?__(?:device|global)__ .*?\b(\w+)\(", l)
        if m:
            marks.append((i, m.group(1)))
    return marks

def main(p):
    rows = list(csv.reader(open(p)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
    h = rows[hi]; iex = h.index("Instructions Executed"); ist = h.index("Warp Stall Sampling (All Samples)")
    marks = ranges()
    g = collections.defaultdict(lambda: [0, 0]); ti = ts = 0
    for r in rows[hi + 1:]:
        if len(r) > iex and r[2] == "-":
            try:
                ln = int(r[0]); n = int(r[iex] or 0); s = int(r[ist] or 0)
            except ValueError:
                continue
            name = "?"
            for (l0, nm) in marks:
                if l0 <= ln: name = nm
            if ln < 60 and ('shfl' in r[1] or 'x += y' in r[1] or 'sum +=' in r[1]): name = "scan helpers"
            g[name][0] += n; g[name][1] += s; ti += n; ts += s
    for k, v in sorted(g.items(), key=lambda kv: -kv[1][1]):
        print(f"{100*v[0]/ti:5.1f}% inst  {100*v[1]/ts:5.1f}% stall  {k}")

main(sys.argv[1])
