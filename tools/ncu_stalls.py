"""Stall-reason breakdown of the SASS instructions mapped to given source
lines (or to all lines of one engine function).
usage: python tools/ncu_stalls.py <sass.csv> <lib.so> <kernel> <file:line>[,<file:line>...]|fn=<name>"""
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_lines import line_map  # noqa: E402

prof, lib, kern, sel = sys.argv[1:5]
m = line_map(lib, kern)
rows = list(csv.reader(open(prof)))
hdr, data = rows[1], rows[2:]
ia = hdr.index("Address")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ia], 16)
want = set(sel.split(","))
agg = {hdr[i]: 0 for i in cols}
tot = 0
for r in data:
    k = m.get(int(r[ia], 16) - base, "?")
    if not any(k.startswith(w) or (" <- " + w) in k for w in want):
        continue
    for i in cols:
        v = int(float(r[i] or 0))
        agg[hdr[i]] += v
        tot += v
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]:
    print(f"{100 * v / max(tot, 1):5.1f}%  {k}")
print("samples", tot)
