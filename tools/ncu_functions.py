"""Attribute ncu stall samples to engine functions (innermost amvm_engine.cuh frame).

usage: python tools/ncu_functions.py <sass_prof.csv> <lib.so> <kernel>
"""
import csv
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_lines import line_map  # noqa: E402

prof, lib, kern = sys.argv[1:4]
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2508_13437_b200", "csrc",
                        "amvm_engine.cuh")).read().splitlines()
starts = []
for i, l in enumerate(src):
    m = re.match(r"\s+__device__ [\w:<>\*&\s]+? (\w+)\(", l)
    if m:
        starts.append((i + 1, m.group(1)))


def fn_of(line):
    name = "?"
    for st, nm in starts:
        if st <= line:
            name = nm
        else:
            break
    return name


m = line_map(lib, kern)
rows = list(csv.reader(open(prof)))
hdr, data = rows[1], rows[2:]
ia, iss = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][ia], 16)
agg, tot = {}, 0
for r in data:
    k = m.get(int(r[ia], 16) - base) or "?"
    parts = [p for p in k.split(" <- ") if p.startswith("amvm_engine")]
    s = int(r[iss] or 0)
    tot += s
    f = fn_of(int(parts[0].split(":")[1])) if parts else "other"
    agg[f] = agg.get(f, 0) + s
for f, s in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{100 * s / tot:5.1f}%  {f}")
