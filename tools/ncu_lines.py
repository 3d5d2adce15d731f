"""Aggregate ncu SASS-level stall samples by CUDA source line.

usage: python tools/ncu_lines.py <sass_prof.csv> <lib.so> <kernel-mangled-name> [top]
(sass_prof.csv = `ncu -i rep --page source --csv --print-source=sass`)
"""
import csv
import os
import re
import subprocess
import sys
import tempfile


def line_map(lib, kern):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    out = ""
    for cub in sorted(f for f in os.listdir(d) if f.endswith(".cubin")):  # one per translation unit
        o = subprocess.run(["nvdisasm", "-gi", os.path.join(d, cub)], capture_output=True, text=True).stdout
        if f".text.{kern}:" in o:
            out = o
            break
    m, cur, inside, block = {}, None, False, []
    for line in out.splitlines():
        if line.startswith(".text."):
            inside = line[6:].rstrip(":") == kern
            continue
        if not inside:
            continue
        mm = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if mm:
            block.append(f"{os.path.basename(mm.group(1))}:{mm.group(2)}")
            continue
        mo = re.search(r"/\*([0-9a-f]{4,})\*/", line)
        if mo:
            if block:
                cur = block[0] + (" <- " + block[1] if len(block) > 1 else "")
                block = []
            m[int(mo.group(1), 16)] = cur
    return m


def main():
    prof, lib, kern = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    m = line_map(lib, kern)
    rows = list(csv.reader(open(prof)))
    hdr, data = rows[1], rows[2:]
    ia, iss = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    base = int(data[0][ia], 16)
    agg, tot = {}, 0
    for r in data:
        s = int(r[iss] or 0)
        tot += s
        k = m.get(int(r[ia], 16) - base, "?")
        agg[k] = agg.get(k, 0) + s
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100 * v / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main()
