"""Print the SASS (with source lines) around the instructions of a given source line.

usage: python tools/sass_at.py <lib.so> <kernel> <pattern-in-source-line> [before] [after]
"""
import os
import re
import subprocess
import sys
import tempfile

lib, kern, pat = sys.argv[1:4]
before = int(sys.argv[4]) if len(sys.argv) > 4 else 15
after = int(sys.argv[5]) if len(sys.argv) > 5 else 60
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-gi", os.path.join(d, cub)], capture_output=True, text=True).stdout
inside, cur, block, out = False, None, [], []
for ln in txt.splitlines():
    if ln.startswith(".text."):
        inside = ln[6:].rstrip(":") == kern
        continue
    if not inside:
        continue
    mm = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if mm:
        block.append((os.path.basename(mm.group(1)), int(mm.group(2))))
        continue
    mo = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if mo:
        if block:
            cur, block = block[0], []
        out.append((int(mo.group(1), 16), cur, mo.group(2).strip()))
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2508_13437_b200", "csrc",
                        "amvm_engine.cuh")).read().splitlines()
tgt = [i + 1 for i, l in enumerate(src) if pat in l][0]
idx = [k for k, o in enumerate(out) if o[1] and o[1][0] == "amvm_engine.cuh" and o[1][1] == tgt]
print("line", tgt, "instructions", len(idx))
k0 = idx[0]
for o in out[max(0, k0 - before):k0 + after]:
    print(hex(o[0]), o[1][1] if o[1] else None, o[2][:100])
