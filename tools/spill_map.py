"""Static map of local-memory instructions (STL/LDL) in one kernel of the
built library, by source line.  Usage (dev container, no GPU):

    python tools/spill_map.py [kernel-substring] [obj]

It extracts the sm_100a cubin from the object with cuobjdump, disassembles it
with line info (nvdisasm -g) and counts STL/LDL per (file, line) inside the
named kernel's .text section.  Pair it with the dynamic counts of an ncu
capture (sass__inst_executed_local_loads/stores vs smsp__inst_executed.sum)
to see whether the local traffic sits on a hot path."""

from __future__ import annotations

import collections
import glob
import os
import re
import subprocess
import sys
import tempfile


def main() -> None:
    kern = sys.argv[1] if len(sys.argv) > 1 else "_Z7k_solveILi256ELb0E"
    obj = sys.argv[2] if len(sys.argv) > 2 else os.path.join(os.path.dirname(__file__), "..",
                                                            "paper_2508_13437_b200", "_obj", "amvm.o")
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, check=True,
                       capture_output=True)
        cubin = sorted(glob.glob(os.path.join(td, "*sm_100a*.cubin")))[0]
        sass = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True, check=True).stdout
    inside, cur = False, None
    cnt: collections.Counter = collections.Counter()
    total = 0
    for line in sass.split("\n"):
        if line.startswith(".text."):
            inside = kern in line
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        op = re.search(r"\b(STL|LDL)(\.[0-9A-Z.]+)?\s", line)
        if op:
            cnt[(cur, op.group(1))] += 1
            total += 1
        elif re.search(r"/\*[0-9a-f]{4,}\*/", line):
            cnt[("all", "sass")] += 1
    print(f"kernel {kern}: {cnt[('all', 'sass')]} SASS instructions, {total} local (STL/LDL)")
    by_line = collections.Counter()
    for (k, op), v in cnt.items():
        if k != "all":
            by_line[k] += v
    for (f, ln), v in by_line.most_common(40):
        print(f"{v:5d}  {f}:{ln}  (STL {cnt[((f, ln), 'STL')]}, LDL {cnt[((f, ln), 'LDL')]})")


if __name__ == "__main__":
    main()
