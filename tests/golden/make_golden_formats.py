"""Golden fixtures for the text formats (dmmv.io, /root/reference/pkg/src/dmmv/io.py,
and the run artifacts of dmmv.cli.cmd_solve, cli.py:99-140), made by running
the UNMODIFIED reference in the dev container:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_formats.py

Writes tests/golden/formats.json: for each case the instance text, the LP
text, the reference's solution line, and trace.csv / report.txt of a short
solve (report minus the wall-time line).
"""

from __future__ import annotations

import io
import json
import os
import sys
import tempfile

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")
import dmmv  # noqa: E402
from dmmv import cli as ref_cli  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    rng = np.random.default_rng(8147)
    out = []
    for m, n, nlev, with_init in [(5, 3, 4, True), (12, 9, 5, False), (20, 10, 6, True),
                                  (3, 30, 3, False), (24, 6, 16, False)]:
        A = rng.uniform(-1, 1, (m, n))
        A[rng.uniform(size=A.shape) < 0.15] = 0.0           # zero coefficients skip in LP
        lv = np.sort(rng.choice(np.linspace(-2, 2, 41), nlev, replace=False))
        b = A @ rng.uniform(lv[0], lv[-1], n) + rng.normal(0, 0.1, m)
        init = rng.uniform(lv[0], lv[-1], n) if with_init else None
        out.append(dmmv.Instance(A, b, dmmv.ValueSet(lv), continuous_init=init))
    # awkward floats (repr round trip)
    out.append(dmmv.Instance(np.array([[0.1, 1e300], [-1 / 3, 5e-324]]), np.array([-0.0, 2.5]),
                             dmmv.ValueSet([-1e-17, 0.3, 7.0])))
    return out


def main():
    recs = []
    insts = cases()
    for k, inst in enumerate(insts):
        text = dmmv.instance_to_text(inst)
        lp = io.StringIO()
        dmmv.export_lp(inst, lp)
        rec = {"instance": text, "lp": lp.getvalue()}
        recs.append(rec)
        if k == len(insts) - 1:
            continue  # the awkward-float case: formats only (its solve overflows)
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "inst.txt")
            with open(path, "w") as fh:
                fh.write(text)
            outdir = os.path.join(td, "run")
            iters = 6
            rc = ref_cli.main(["solve", "--instance", path, "--iters", str(iters), "--seed", str(k),
                               "--out", outdir])
            assert rc == 0
            report = open(os.path.join(outdir, "report.txt")).read()
            trace = open(os.path.join(outdir, "trace.csv")).read()
            sol = open(os.path.join(outdir, "solution.txt")).read()
        rec.update({"iters": iters, "seed": k,
                     "report": [ln for ln in report.splitlines()
                                if not ln.startswith(("wall_time_s", "instance:"))],
                     "trace": trace, "solution": sol})
    with open(os.path.join(HERE, "formats.json"), "w") as fh:
        json.dump({"reference": "dmmv " + dmmv.__version__, "cases": recs}, fh, indent=0)
    print(f"wrote {len(recs)} cases")


if __name__ == "__main__":
    main()
