"""Full-depth PTQ-layer goldens: C5 rows {0, 1, 14335} and C4 rows {0, 3071}
at 100 ALNS iterations (the SURVEY.md §8d per-row depth), made by running the
UNMODIFIED reference in the dev container:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_layers.py

Each row is an independent ``dmmv.solve`` of the reference's ``build_quant``
instance for that row (builders.py:355-372 semantics with the shared X of
recipes.ptq_layer; seed = row index), run in its own process (≈7 min per C5
row on one core).  The fixture stores the reference's report for every row;
X and W are regenerated from their seeds by ``recipes.ptq_layer`` (sha-checked)
so the GPU test can push the WHOLE layer shape through ``ptq.solve_layer``'s
chunked path and compare these rows bit for bit.
"""

from __future__ import annotations

import os
import subprocess
import sys
import tempfile

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))

LAYERS = {
    # name: (d, total rows, rows to pin)
    "c5": (4096, 14336, (0, 1, 14335)),
    "c4": (768, 3072, (0, 3071)),
}
ITERS = 100


def one(name: str, row: int, out: str) -> None:
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.path.insert(0, ROOT)
    import dmmv
    from tests.golden import make_golden as mg
    from tests.golden import recipes

    d, total, _ = LAYERS[name]
    X, W = recipes.ptq_layer(d, total)
    data = recipes.ptq_row(X, W[row])
    inst, cfg = mg.mk(data, dict(max_iters=ITERS, seed=row))
    rec = mg.solve_record(inst, cfg, store_A=False)
    rec.pop("continuous_init", None)
    rec["row"] = row
    rec["X_sha"] = mg.sha(X)
    rec["W_sha"] = mg.sha(W)
    np.savez(out, **{k: np.asarray(v) for k, v in rec.items()})


def main() -> None:
    assert os.environ.get("OPENBLAS_NUM_THREADS") == "1"
    if len(sys.argv) == 5 and sys.argv[1] == "--one":
        one(sys.argv[2], int(sys.argv[3]), sys.argv[4])
        return
    tmp = tempfile.mkdtemp(prefix="golden_layers_")
    jobs = []
    for name, (_, _, rows) in LAYERS.items():
        for r in rows:
            out = os.path.join(tmp, f"{name}_{r}.npz")
            jobs.append((name, r, out, subprocess.Popen(
                [sys.executable, __file__, "--one", name, str(r), out])))
    for name, r, out, p in jobs:
        if p.wait() != 0:
            raise SystemExit(f"{name} row {r} failed")
    sys.path.insert(0, ROOT)
    from tests.golden import make_golden as mg

    for name, (_, _, rows) in LAYERS.items():
        recs = []
        for r in rows:
            with np.load(os.path.join(tmp, f"{name}_{r}.npz")) as z:
                recs.append({k: z[k] for k in z.files})
        mg.save(f"layer_{name}", recs)


if __name__ == "__main__":
    main()
