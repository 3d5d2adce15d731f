"""Golden fixtures for the candidate-move scorer, made with the UNMODIFIED
reference's own move (dmmv.core.apply_shift, core.py:208-225, whose
objective update is the one_opt candidate objective of localsearch.py:76-78):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_scoring.py

For each case: A, b, levels, a start assignment, and t_all[j, l] = the
objective the reference reports after ``apply_shift(inst, copy, j, l)`` for
every level-changing move (the current objective where l == idx_j).
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")
import dmmv  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(4242)
    out = {}
    cases = [(40, 12, 5, False), (1, 6, 4, False), (70, 20, 16, False), (33, 9, 3, True), (200, 16, 8, True),
             (17, 5, 40, False)]
    for k, (m, n, nlev, integer) in enumerate(cases):
        if integer:
            A = rng.integers(-3, 4, (m, n)).astype(float)
            lv = np.arange(nlev, dtype=float) - nlev // 2
        else:
            A = rng.normal(0, 1, (m, n))
            lv = np.sort(rng.choice(np.linspace(-4, 4, 4 * nlev + 1), nlev, replace=False))
        b = A @ lv[rng.integers(0, nlev, n)] + rng.normal(0, 0.3, m)
        inst = dmmv.Instance(A, b, dmmv.ValueSet(lv))
        idx = rng.integers(0, nlev, n)
        idx[:2] = [0, nlev - 1]
        sol = dmmv.Solution.from_indices(inst, idx)
        t = np.empty((n, nlev))
        for j in range(n):
            for lvl in range(nlev):
                t[j, lvl] = dmmv.apply_shift(inst, sol.copy(), j, lvl).objective
        for key, v in {"A": A, "b": b, "levels": lv, "idx": idx, "residual": sol.residual,
                       "objective": np.float64(sol.objective), "t_all": t}.items():
            out[f"{k}/{key}"] = v
    out["count"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(HERE, "scoring.npz"), **out)
    print(f"wrote {len(cases)} cases")


if __name__ == "__main__":
    main()
