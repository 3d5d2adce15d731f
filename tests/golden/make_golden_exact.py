"""Golden fixtures for the exact oracle (dmmv.oracle.brute_force,
/root/reference/pkg/src/dmmv/oracle.py:38-111), by running the UNMODIFIED
reference in the dev container:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_exact.py

Each record stores A, b, levels and the reference's (best_idx, best_t,
enumerated) for prune=False and prune=True.
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")
import dmmv  # noqa: E402
from dmmv import oracle as ref_oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    rng = np.random.default_rng(2508)
    out = []
    # random float instances, varied shapes (total <= ~5e5 so the pruned DFS stays quick)
    for m, n, nlev in [(12, 4, 5), (40, 6, 4), (7, 8, 3), (64, 5, 8), (20, 10, 3), (33, 3, 16), (5, 12, 2),
                       (100, 4, 6), (1, 6, 5), (16, 1, 9)]:
        A = rng.uniform(-1, 1, (m, n))
        lv = np.sort(rng.choice(np.linspace(-3, 3, 61), nlev, replace=False))
        b = A @ rng.uniform(lv[0], lv[-1], n) + rng.normal(0, 0.05, m)
        out.append((A, b, lv))
    # integer instances: exact arithmetic, many objective ties (lexicographic tie-break)
    for m, n, nlev in [(6, 5, 4), (10, 7, 3), (3, 9, 2), (8, 6, 5)]:
        A = rng.integers(-2, 3, (m, n)).astype(float)
        lv = np.arange(nlev, dtype=float) - nlev // 2
        b = rng.integers(-4, 5, m).astype(float)
        out.append((A, b, lv))
    # planted zero objective
    A = rng.integers(-3, 4, (9, 6)).astype(float)
    lv = np.array([-1.0, 0.0, 2.0])
    out.append((A, A @ lv[rng.integers(0, 3, 6)], lv))
    # single level (numpy: one code -> dgemv over the rows)
    out.append((rng.uniform(-1, 1, (4, 3)), rng.uniform(-1, 1, 4), np.array([0.5])))
    out.append((rng.uniform(-1, 1, (7, 21)), rng.uniform(-1, 1, 7), np.array([-0.25])))
    # m = 1 (numpy: dgemv over the codes of each 2^15 chunk; one code too -> ddot)
    out.append((rng.uniform(-1, 1, (1, 7)), rng.uniform(-1, 1, 1), np.linspace(-1, 1, 5)))
    out.append((rng.uniform(-1, 1, (1, 37)), rng.uniform(-1, 1, 1), np.array([0.75])))
    return out


def swap_cases():
    """(A, b, levels, idx) for exhaustive_swap_check: random starts, a start
    after the reference's own local search (few improving pairs, boundary
    ties), integer data (exact ties) and m = 1 (numpy's ddot path)."""
    from dmmv import localsearch as ls

    rng = np.random.default_rng(137)
    out = []
    for m, n, nlev in [(30, 12, 5), (64, 20, 8), (9, 16, 4), (1, 10, 6), (120, 7, 16)]:
        A = rng.uniform(-1, 1, (m, n))
        lv = np.linspace(-2, 2, nlev)
        b = A @ rng.uniform(-2, 2, n)
        out.append((A, b, lv, rng.integers(0, nlev, n)))
    A = rng.uniform(-1, 1, (40, 24))
    lv = np.linspace(-3, 3, 7)
    b = A @ rng.uniform(-3, 3, 24)
    inst = dmmv.Instance(A, b, dmmv.ValueSet(lv))
    sol = dmmv.Solution.from_indices(inst, rng.integers(0, 7, 24))
    ls.local_search(inst, sol, dmmv.FilterConfig())
    out.append((A, b, lv, sol.idx.copy()))
    A = rng.integers(-2, 3, (10, 9)).astype(float)
    lv = np.arange(5, dtype=float) - 2
    out.append((A, rng.integers(-3, 4, 10).astype(float), lv, rng.integers(0, 5, 9)))
    return out


def swap_main() -> None:
    from dmmv import localsearch as ls

    rec = {}
    cs = swap_cases()
    for k, (A, b, lv, idx) in enumerate(cs):
        inst = dmmv.Instance(A, b, dmmv.ValueSet(lv))
        sol = dmmv.Solution.from_indices(inst, idx)
        n = inst.n
        T = np.full((n, n), np.nan)
        V = np.zeros((n, n), np.int32)
        x = sol.values(inst)
        for i in range(n):
            for j in range(n):
                if i == j or x[i] <= x[j]:
                    continue
                sw = sol.idx.copy()
                sw[i], sw[j] = sw[j], sw[i]
                T[i, j] = dmmv.compute_residual(inst, sw)[1]
                V[i, j] = ls.is_improving(inst, sol, ls.SwapCandidate(i, j, float(x[i] - x[j])))
        rep = ref_oracle.exhaustive_swap_check(inst, sol)
        rec.update({f"{k}/A": A, f"{k}/b": b, f"{k}/levels": lv, f"{k}/idx": sol.idx.astype(np.int32),
                    f"{k}/residual": sol.residual, f"{k}/objective": sol.objective, f"{k}/T": T, f"{k}/V": V,
                    f"{k}/pairs_checked": rep.pairs_checked, f"{k}/n_discrepancies": len(rep.discrepancies),
                    f"{k}/n_boundary": len(rep.boundary)})
    np.savez_compressed(os.path.join(HERE, "swap_check.npz"), count=len(cs), **rec)
    print(f"{len(cs)} swap_check records")


def main() -> None:
    rec = {}
    cs = cases()
    for k, (A, b, lv) in enumerate(cs):
        inst = dmmv.Instance(A, b, dmmv.ValueSet(lv))
        r0 = ref_oracle.brute_force(inst)
        r1 = ref_oracle.brute_force(inst, prune=True)
        rec.update({f"{k}/A": A, f"{k}/b": b, f"{k}/levels": lv,
                    f"{k}/best_idx": r0.best_idx.astype(np.int32), f"{k}/best_t": r0.best_t,
                    f"{k}/enumerated": r0.enumerated,
                    f"{k}/pruned_best_idx": r1.best_idx.astype(np.int32), f"{k}/pruned_best_t": r1.best_t,
                    f"{k}/pruned_enumerated": r1.enumerated})
    np.savez_compressed(os.path.join(HERE, "brute_force.npz"), count=len(cs), **rec)
    print(f"{len(cs)} brute_force records")


if __name__ == "__main__":
    main()
    swap_main()
