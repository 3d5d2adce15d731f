"""Full-size C3 slice golden (256^2 phantom, 180 angles: m = 46080, n = 65536,
3 grey levels) for the sparse engine, made with the CPU oracle port (the
unmodified Python reference cannot run this size: its find_candidates builds
a 34 GB n x n matrix).  Dev container only (needs ~50 GB: A and its column-major copy):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_c3full.py

Inputs, all reproducible bit for bit on the GPU box: the projector is the
package's host restatement of the reference's parallel_beam_matrix (sha-
pinned against the reference at 64^2 and 128^2, tests/test_tomo_*), the
squares phantom on levels (0, 1, 2), uniform noise of seed 0 with eta = 5% of
the largest row sum (numpy order on the dense matrix), b = A @ truth + noise
(numpy's dense dgemv order), the start idx0 = nearest level of
0.7 * truth (a deliberately imperfect start; the reference would use SIRT),
ALNS seed 0, two iterations.  The fixture stores b, idx0 and the oracle's
report (trace, best objective, best codes)."""

from __future__ import annotations

import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2508_13437_b200 import tomo  # noqa: E402
from tests.golden import make_golden as mg  # noqa: E402

SIDE, ANGLES, ITERS = 256, 180, 2
LV = np.array([0.0, 1.0, 2.0])


def main() -> None:
    t0 = time.time()
    A = tomo.projection_matrix(SIDE, ANGLES)
    m, n = A.shape
    eta = 0.05 * float(A.sum(axis=1).max())
    truth = LV[np.minimum(tomo.phantom("squares", SIDE), 2)].ravel()
    b = A @ truth + np.random.default_rng(0).uniform(-eta, eta, m)
    idx0 = np.argmin(np.abs((0.7 * truth)[:, None] - LV[None, :]), axis=1)
    r0 = A @ LV[idx0] - b
    obj0 = float(np.max(np.abs(r0)))
    print(f"built in {time.time() - t0:.1f} s; m={m} n={n} nnz={int((A != 0).sum())} obj0={obj0}", flush=True)
    prm = O.make_params(n, max_iters=ITERS)
    t1 = time.time()
    out = O.solve(A, b, LV, idx0, r0, obj0, 0, prm, O.pcg_from_seed(0), colmajor=True)
    print(f"oracle {ITERS} iterations in {time.time() - t1:.1f} s: best {out['best_objective'][0]}", flush=True)
    rec = {"side": SIDE, "angles": ANGLES, "m": m, "n": n, "eta": eta, "b": b, "idx0": idx0.astype(np.int8),
           "obj0": obj0, "r0_sha": mg.sha(r0), "A_sha": mg.sha(A), "iterations": int(out["iterations"][0]),
           "best_objective": float(out["best_objective"][0]), "best_idx": out["best_idx"][0].astype(np.int8),
           "trace_current_t": out["trace_current_t"][0, :ITERS], "trace_best_t": out["trace_best_t"][0, :ITERS],
           "trace_pair": out["trace_pair"][0, :ITERS], "trace_accepted": out["trace_accepted"][0, :ITERS],
           "moves_ref": int(out["moves_scored"][0, 0]), "seconds": time.time() - t1}
    mg.save("solve_c3full", [rec])


if __name__ == "__main__":
    main()
