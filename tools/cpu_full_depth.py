"""CPU baseline at full depth (dev container): the oracle port on 64 fixed
random rows of the C5 layer x 100 ALNS iterations (BASELINE.md §3 plan),
all host threads; writes profiles/r02_cpu_full_depth.json (mean row time,
the whole-layer extrapolation) and tests/golden/c5_fulldepth64.npz (the
oracle's results for those rows: the GPU test compares them bitwise).

    OPENBLAS_NUM_THREADS=1 python tools/cpu_full_depth.py
"""
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402

ROWS, ITERS = 64, 100
rows = np.sort(np.random.default_rng(123).choice(bench.D_OUT, ROWS, replace=False))
X, Wall = bench.layer_rows(0, bench.D_OUT)
W = Wall[rows]
B, L, I0, R0, OB = [], [], [], [], []
for w in W:
    lv = np.linspace(float(w.min()), float(w.max()), 16)
    b = X @ w
    idx = np.argmin(np.abs(w[:, None] - lv[None, :]), axis=1)
    r = X @ lv[idx] - b
    B.append(b); L.append(lv); I0.append(idx); R0.append(r); OB.append(float(np.max(np.abs(r))))
threads = len(os.sched_getaffinity(0))
prm = O.make_params(bench.D_IN, max_iters=ITERS)
t0 = time.perf_counter()
out = O.solve(X, np.stack(B), np.stack(L), np.stack(I0), np.stack(R0), np.array(OB), np.zeros(ROWS), prm,
              [O.pcg_from_seed(int(r)) for r in rows], threads=threads)
dt = time.perf_counter() - t0
moves = int(out["moves_scored"][:, 0].sum())
row_s = dt * threads / ROWS  # one row, 100 iterations, one core
rec = {"rows": rows.tolist(), "iterations": ITERS, "threads": threads, "seconds": dt,
       "moves_reference_equivalent": moves, "moves_per_s": moves / dt,
       "mean_row_seconds_per_core": row_s,
       "extrapolated_full_layer_s_on_these_cores": row_s * bench.D_OUT / threads,
       "extrapolated_full_layer_s_on_16_cores": row_s * bench.D_OUT / 16,
       "host": bench.host_info(threads),
       "note": "extrapolated: T_cpu = mean row time x 14336 / cores (rows are independent)"}
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
json.dump(rec, open(os.path.join(ROOT, "profiles", "r02_cpu_full_depth.json"), "w"), indent=1)
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c5_fulldepth64.npz"), rows=rows,
                    best_objective=out["best_objective"], best_idx=out["best_idx"].astype(np.int8),
                    iterations=out["iterations"], trace_current_t=out["trace_current_t"],
                    trace_best_t=out["trace_best_t"], trace_pair=out["trace_pair"],
                    trace_accepted=out["trace_accepted"], moves_ref=out["moves_scored"][:, 0])
print(json.dumps({k: rec[k] for k in ("seconds", "mean_row_seconds_per_core", "extrapolated_full_layer_s_on_16_cores")}))
