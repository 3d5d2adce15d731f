"""Full C5 layer (14336 rows x 100 ALNS iterations) on one GPU, timed end to
end through ptq.solve_layer, plus a sampled CPU-oracle extrapolation."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_13437_b200 import SolverConfig, ptq  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 14336
X = np.random.default_rng(0).standard_normal((2048, 4096))
W = np.random.default_rng(1).standard_normal((14336, 4096))[:rows] * 0.02
Xh, Wh = torch.from_numpy(X).pin_memory(), torch.from_numpy(W).pin_memory()
torch.cuda.synchronize()
t0 = time.perf_counter()
rep = ptq.solve_layer(Xh, Wh, bits=4, cfg=SolverConfig(max_iters=iters))
dt = time.perf_counter() - t0
moves = int(rep.moves_scored[:, 0].sum())
print(json.dumps({"rows": rows, "iters": iters, "seconds": round(dt, 2), "moves_ref": moves,
                  "moves_per_s": moves / dt, "mean_initial_linf": float(rep.initial_objective.mean()),
                  "mean_final_linf": float(rep.objective.mean()),
                  "mean_improvement_pct": float(100 * (1 - rep.objective / rep.initial_objective).mean()),
                  "iterations_min_max": [int(rep.iterations.min()), int(rep.iterations.max())]}), flush=True)
