"""Run the sparse engine several times on the same slice batch: per-slice
moves and event counters must not change between runs (diagnostic)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_13437_b200 import SolverConfig, tomo  # noqa: E402

fe = tomo.build_tomo_device(24, (0.0, 1.0, 2.0), 16, 0.2, seeds=tuple(range(8)),
                            phantom_kinds=("squares", "disk", "checker"), sirt_iters=30)
sp = tomo.SparseSliceBatch(fe["csr"], fe["m"], fe["n"], fe["B"], fe["levels"], fe["idx0"])
cfg = SolverConfig(max_iters=12, destroy_rate=0.02)
runs = []
for r in range(6):
    o = sp.solve(cfg, seeds=np.arange(8), trace=True)
    sp.check_status()
    runs.append((o["moves_scored"].cpu().numpy().copy(), o["phase_cycles"][:, 8:].cpu().numpy().copy(),
                 o["best_objective"].cpu().numpy().copy()))
for r, (mv, ev, bo) in enumerate(runs):
    print(r, mv[:, 0].tolist(), "fc_calls", ev[:, 0].tolist(), "surv", ev[:, 1].tolist(), "swaps", ev[:, 2].tolist())
