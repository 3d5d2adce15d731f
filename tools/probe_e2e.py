"""Where the end-to-end (public API, host buffers) time of the C5 bench step
goes: ptq.solve_layer's stages, each closed by a device sync."""
import sys
import time

import numpy as np

sys.path.insert(0, '/root/repo')
import torch  # noqa: E402

from paper_2508_13437_b200 import SolverConfig, ptq  # noqa: E402
from paper_2508_13437_b200 import _native as N  # noqa: E402

rows = 1792
X = np.random.default_rng(0).standard_normal((2048, 4096))
W = (np.random.default_rng(1).standard_normal((14336, 4096)) * 0.02)[:rows].copy()
Xh = torch.from_numpy(X).pin_memory()
Wh = torch.from_numpy(W).pin_memory()
cfg = SolverConfig(max_iters=2)
seeds = np.arange(rows)
for rep in range(3):
    T = {}
    torch.cuda.synchronize()
    t = time.perf_counter()

    def mark(k):
        global t
        torch.cuda.synchronize()
        now = time.perf_counter()
        T[k] = round((now - t) * 1e3, 2)
        t = now

    lb = ptq.LayerBatch(Xh, Wh, bits=4)
    mark("LayerBatch (H2D, transpose, isfinite)")
    lb.prepare()
    mark("prepare (levels, B, start residual)")
    o = lb.solve(cfg, seeds=seeds)
    mark("solve (seeds + k_transpose + k_solve)")
    lb.check_status()
    mark("status")
    host = {k: v.cpu().numpy() for k, v in o.items()}
    mark("D2H all outputs")
    t_all = sum(T.values())
    print(rep, round(t_all, 1), T, flush=True)
