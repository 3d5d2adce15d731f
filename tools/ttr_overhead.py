"""Host overhead of solve_from on C1 (wall at 1, 10, 774 iterations; median of 5)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_13437_b200 as P  # noqa: E402
from paper_2508_13437_b200.controller import solve_from  # noqa: E402
from tests.golden_io import cfg_kwargs, load, named_A  # noqa: E402

rec = load("solve_c1")[0]
A = named_A("c1", rec)
inst = P.Instance(A, rec["b"], P.ValueSet(rec["levels"]))
start = P.Solution(rec["idx0"], rec["r0"], rec["obj0"], 0)
kw = cfg_kwargs(rec)
for its in (1, 10, 774):
    cfg = P.SolverConfig(**(kw | {"max_iters": its}))
    solve_from(inst, start, cfg)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        solve_from(inst, start, cfg)
        ts.append(time.perf_counter() - t0)
    print(its, "iterations: wall ms", round(statistics.median(ts) * 1e3, 3))
import cProfile, pstats  # noqa: E402
cfg = P.SolverConfig(**(kw | {"max_iters": 1}))
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    solve_from(inst, start, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
