"""One single-instance solve of a golden config (c1 / c2 / c5row) after one
warm-up solve: the second k_solve launch is the one to profile, e.g.
ncu -k regex:k_solve --launch-skip 1 --launch-count 1 python tools/solve_one.py c2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2508_13437_b200 import SolverConfig, tomo  # noqa: E402
from tests.golden_io import cfg_kwargs, load, named_A  # noqa: E402

nm = sys.argv[1] if len(sys.argv) > 1 else "c2"
rec = load(f"solve_{nm}")[0]
A = named_A(nm, rec)
sb = tomo.SliceBatch(A, rec["b"][None], rec["levels"], rec["idx0"][None])
cfg = SolverConfig(**cfg_kwargs(rec))
for _ in range(2):
    o = sb.solve(cfg, seeds=[int(cfg.seed)])
torch.cuda.synchronize()
sb.check_status()
print(nm, float(o["best_objective"][0]), float(rec["best_objective"]))
