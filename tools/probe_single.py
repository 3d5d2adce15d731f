"""Per-phase engine cycles of single-instance solves (C1, C2, C5 row) on one
CTA: where the latency of a lone instance goes."""
import sys
import time

import numpy as np

sys.path.insert(0, '/root/repo')
import torch  # noqa: E402

from paper_2508_13437_b200 import SolverConfig, tomo  # noqa: E402
from tests.golden_io import cfg_kwargs, load, named_A  # noqa: E402

names = ["select+copy", "rand-destroy", "worst-destroy", "repair", "one_opt", "find_candidates", "swap_eval", "accept"]
ev = ["fc_calls", "fc_survivors", "swaps", "oo_exact_scans", "oo_moves", "oo_windows", "impact_calls", "refreshes"]
for nm in ["c1", "c2", "c5row"]:
    rec = load(f"solve_{nm}")[0]
    A = named_A(nm, rec)
    sb = tomo.SliceBatch(A, rec["b"][None], rec["levels"], rec["idx0"][None])
    cfg = SolverConfig(**cfg_kwargs(rec))
    sb.solve(cfg, seeds=[int(cfg.seed)])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    o = sb.solve(cfg, seeds=[int(cfg.seed)])
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    pc = o["phase_cycles"].cpu().numpy()[0]
    tot = pc[:8].sum()
    print(nm, f"{dt * 1e3:.1f} ms", f"{tot / 1.965e6:.1f} ms busy", "best", float(o["best_objective"][0]),
          {k: round(float(v / tot), 3) for k, v in zip(names, pc[:8])}, dict(zip(ev, pc[8:16].tolist())), flush=True)
