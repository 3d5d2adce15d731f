"""Phase breakdown of single-instance solves (C1, C2 goldens) on one CTA:
microseconds per iteration and where the cycles go (diagnostic)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_13437_b200 import SolverConfig, tomo  # noqa: E402
from tests.golden_io import cfg_kwargs, load, named_A  # noqa: E402

PH = ["select+copy", "rand-destroy", "worst-destroy", "repair", "one_opt", "find_candidates", "swap_eval", "accept"]
EV = ["fc_calls", "fc_survivors", "swaps", "oo_exact", "oo_moves", "oo_windows", "impact", "refresh"]
if os.environ.get("FCPROF"):  # libamvm built with -DAMVM_FC_PROFILE: pc[8..13] = find_candidates sub-phase cycles
    EV = ["fc_select_rows", "fc_buckets_sort", "fc_staging", "fc_pass_total", "fc_drain", "fc_overflow_sort", "-", "-"]
for name in sys.argv[1:] or ["c1", "c2"]:
    rec = load(f"solve_{name}")[0]
    A = named_A(name, rec)
    sb = tomo.SliceBatch(A, rec["b"][None], rec["levels"], rec["idx0"][None])
    cfg = SolverConfig(**cfg_kwargs(rec))
    sb.solve(cfg, seeds=[cfg.seed]); sb.check_status()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    o = sb.solve(cfg, seeds=[cfg.seed])
    b.record(); torch.cuda.synchronize(); sb.check_status()
    ms = a.elapsed_time(b)
    it = int(o["iterations"][0])
    pc = o["phase_cycles"][0].cpu().numpy()
    tot = pc[:8].sum()
    print(json.dumps({"config": name, "iterations": it, "us_per_iteration": round(ms * 1e3 / it, 1),
                      "kcycles_per_iteration": round(tot / it / 1e3, 1),
                      "phase_share": {k: round(float(v / tot), 3) for k, v in zip(PH, pc[:8])},
                      "events_per_iteration": {k: round(float(v / it), 2) for k, v in zip(EV, pc[8:])},
                      "fc_calls_note": "with FCPROF these are cycles per iteration",
                      "best": float(o["best_objective"][0]), "golden_best": float(rec["best_objective"])}))
