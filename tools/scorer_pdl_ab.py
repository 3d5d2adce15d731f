"""A/B of programmatic dependent launch on the scorer's back-to-back
launches (bench.py's cycled measurement), alternating, in one process."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

dev = torch.device("cuda", 0)
X = np.random.default_rng(0).standard_normal((2048, 4096))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for rep in range(3):
    for p in ("1", "0"):
        os.environ["AMVM_SCORE_PDL"] = p
        r = bench.scorer_roofline(X, dev, flush, reps=5, batch=8)
        ro = r["roofline"]
        print(json.dumps({"pdl_env": p, "cycled_us": round(r["adjacent_cycled"]["ms_per_launch"] * 1e3, 2),
                          "with_best_us": round(ro["with_fused_best_move"]["ms_per_launch"] * 1e3, 2),
                          "forced_off_us": round(ro["without_pdl"]["ms_per_launch"] * 1e3, 2),
                          "host_issued_us": round(ro["host_issued_ms_per_launch"] * 1e3, 2)}), flush=True)
