"""Launch the candidate-move scorer once per mode on the C5 shapes (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402

X, _ = bench.layer_rows(0, 1)
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
print(bench.scorer_roofline(X, dev, flush, reps=int(os.environ.get("REPS", "20")), batch=64))
