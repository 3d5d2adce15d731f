"""bench.py's C3-slices leg alone (diagnostic)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

r = bench.c3_leg(torch.device("cuda", 0))
print(json.dumps({k: r[k] for k in ("value", "parity", "dense_engine", "device_ms")}))
